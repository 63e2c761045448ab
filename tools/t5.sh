mkdir -p gpurun_out/r2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_zhp -c 1 -o gpurun_out/r2/zhp2_p8 python tools/run_step.py --p 8 --steps 1 --kernel 4 > gpurun_out/r2/ncu_zhp2.log 2>&1; tail -3 gpurun_out/r2/ncu_zhp2.log
