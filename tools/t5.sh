mkdir -p gpurun_out/r2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_zhp -c 1 -o gpurun_out/r2/zhp3_p8 python tools/run_step.py --p 8 --steps 1 --kernel 4 > gpurun_out/r2/ncu_zhp3.log 2>&1; tail -1 gpurun_out/r2/ncu_zhp3.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_zhp -c 1 -o gpurun_out/r2/zhp3_p4 python tools/run_step.py --p 4 --steps 1 --kernel 4 > gpurun_out/r2/ncu_zhp3b.log 2>&1; tail -1 gpurun_out/r2/ncu_zhp3b.log
