mkdir -p gpurun_out/r2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_zhp -c 1 -o gpurun_out/r2/zhp_p8_v4 -f python tools/run_step.py --p 8 --steps 1 > gpurun_out/r2/ncu_zhp8.log 2>&1; tail -3 gpurun_out/r2/ncu_zhp8.log
