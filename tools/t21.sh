mkdir -p gpurun_out/r2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_coefz -c 1 -o gpurun_out/r2/coefz_v2 -f python tools/run_step.py --p 4 --steps 1 > gpurun_out/r2/ncu_coefz.log 2>&1; tail -3 gpurun_out/r2/ncu_coefz.log
