mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_zfullsize.py -q -x -k "coef" 2>&1 | tail -2
for p in 2 3 4; do timeout 300 python tools/time_step.py --p $p --reps 7; done
timeout 300 python tools/time_step.py --config C5 --p 4 --reps 3
