# z-line launches on forked streams (measurement switch WQ_ZL_FORK)
mkdir -p gpurun_out/s14
for F in 0 1 2; do
  WQ_ZL_FORK=$F timeout 600 python tools/time_kernels.py --p 2,3,4,6 --kernels 3 --reps 7 > gpurun_out/s14/fork_$F.jsonl 2>&1
  echo "== fork $F"; cut -c1-140 gpurun_out/s14/fork_$F.jsonl
done
WQ_ZL_FORK=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "uniform_lines or graph or repeatable or plane_ranges" > gpurun_out/s14/parity.log 2>&1; tail -2 gpurun_out/s14/parity.log
WQ_ZL_FORK=1 timeout 600 python tools/time_kernels.py --config C5 --p 4 --kernels 3 --reps 3 > gpurun_out/s14/c5_fork1.jsonl 2>&1
timeout 600 python tools/time_kernels.py --config C5 --p 4 --kernels 3 --reps 3 > gpurun_out/s14/c5_fork0.jsonl 2>&1
cut -c1-140 gpurun_out/s14/c5_*.jsonl
