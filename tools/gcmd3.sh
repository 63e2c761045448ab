timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coef or zline or agree or slabs or form_host or (baseline_sampled and 5-C) or (full_parity_small and 5-3)" 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_coef -c 2 python tools/run_step.py --p 4 --steps 1 2>&1 | grep -E "duration"
