timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "zline or agree or slabs or form_host or (baseline_sampled and 5-C) or (full_parity_small and 5-3)" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -8
WQ_DEBUG=1 timeout 200 python tools/time_kernels.py --p 2,3,4 --kernels 0 2>&1 | tail -4
