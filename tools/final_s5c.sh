# Session-5 third battery: every-row zero-row-sum invariant at full size (printed worst ratios), then the whole GPU suite.
mkdir -p gpurun_out/s5c
timeout 1500 python -m pytest tests/test_gpu_zfullsize.py -m gpu -q -s > gpurun_out/s5c/zfullsize.log 2>&1; grep -a "worst\|passed\|failed\|Error\|assert" gpurun_out/s5c/zfullsize.log | tail -30
timeout 1500 python -m pytest tests -m gpu -q --durations=10 --deselect tests/test_gpu_zfullsize.py > gpurun_out/s5c/gpu_tests_rest.log 2>&1; tail -3 gpurun_out/s5c/gpu_tests_rest.log
