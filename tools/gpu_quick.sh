# quick GPU battery: parity + sgq + convergence tests (no full-size), smoke
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sgq.py tests/test_convergence_1d.py -m gpu -q --durations=15 -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/r2/gpu_quick.log 2>&1; tail -40 gpurun_out/r2/gpu_quick.log
