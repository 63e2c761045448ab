# Session-5 closing run: the whole GPU suite on the final tree (incl. the mass-shape and every-row tests), smoke.
mkdir -p gpurun_out/s5e
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/s5e/gpu_tests.log 2>&1; tail -14 gpurun_out/s5e/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s5e/smoke.log 2>&1; tail -1 gpurun_out/s5e/smoke.log
