# ZHP iteration battery: parity tests touching ZHP, kernel timings
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_zfullsize.py -m gpu -q -x -k "${PYTEST_K:-ZHP or zhp or 4- or uniform or graded or slabs or repeatable or coefficients}" > gpurun_out/r2/zhp_tests.log 2>&1; tail -3 gpurun_out/r2/zhp_tests.log
VARIANTS="${VARIANTS}" bash tools/zhp_variants.sh
