# Round-end GPU battery: full GPU tests, smoke, bench line, launch list, ncu captures of the headline
# assembly (z-line, C4 p=4), ZHP (C4 p=8) and the coefficient field.
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/final/gpu_tests.log 2>&1; tail -3 gpurun_out/final/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; tail -c 300 gpurun_out/final/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/ref.json 2> gpurun_out/final/ref.err; tail -c 300 gpurun_out/final/ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/final/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_zline -c 3 -o gpurun_out/final/zline_p4 python tools/run_step.py --p 4 --steps 1 > gpurun_out/final/ncu_full.log 2>&1; tail -1 gpurun_out/final/ncu_full.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_zhp -c 2 -o gpurun_out/final/zhp_p8 python tools/run_step.py --p 8 --steps 1 > gpurun_out/final/ncu_zhp.log 2>&1; tail -1 gpurun_out/final/ncu_zhp.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_coefz|k_dnet" -c 2 -o gpurun_out/final/coef_p4 python tools/run_step.py --p 4 --steps 1 > gpurun_out/final/ncu_coef.log 2>&1; tail -1 gpurun_out/final/ncu_coef.log
timeout 600 python studies/convergence_1d.py --out gpurun_out/final/convergence_1d.json > /dev/null 2>&1; ls -la gpurun_out/final/convergence_1d.json
timeout 900 python tools/time_step.py --p 4 --reps 7 > gpurun_out/final/time_step_p4.json 2>&1
timeout 1800 python tools/time_kernels.py --p 2,3,4,5,6,7,8,9,10 --kernels 0 --reps 3 > gpurun_out/final/time_kernels_stiff.jsonl 2>&1
timeout 1800 python tools/time_kernels.py --p 2,3,4,5,6,7,8,9,10 --kernels 0 --reps 3 --matrix mass > gpurun_out/final/time_kernels_mass.jsonl 2>&1
timeout 1800 python tools/time_slab.py --p 4 > gpurun_out/final/slab_c4p4.jsonl 2>&1
timeout 1800 python tools/time_slab.py --p 8 --reps 2 > gpurun_out/final/slab_c4p8.jsonl 2>&1
timeout 1800 python tools/time_slab.py --config C5 --p 4 --reps 2 > gpurun_out/final/slab_c5.jsonl 2>&1
ls -la gpurun_out/final/
