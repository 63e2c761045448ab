# ZHP launch-parameter sweep (rows per step R, pipeline depth D) at C4
mkdir -p gpurun_out/r2
for R in 1 2 3 4; do for D in 2 3; do
 echo "stiff p=8 R=$R D=$D $(WQ_ZHP_R=$R WQ_ZHP_D=$D timeout 300 python tools/time_kernels.py --p 8 --kernels 4 --reps 2 2>&1 | cut -c1-110)"
done; done > gpurun_out/r2/zhp_sweep.txt
for R in 2 3 4 6; do
 echo "mass p=8 R=$R $(WQ_ZHP_R=$R timeout 300 python tools/time_kernels.py --p 8 --kernels 4 --reps 2 --matrix mass 2>&1 | cut -c1-110)"
 echo "stiff p=10 R=$R $(WQ_ZHP_R=$R timeout 300 python tools/time_kernels.py --p 10 --kernels 4 --reps 1 2>&1 | cut -c1-110)"
done >> gpurun_out/r2/zhp_sweep.txt
cat gpurun_out/r2/zhp_sweep.txt
