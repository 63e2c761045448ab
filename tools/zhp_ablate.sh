mkdir -p gpurun_out/r2
for A in 0 1 2 3 7; do for P in 8; do
 echo "abl=$A" ; WQ_ZHP_ABLATE=$A timeout 300 python tools/time_kernels.py --p $P --kernels 4 --reps 2 2>&1 | cut -c1-160
done; done > gpurun_out/r2/zhp_abl.txt
for A in 0 1 2 3; do echo "mass abl=$A"; WQ_ZHP_ABLATE=$A timeout 300 python tools/time_kernels.py --p 4,8 --kernels 4 --reps 2 --matrix mass 2>&1 | cut -c1-160; done >> gpurun_out/r2/zhp_abl.txt
cat gpurun_out/r2/zhp_abl.txt
