# per-rank slab step times, cost- vs nnz-balanced cuts
mkdir -p gpurun_out/r2
out=gpurun_out/r2/slabs_balance.jsonl; : > $out
for B in cost nnz; do
  timeout 900 python tools/time_slab.py --config C5 --p 4 --world ${W:-4,8} --reps 2 --balance $B >> $out 2>&1
  timeout 600 python tools/time_slab.py --p 4 --world ${W:-4,8} --reps 3 --balance $B >> $out 2>&1
  timeout 900 python tools/time_slab.py --p 8 --world ${W:-4,8} --reps 2 --balance $B >> $out 2>&1
done
cut -c1-330 $out
