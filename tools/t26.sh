for P in 4 5 6; do
for K in 3 4; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_zline|k_zhp" python tools/run_step.py --p $P --steps 1 --kernel $K 2>/dev/null | grep -E "k_zline|k_zhp" | awk -F'","' '{print $5, $NF}' | cut -c1-150 | sed "s/^/p$P k$K /"
done; done
