# copy the round-end battery (tools/final_run.sh -> gpurun_out/final) into profiles/ (tracked)
set -e
F=gpurun_out/final
tail -n 1 $F/bench.json > profiles/r02_bench_line.json
tail -n 1 $F/ref.json > profiles/r02_reference_line.json
cp $F/launches.csv profiles/r02_launches_bench.csv
cat $F/time_kernels_stiff.jsonl $F/time_kernels_mass.jsonl > profiles/r02_auto_sweep.jsonl
cat $F/slab_c4p4.jsonl $F/slab_c4p8.jsonl $F/slab_c5.jsonl > profiles/r02_slab_scaling.jsonl
cp $F/time_step_p4.json profiles/r02_time_step_p4.json
cp $F/convergence_1d.json profiles/r02_convergence_1d.json
cp $F/zline_p4.ncu-rep profiles/r02_zline_p4.ncu-rep
cp $F/zhp_p8.ncu-rep profiles/r02_zhp_p8.ncu-rep
python tools/ncu_kernels_json.py $F/zline_p4.ncu-rep profiles/r02_zline_p4_summary.json "C4 p=4 stiffness z-line launches (uniform / interior / boundary lines), round 2 final" > /dev/null
python tools/ncu_kernels_json.py $F/zhp_p8.ncu-rep profiles/r02_zhp_p8_summary.json "C4 p=8 stiffness ZHP launches (interior / boundary lines), round 2 final" > /dev/null
python tools/ncu_kernels_json.py $F/coef_p4.ncu-rep profiles/r02_coef_p4_summary.json "C4 p=4 coefficient field (k_dnet, k_coefz), round 2 final" > /dev/null
python tools/ncu_sass_regions.py profiles/r02_zline_p4.ncu-rep --kernel "(int)4, (bool)0, (bool)1" > profiles/r02_zline_p4_sass_regions.txt
python tools/ncu_sass_regions.py profiles/r02_zline_p4.ncu-rep --kernel "(int)4, (bool)1" --top 8 >> profiles/r02_zline_p4_sass_regions.txt
python tools/ncu_sass_regions.py profiles/r02_zhp_p8.ncu-rep > profiles/r02_zhp_p8_sass_regions.txt
python tools/ncu_sass_regions.py $F/coef_p4.ncu-rep --kernel k_coefz > profiles/r02_coef_p4_sass_regions.txt
python - <<'PY'
import json
d = json.load(open("profiles/r02_zline_p4_summary.json"))
def gb(s):
    v, u = s.split()
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
t = sum(gb(k["dram__bytes_read.sum"]) + gb(k["dram__bytes_write.sum"]) for k in d["kernels"])
json.dump({"C4p4": t, "_source": "profiles/r02_zline_p4_summary.json: dram__bytes_read.sum + dram__bytes_write.sum over the three k_zline launches of one wq_assemble call (ncu --set full, round 2 final)"},
          open("profiles/ncu_traffic.json", "w"), indent=1)
print("traffic", t)
PY
