# boundary-line launch time by kind of boundary line (measurement switch WQ_ZL_BND_FILTER; values invalid)
mkdir -p gpurun_out/r2
for F in none 0 1 2; do
  if [ $F = none ]; then unset WQ_ZL_BND_FILTER; else export WQ_ZL_BND_FILTER=$F; fi
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/bnd_$F.csv python tools/time_kernels.py --p ${ZL_P:-4,6} --kernels 3 --reps 1 > /dev/null 2>&1
  echo "== filter $F"; python tools/launch_summary.py gpurun_out/r2/bnd_$F.csv | grep "k_zline<., 1"
done
