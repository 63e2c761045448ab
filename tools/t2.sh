mkdir -p gpurun_out/r2
for cfg in "2 2 1" "2 2 2" "4 2 1" "4 4 1" "2 4 1" "4 2 2" "1 1 1"; do
  set -- $cfg
  echo "NB=$1 R=$2 CTAS=$3"
  WQ_ZHP_NB=$1 WQ_ZHP_R=$2 WQ_ZHP_CTAS=$3 timeout 300 python tools/time_kernels.py --p 4,8 --kernels 4 --reps 3 2>&1 | grep -v "^$"
done
