for r in 1 2 3; do for nb in 1 2 3 4; do
  echo "R=$r NB=$nb"; WQ_ZHP_R=$r WQ_ZHP_NB=$nb timeout 300 python tools/time_kernels.py --p 8 --kernels 4 --reps 2 2>&1 | grep -v "^$" | cut -c1-120
done; done
for r in 1 2 3 4; do for nb in 2 4 6; do
  echo "R=$r NB=$nb"; WQ_ZHP_R=$r WQ_ZHP_NB=$nb timeout 300 python tools/time_kernels.py --p 4 --kernels 4 --reps 2 2>&1 | grep -v "^$" | cut -c1-120
done; done
