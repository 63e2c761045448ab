for c in 1 2 3 4; do
  L=paper_1605_01238_b200/build/libwq_c$c.so
  echo "CPT $c"; WQ_LIB_DEBUG_PATH=$L timeout 600 python tools/time_kernels.py --p 4,6,7,8,9,10 --kernels 4 --reps 2 2>&1 | grep cfg | cut -c1-100
  WQ_LIB_DEBUG_PATH=$L timeout 600 python tools/time_kernels.py --p 6,8,10 --kernels 4 --reps 2 --matrix mass 2>&1 | grep cfg | cut -c1-100
done
