for m in 7 0 3 4; do
  L=paper_1605_01238_b200/build/libwq_u$m.so; [ $m = 7 ] && L=paper_1605_01238_b200/libwq.so
  echo "U $m"; WQ_LIB_DEBUG_PATH=$L timeout 400 python tools/time_kernels.py --p 4,6,8 --kernels 4 --reps 3 2>&1 | grep cfg | cut -c1-100
done
