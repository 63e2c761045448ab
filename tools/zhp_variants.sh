# time the ZHP kernel for measurement variants (tools/build_variant.py) against the default build
mkdir -p gpurun_out/r2
out=gpurun_out/r2/zhp_variants.txt; : > $out
for V in default ${VARIANTS:-spa0 spa1}; do
  if [ $V = default ]; then unset WQ_LIB_DEBUG_PATH; else export WQ_LIB_DEBUG_PATH=paper_1605_01238_b200/build/libwq_$V.so; fi
  echo "== $V" >> $out
  timeout 600 python tools/time_kernels.py --p ${ZP_S:-5,7,8,10} --kernels 4 --reps 2 2>&1 | cut -c1-120 >> $out
  timeout 600 python tools/time_kernels.py --p ${ZP_M:-4,6,8,10} --kernels 4 --reps 2 --matrix mass 2>&1 | cut -c1-120 >> $out
done
unset WQ_LIB_DEBUG_PATH
cat $out
