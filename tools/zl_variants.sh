# time the z-line kernel for measurement variants (tools/build_variant.py) against the default build
mkdir -p gpurun_out/r2
out=gpurun_out/r2/zl_variants.txt; : > $out
for V in default ${VARIANTS}; do
  if [ $V = default ]; then unset WQ_LIB_DEBUG_PATH; else export WQ_LIB_DEBUG_PATH=paper_1605_01238_b200/build/libwq_$V.so; fi
  echo "== $V $(timeout 600 python tools/time_kernels.py --p ${ZL_P:-4} --kernels 3 --reps 5 2>&1 | cut -c1-120)" >> $out
done
unset WQ_LIB_DEBUG_PATH
cat $out
