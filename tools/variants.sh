# Time variant libraries (tools/build_variant.py) against each other: tools/variants.sh "<time_kernels args>" name...
args=$1; shift
mkdir -p gpurun_out/var
for v in "$@"; do
  lib=paper_1605_01238_b200/build/libwq_$v.so
  for rep in 1 2; do
    WQ_LIB_DEBUG_PATH=$lib timeout 600 python tools/time_kernels.py $args 2>&1 | grep -v '^#' | sed "s/^/$v r$rep /"
  done
done | tee gpurun_out/var/variants.log
