#!/bin/bash
# A/B library: the current sources with csrc/spmm_simt.cu replaced by build_ab/spmm_simt_base.cu
# -> build_ab/libnmspmm_base.so (select with NM_LIB_PATH in timing scripts)
set -e
cd "$(dirname "$0")/.."
P=paper_2503_01253_b200
ARCH="-gencode arch=compute_100a,code=sm_100a"
objs=""
for f in $P/csrc/*.cu; do
  src=$f; [ "$(basename $f)" = spmm_simt.cu ] && src=build_ab/spmm_simt_base.cu
  o=build_ab/$(basename $f).o
  cp $src build_ab/_tmp_$(basename $f)
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include -I $P/csrc -c build_ab/_tmp_$(basename $f) -o $o &
  objs="$objs $o"
done
wait
nvcc $ARCH -shared -o build_ab/libnmspmm_base.so $objs -lcudart
rm -f build_ab/_tmp_*
