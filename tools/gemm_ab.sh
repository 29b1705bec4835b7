#!/bin/bash
# A/B of two libzpp builds on GEMM shapes: CUDA-event time, then ncu DRAM bytes per launch.
# usage: tools/gemm_ab.sh LIB_A LIB_B "M N K a_t b_t epi" ...
A=$1; B=$2; shift 2
mkdir -p gpurun_out
for shape in "$@"; do
  for L in $A $B; do
    echo "== $L $shape"
    ZPP_LIB_AB=$L python tools/gemm_one.py $shape
    ZPP_LIB_AB=$L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:gemm_tcgen05 -s 3 -c 1 --csv python tools/gemm_one.py $shape 2>/dev/null | grep -E "dram__bytes|gpu__time" | \
      awk -F'","' '{print "   " $(NF-2) " " $(NF-1) " " $NF}'
  done
done
