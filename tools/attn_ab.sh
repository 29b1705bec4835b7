#!/bin/bash
# attention backward A/B: correctness tests on the current build, then timing of the current
# build ("cur") against the libraries named in $LIBS (builds of other variants, see `make variant`)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -k "attention" -q -x --timeout 120 > gpurun_out/attn_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/attn_tests.log
tail -3 gpurun_out/attn_tests.log
for a in "2 2048 32 128" "1 4096 32 128" "2 2048 40 128"; do
  for r in 1 2; do
    for L in cur $LIBS; do
      echo -n "$L "
      if [ $L = cur ]; then timeout 60 python tools/attn_bench.py $a; else ZPP_LIB_AB=$L timeout 60 python tools/attn_bench.py $a; fi
    done
  done
done
if [ "$1" = "ncu" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_bwd -s 6 -c 4 --csv \
    python tools/attn_bench.py 2 2048 32 128 > gpurun_out/ncu_attn_launch.csv 2>&1
  ncu --set full --clock-control none --import-source on -k regex:attn_bwd_dkdv -s 3 -c 1 -o gpurun_out/attnbwd2 \
    python tools/attn_bench.py 2 2048 32 128 > gpurun_out/ncu_attn.log 2>&1; tail -2 gpurun_out/ncu_attn.log
fi
