#!/bin/bash
# attention kernels: correctness tests, timing at the bench shapes, one ncu --set full of the backward
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -k "attention" -q -x --timeout 120 > gpurun_out/attn_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/attn_tests.log
tail -3 gpurun_out/attn_tests.log
for a in "2 2048 32 128" "1 2048 32 128" "1 4096 32 128" "2 2048 40 128"; do timeout 60 python tools/attn_bench.py $a; done
if [ "$1" = "ncu" ]; then
  ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 4 -c 2 -o gpurun_out/attnbwd \
    python tools/attn_bench.py 2 2048 32 128 > gpurun_out/ncu_attn.log 2>&1; tail -2 gpurun_out/ncu_attn.log
fi
