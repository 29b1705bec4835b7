#!/bin/bash
# HBM-kernel A/B: tools/hbm_bench.py at several (T, h) with the current build and with $LIB_B
for sh in "4096 4096" "4096 2048" "8192 4096" "4096 5120"; do
  echo "== T h = $sh"
  timeout 60 python tools/hbm_bench.py $sh 2>&1 | grep -E "^norm_param|^colsum"
  ZPP_LIB_AB=$LIB_B timeout 60 python tools/hbm_bench.py $sh 2>&1 | grep -E "^norm_param|^colsum" | sed "s/^/  old /"
done
