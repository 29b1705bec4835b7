#!/bin/bash
# A/B of the packed-row LayerNorm variants (ZPP_LN_PK=1) on the HBM microbenchmark and
# the LN / RMSNorm kernel parity tests with the variant on; then the N=1 bench with each.
mkdir -p gpurun_out
for pk in 0 1 0 1; do
  echo "== ZPP_LN_PK=$pk" >> gpurun_out/r01d_ln_pk_ab.txt
  ZPP_LN_PK=$pk timeout 300 python tools/hbm_bench.py 4096 4096 >> gpurun_out/r01d_ln_pk_ab.txt 2>&1
done
ZPP_LN_PK=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "layernorm or rmsnorm" > gpurun_out/r01d_ln_pk_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/r01d_ln_pk_tests.txt
for pk in 1 0; do
  ZPP_LN_PK=$pk timeout 600 python bench.py > gpurun_out/r01d_bench_lnpk$pk.json 2> gpurun_out/r01d_bench_lnpk$pk.err
done
