#!/bin/bash
# A/B of the column-reduction split target (ZPP_CR_WAVES) on the HBM kernel microbenchmark,
# plus the kernel parity tests that cover colred (LN/RMSNorm param grads, bias colsum).
mkdir -p gpurun_out
for w in 2 4 8; do
  echo "== ZPP_CR_WAVES=$w" >> gpurun_out/r01d_colred_ab.txt
  ZPP_CR_WAVES=$w timeout 300 python tools/hbm_bench.py >> gpurun_out/r01d_colred_ab.txt 2>&1
done
for w in 2 4; do
  ZPP_CR_WAVES=$w timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "layernorm or rmsnorm or colsum" \
    >> gpurun_out/r01d_colred_tests.txt 2>&1
  echo "waves=$w rc=$?" >> gpurun_out/r01d_colred_tests.txt
done
