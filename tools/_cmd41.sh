mkdir -p gpurun_out/c41
for m in 0 12 16 0 12 16; do echo "== ZPP_LN_FWD_MINB=$m"; ZPP_LN_FWD_MINB=$m timeout 300 python tools/hbm_bench.py 2>&1 | grep layernorm_fwd; done > gpurun_out/c41/ln_fwd_minb.txt
ZPP_LN_FWD_MINB=12 timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "layernorm or rmsnorm" > gpurun_out/c41/tests12.txt 2>&1; echo rc12=$? >> gpurun_out/c41/tests12.txt
cat gpurun_out/c41/ln_fwd_minb.txt; tail -2 gpurun_out/c41/tests12.txt
