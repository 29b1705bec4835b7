mkdir -p gpurun_out/c35
ZPP_LN_NT=64 timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "norm" > gpurun_out/c35/k.log 2>&1; echo ktests64 rc=$?; tail -1 gpurun_out/c35/k.log
for e in 0 64 0 64; do echo "ZPP_LN_NT=$e"; ZPP_LN_NT=$e timeout 120 python tools/hbm_bench.py 2>&1 | head -2; done | tee gpurun_out/c35/hbm.txt
