mkdir -p gpurun_out/c5
timeout 300 python -m pytest tests/test_kernels_gpu.py -k "attention" -x -q 2>&1 | tail -2
timeout 300 python tools/attn_bench.py 2>&1 | tail -3
ZPP_ATTN_TRACE=1 timeout 120 python tools/attn_one.py > gpurun_out/c5/attn_trace.log 2>&1
grep "fwd it" gpurun_out/c5/attn_trace.log | head -16
grep "^it" gpurun_out/c5/attn_trace.log | head -5
