timeout 200 python -m pytest tests/test_kernels_gpu.py -k "attention" -x -q 2>&1 | tail -3
timeout 120 python tools/attn_bench.py 2>&1 | tail -3
ZPP_ATTN_BWD_FUSED=1 timeout 120 python tools/attn_bench.py 2>&1 | tail -2 | head -1
timeout 120 python tools/attn_bench.py 1 4096 32 128 2>&1 | head -1
timeout 300 python -m pytest tests/test_engine_gpu.py -k "single or llama" -x -q 2>&1 | tail -2
