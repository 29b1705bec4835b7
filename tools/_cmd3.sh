mkdir -p gpurun_out/c3
export CUDA_MODULE_LOADING=EAGER
( ZPP_DEBUG_SYNC=1 timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29540 tests/dist_worker.py 1 1 4 2 2 gpurun_out/c3 2 dp_outer > gpurun_out/c3/dp_outer.log 2>&1; echo rc=$? >> gpurun_out/c3/dp_outer.log )
timeout 300 python tools/attn_bench.py > gpurun_out/c3/attn_bench.log 2>&1
ZPP_ATTN_TRACE=1 timeout 120 python tools/attn_one.py > gpurun_out/c3/attn_trace.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -k "rmsnorm or swiglu or rope or attention or llama or single" -x -q > gpurun_out/c3/pytest.log 2>&1; echo rc=$? >> gpurun_out/c3/pytest.log
tail -3 gpurun_out/c3/pytest.log; cat gpurun_out/c3/attn_bench.log; tail -5 gpurun_out/c3/dp_outer.log
