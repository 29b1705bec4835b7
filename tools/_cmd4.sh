mkdir -p gpurun_out/c4
export CUDA_MODULE_LOADING=EAGER
for mode in dp_outer zero1_outer; do
  mkdir -p gpurun_out/c4/$mode
  timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29541 tests/dist_worker.py 1 1 4 2 2 gpurun_out/c4/$mode 2 $mode > gpurun_out/c4/$mode.log 2>&1; echo "$mode rc=$?"; cat gpurun_out/c4/$mode/rank*.txt | cut -c1-300
done
timeout 300 python -m pytest tests/test_kernels_gpu.py -k "attention" -x -q 2>&1 | tail -2
timeout 300 python tools/attn_bench.py 2>&1 | tail -3
ZPP_ATTN_TRACE=1 timeout 120 python tools/attn_one.py > gpurun_out/c4/attn_trace.log 2>&1
head -4 gpurun_out/c4/attn_trace.log
