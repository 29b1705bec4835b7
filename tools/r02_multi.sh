#!/bin/bash
# 4-GPU verification: full GPU test suite, N=2 / N=4 bench lines, NCCL bandwidth of the stage-sized AG / RS / P2P
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02_pytest_gpu_4gpu_final.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_gpu_4gpu_final.log
timeout 900 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu \
  > gpurun_out/r02_bench_n2.json 2> gpurun_out/r02_bench_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu \
  > gpurun_out/r02_bench_n4.json 2> gpurun_out/r02_bench_n4.err
cut -c1-250 gpurun_out/r02_bench_n2.json gpurun_out/r02_bench_n4.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 \
  tools/comm_bench.py > gpurun_out/r02_comm_n4.json 2> gpurun_out/r02_comm_n4.err; tail -2 gpurun_out/r02_comm_n4.json
