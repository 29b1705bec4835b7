#!/bin/bash
# End-of-round verification on a 4-GPU box: smoke, the full GPU test suite, the default N=1 bench
# line (with its CPU baseline) and the reference arm, then N=2 / N=4 bench lines.
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_final_smoke.log 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/r02_final_smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02_final_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02_final_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02_final_bench_n1.json 2> gpurun_out/r02_final_bench_n1.err
echo "bench n1 rc=$?"; cut -c1-300 gpurun_out/r02_final_bench_n1.json
timeout 900 python bench.py --impl reference > gpurun_out/r02_final_bench_ref.json 2> gpurun_out/r02_final_bench_ref.err
echo "bench ref rc=$?"; cut -c1-300 gpurun_out/r02_final_bench_ref.json
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29620 + n)) bench.py --gpus $n --steps 10 --warmup 3 --no-cpu \
    > gpurun_out/r02_final_bench_n$n.json 2> gpurun_out/r02_final_bench_n$n.err
  echo "bench n$n rc=$?"; cut -c1-300 gpurun_out/r02_final_bench_n$n.json
done
