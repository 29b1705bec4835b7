mkdir -p gpurun_out/c37
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/c37/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/c37/pytest.log
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N > gpurun_out/c37/bench_n$N.json 2> gpurun_out/c37/bench_n$N.err; echo bench n$N rc=$?; cut -c1-200 gpurun_out/c37/bench_n$N.json
done
