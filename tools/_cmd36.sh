mkdir -p gpurun_out/c36
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c36/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/c36/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c36/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/c36/smoke.log
timeout 900 python bench.py > gpurun_out/c36/bench.json 2> gpurun_out/c36/bench.err; echo bench rc=$?; cut -c1-200 gpurun_out/c36/bench.json
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N \
   bench.py --gpus $N > gpurun_out/c36/bench_n$N.json 2> gpurun_out/c36/bench_n$N.err
echo "N=$N rc=$?"; cut -c1-200 gpurun_out/c36/bench_n$N.json
done
