mkdir -p gpurun_out/c40
timeout 600 python bench.py > gpurun_out/c40/bench_n1.json 2> gpurun_out/c40/bench_n1.err; echo bench n1 rc=$?
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $N > gpurun_out/c40/bench_n$N.json 2> gpurun_out/c40/bench_n$N.err; echo bench n$N rc=$?
done
timeout 600 python bench.py --impl reference > gpurun_out/c40/bench_ref_n1.json 2> gpurun_out/c40/bench_ref_n1.err; echo ref rc=$?
for f in gpurun_out/c40/*.json; do echo $f; tail -1 $f | cut -c1-160; done
