mkdir -p gpurun_out/c12
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N \
   bench.py --gpus $N --steps 5 --warmup 3 --no-cpu > gpurun_out/c12/bench_n$N.json 2> gpurun_out/c12/bench_n$N.err
echo "N=$N rc=$?"; cut -c1-300 gpurun_out/c12/bench_n$N.json; tail -3 gpurun_out/c12/bench_n$N.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29520 \
   bench.py --gpus 4 --split 1x4:8:2:1 --steps 5 --warmup 3 --no-cpu > gpurun_out/c12/bench_n4_1x4.json 2> gpurun_out/c12/bench_n4_1x4.err
echo "1x4 rc=$?"; cut -c1-300 gpurun_out/c12/bench_n4_1x4.json
