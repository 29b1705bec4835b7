mkdir -p gpurun_out/c23
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N \
   bench.py --gpus $N > gpurun_out/c23/bench_n$N.json 2> gpurun_out/c23/bench_n$N.err
echo "N=$N rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/c23/bench_n$N.json').read().strip().splitlines()[-1]); print('N$N', d['value'], d['ms_per_step'], d['config']['workload'], d['clocks'], d['exposed_comm_ms_per_step'], d['p2p_wait_ms_per_step'], d['e2e'], d['max_mem_gb'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N \
   bench.py --gpus $N --impl reference --steps 1 --warmup 0 > gpurun_out/c23/ref_n$N.json 2> gpurun_out/c23/ref_n$N.err
echo "ref N=$N rc=$?"; cut -c1-200 gpurun_out/c23/ref_n$N.json
done
timeout 900 python -m pytest tests/test_engine_gpu.py -q -x -k "multi_gpu or early" > gpurun_out/c23/mg.log 2>&1; echo mg rc=$?; tail -2 gpurun_out/c23/mg.log
