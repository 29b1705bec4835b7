mkdir -p gpurun_out/c16
for e in 0 2 3; do echo "EMU=$e"; ZPP_ATTN_EMU=$e timeout 120 python tools/attn_bench.py 2>&1; done > gpurun_out/c16/attn_bench.txt; cat gpurun_out/c16/attn_bench.txt
timeout 900 python -m pytest tests/test_engine_gpu.py -q -x -k "early or multi_gpu" > gpurun_out/c16/ab_tests.log 2>&1; echo ab tests rc=$?; tail -5 gpurun_out/c16/ab_tests.log
for N in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N tools/comm_bench.py > gpurun_out/c16/comm_n$N.json 2> gpurun_out/c16/comm_n$N.err; echo comm N=$N rc=$?; cat gpurun_out/c16/comm_n$N.json
done
for e in 0 2; do
ZPP_ATTN_EMU=$e timeout 600 python bench.py --no-cpu > gpurun_out/c16/bench_emu$e.json 2> gpurun_out/c16/bench_emu$e.err
python -c "
import json; d=json.loads(open('gpurun_out/c16/bench_emu$e.json').read().strip().splitlines()[-1]); print('EMU=$e', d['value'], d['ms_per_step'], d['clocks'], d['roofline']['achieved'], d['loss'])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 \
   bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/c16/bench_n2.json 2> gpurun_out/c16/bench_n2.err
echo "N=2 rc=$?"; cut -c1-200 gpurun_out/c16/bench_n2.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 \
   bench.py --gpus 2 --split 1x2:8:2:1 --steps 5 --warmup 3 --no-cpu > gpurun_out/c16/bench_n2_1x2.json 2> gpurun_out/c16/bench_n2_1x2.err
echo "N=2 1x2 rc=$?"; cut -c1-200 gpurun_out/c16/bench_n2_1x2.json
