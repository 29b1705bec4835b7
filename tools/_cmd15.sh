mkdir -p gpurun_out/c15
for e in 0 2 3; do echo "EMU=$e"; ZPP_ATTN_EMU=$e timeout 120 python tools/attn_bench.py 2>&1; done > gpurun_out/c15/attn_bench.txt; cat gpurun_out/c15/attn_bench.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/waits.py --gpus 4 > gpurun_out/c15/waits_2x2.txt 2>&1; echo rc=$?; grep -v "^\*\|OMP" gpurun_out/c15/waits_2x2.txt | head -70
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/waits.py --gpus 4 --split 1x4:8:2:1 > gpurun_out/c15/waits_1x4.txt 2>&1; echo rc=$?; grep -v "^\*\|OMP" gpurun_out/c15/waits_1x4.txt | head -70
for N in 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N \
   bench.py --gpus $N --steps 5 --warmup 3 --no-cpu > gpurun_out/c15/bench_n$N.json 2> gpurun_out/c15/bench_n$N.err
echo "N=$N rc=$?"; cut -c1-200 gpurun_out/c15/bench_n$N.json; grep -o '"exposed_comm_ms_per_step.\{0,60\}' gpurun_out/c15/bench_n$N.json; grep -o '"clocks.\{0,120\}' gpurun_out/c15/bench_n$N.json
ZPP_EARLY_OPT=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N \
   bench.py --gpus $N --steps 5 --warmup 3 --no-cpu > gpurun_out/c15/bench_n${N}_noearly.json 2> gpurun_out/c15/bench_n${N}_noearly.err
echo "N=$N noearly rc=$?"; cut -c1-200 gpurun_out/c15/bench_n${N}_noearly.json; grep -o '"exposed_comm_ms_per_step.\{0,60\}' gpurun_out/c15/bench_n${N}_noearly.json
done
