mkdir -p gpurun_out/c18
for sp in "1x1:16:2:1"; do
  timeout 600 python bench.py --no-cpu --split $sp --mb-size 2 > gpurun_out/c18/b.json 2> gpurun_out/c18/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/c18/b.json').read().strip().splitlines()[-1]); print('N1 $sp b2', d['value'], d['ms_per_step'], d['clocks'], d['roofline']['achieved'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1 | tee -a gpurun_out/c18/batch.txt
done
for N in 2 4; do
 if [ $N = 2 ]; then SP=2x1:16:8:2; else SP=2x2:16:8:2; fi
 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N \
   bench.py --gpus $N --split $SP --mb-size 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/c18/bn$N.json 2> gpurun_out/c18/bn$N.err
 echo "N=$N rc=$?"
 python -c "
import json; d=json.loads(open('gpurun_out/c18/bn$N.json').read().strip().splitlines()[-1]); print('N$N $SP b2', d['value'], d['ms_per_step'], d['clocks'], d['exposed_comm_ms_per_step'], d['p2p_wait_ms_per_step'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1 | tee -a gpurun_out/c18/batch.txt
 tail -3 gpurun_out/c18/bn$N.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29589 \
   bench.py --gpus 4 --split 1x4:8:2:1 --mb-size 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/c18/bn4_1x4.json 2> gpurun_out/c18/bn4_1x4.err
python -c "
import json; d=json.loads(open('gpurun_out/c18/bn4_1x4.json').read().strip().splitlines()[-1]); print('N4 1x4:8:2:1 b2', d['value'], d['ms_per_step'], d['clocks'], d['exposed_comm_ms_per_step'], d['p2p_wait_ms_per_step'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1 | tee -a gpurun_out/c18/batch.txt
