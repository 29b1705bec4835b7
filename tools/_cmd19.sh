mkdir -p gpurun_out/c19
for sp in "1x1:4:1:1 --mb-size 4" "1x1:8:1:1 --mb-size 4" "1x1:8:2:1 --mb-size 2"; do
  timeout 600 python bench.py --no-cpu --split $sp > gpurun_out/c19/b.json 2> gpurun_out/c19/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/c19/b.json').read().strip().splitlines()[-1]); print('N1 $sp', d['value'], d['ms_per_step'], d['clocks'], d['roofline']['achieved'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1 | tee -a gpurun_out/c19/batch.txt
  tail -2 gpurun_out/c19/b.err
done
for N in 2 4; do
 if [ $N = 2 ]; then SP=2x1:8:4:2; else SP=2x2:8:4:2; fi
 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N \
   bench.py --gpus $N --split $SP --mb-size 4 --steps 5 --warmup 3 --no-cpu > gpurun_out/c19/bn$N.json 2> gpurun_out/c19/bn$N.err
 echo "N=$N rc=$?"
 python -c "
import json; d=json.loads(open('gpurun_out/c19/bn$N.json').read().strip().splitlines()[-1]); print('N$N $SP b4', d['value'], d['ms_per_step'], d['clocks'], d['exposed_comm_ms_per_step'], d['p2p_wait_ms_per_step'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1 | tee -a gpurun_out/c19/batch.txt
 tail -3 gpurun_out/c19/bn$N.err
done
