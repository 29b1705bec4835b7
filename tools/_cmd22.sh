mkdir -p gpurun_out/c22
for cfg in "2 2x1:16:8:4" "4 2x2:16:8:4" "4 4x1:32:8:2"; do
 set -- $cfg; N=$1; SP=$2
 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29601 \
   bench.py --gpus $N --split $SP:2 --steps 5 --warmup 3 --no-cpu > gpurun_out/c22/b.json 2> gpurun_out/c22/b.err
 echo "N=$N $SP rc=$?"
 python -c "
import json; d=json.loads(open('gpurun_out/c22/b.json').read().strip().splitlines()[-1]); print('N$N $SP b2', d['value'], d['ms_per_step'], d['clocks'], d['exposed_comm_ms_per_step'], d['p2p_wait_ms_per_step'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1 | tee -a gpurun_out/c22/splits.txt
 tail -2 gpurun_out/c22/b.err
done
