#!/bin/bash
# usage: tools/n4_sweep.sh "ENV=..." ...   (runs bench at N=4 under each env setting)
for env in "$@"; do
  env $env timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/sweep.json 2> gpurun_out/sweep.err
  echo "== $env rc=$?"
  python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/sweep.json").read().strip().splitlines()[-1])
    print(d["value"], d["ms_per_step"], d["exposed_comm_ms_per_step"], d["p2p_wait_ms_per_step"], d["roofline"]["achieved"])
except Exception as e:
    print("no result", e)
    print(open("gpurun_out/sweep.err").read()[-800:])
PY
done
