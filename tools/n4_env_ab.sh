#!/bin/bash
# N=4 bench (P2 x D2 default split) under different environment settings, one JSON summary per setting.
# usage: tools/n4_env_ab.sh "VAR=value ..." ...   ("-" = unchanged environment)
mkdir -p gpurun_out
i=0
for env in "$@"; do
  [ "$env" = "-" ] && env=""
  env $env timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29700 + i)) bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu > gpurun_out/envab_$i.json 2> gpurun_out/envab_$i.err
  python - "$env" gpurun_out/envab_$i.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"{sys.argv[1] or 'default':32s} {d['value']:9.1f} tok/s  step {d['ms_per_step']:8.1f} ms  "
          f"exposed {d['exposed_comm_ms_per_step']:6.1f}  p2p {d['p2p_wait_ms_per_step']:6.1f}  gemm {d['roofline']['achieved']}")
except Exception as e:
    print(sys.argv[1], "no result", e)
PY
  i=$((i + 1))
done
