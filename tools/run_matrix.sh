#!/bin/bash
# Run bench.py over a list of configurations, one JSON line each, into gpurun_out/<tag>_*.json.
# usage: tools/run_matrix.sh TAG "GPUS|ARGS" ["GPUS|ARGS" ...]
#   e.g. tools/run_matrix.sh r02_c3sweep "4|--split 2x2:8:8:2:2" "4|--split 2x2:16:8:2:2"
TAG=$1; shift
mkdir -p gpurun_out
i=0
for spec in "$@"; do
  n=${spec%%|*}; args=${spec#*|}
  out=gpurun_out/${TAG}_$i.json
  if [ "$n" = "1" ]; then
    timeout 1500 python bench.py --gpus 1 --no-cpu $args > $out 2> $out.err
  else
    timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + i)) bench.py --gpus $n --no-cpu $args > $out 2> $out.err
  fi
  echo "== [$n] $args rc=$?"; tail -1 $out | cut -c1-400
  i=$((i + 1))
done
