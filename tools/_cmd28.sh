mkdir -p gpurun_out/c28
timeout 300 python -m pytest tests/test_engine_gpu.py -q -x -k "cuda_graph" > gpurun_out/c28/g.log 2>&1; echo gtest rc=$?; grep -E "passed|failed|Error|error" gpurun_out/c28/g.log | head -20
for rep in 1 2; do
for g in 1 0; do
  ZPP_CUDA_GRAPH=$g timeout 600 python bench.py --no-cpu > gpurun_out/c28/b.json 2> gpurun_out/c28/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/c28/b.json').read().strip().splitlines()[-1]); print('graph=$g', d['value'], d['ms_per_step'], d['config']['cuda_graph'], d['e2e']['value'], d['gpu_launches'], d['clocks']['sm_mhz'], d['roofline']['achieved'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1 | tee -a gpurun_out/c28/ab.txt
  tail -3 gpurun_out/c28/b.err
done; done
