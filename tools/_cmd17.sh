mkdir -p gpurun_out/c17
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "embedding or attention" > gpurun_out/c17/k.log 2>&1; echo ktests rc=$?; tail -3 gpurun_out/c17/k.log
timeout 900 python -m pytest tests/test_engine_gpu.py -q -x -k "early" > gpurun_out/c17/ab.log 2>&1; echo ab rc=$?; grep -E "passed|failed|FAIL|Error" gpurun_out/c17/ab.log | head -10
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c17/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c17/pytest.log
for sp in "1x1:8:2:1 --mb-size 1" "1x1:4:2:1 --mb-size 2" "1x1:8:2:1 --mb-size 2"; do
  timeout 600 python bench.py --no-cpu --split $sp > gpurun_out/c17/b.json 2> gpurun_out/c17/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/c17/b.json').read().strip().splitlines()[-1]); print('$sp', d['value'], d['ms_per_step'], d['clocks'], d['roofline']['achieved'], d['loss'], d['max_mem_gb'])" 2>&1 | tail -1 | tee -a gpurun_out/c17/mb.txt
done
