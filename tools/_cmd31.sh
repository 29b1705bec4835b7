mkdir -p gpurun_out/c31
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "norm or colsum" > gpurun_out/c31/k.log 2>&1; echo ktests rc=$?; tail -2 gpurun_out/c31/k.log
timeout 120 python tools/hbm_bench.py > gpurun_out/c31/hbm_bench.txt 2>&1; head -5 gpurun_out/c31/hbm_bench.txt
timeout 300 python -m pytest tests/test_engine_gpu.py -q -x -k "single_gpu or llama" > gpurun_out/c31/e.log 2>&1; echo etests rc=$?; tail -1 gpurun_out/c31/e.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu > gpurun_out/c31/bench$i.json 2> gpurun_out/c31/bench$i.err
python -c "
import json; d=json.loads(open('gpurun_out/c31/bench$i.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['clocks'], d['roofline']['achieved'], d['loss'])"
done
