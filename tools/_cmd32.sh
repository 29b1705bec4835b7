mkdir -p gpurun_out/c32
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/c32/k.log 2>&1; echo ktests rc=$?; tail -1 gpurun_out/c32/k.log
timeout 120 python tools/attn_bench.py 2 2048 32 128 2>&1 | tee gpurun_out/c32/attn_bench.txt
timeout 300 python -m pytest tests/test_engine_gpu.py -q -x -k "single_gpu or llama" > gpurun_out/c32/e.log 2>&1; echo etests rc=$?; tail -1 gpurun_out/c32/e.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu > gpurun_out/c32/bench$i.json 2> gpurun_out/c32/bench$i.err
python -c "
import json; d=json.loads(open('gpurun_out/c32/bench$i.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['clocks'], d['roofline']['achieved'], d['loss'])"
done
