mkdir -p gpurun_out/c14
./tools/tmem_rate > gpurun_out/c14/tmem_rate.txt 2>&1; cat gpurun_out/c14/tmem_rate.txt
./tools/mma_rate > gpurun_out/c14/mma_rate.txt 2>&1; cat gpurun_out/c14/mma_rate.txt
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/c14/attn_tests.log 2>&1; echo attn tests rc=$?; tail -3 gpurun_out/c14/attn_tests.log
for e in 0 2 3; do echo "EMU=$e"; ZPP_ATTN_EMU=$e timeout 120 python tools/attn_bench.py 2>&1 | head -2; done | tee gpurun_out/c14/attn_bench.txt
for rep in 1 2; do
for cfg in "ZPP_EARLY_OPT=1 ZPP_ATTN_IMPL=0" "ZPP_EARLY_OPT=0 ZPP_ATTN_IMPL=0" "ZPP_EARLY_OPT=1 ZPP_ATTN_IMPL=2"; do
  env $cfg timeout 600 python bench.py --no-cpu > gpurun_out/c14/b.json 2> gpurun_out/c14/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/c14/b.json').read().strip().splitlines()[-1]); print('$cfg', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['achieved'], d['loss'])" | tee -a gpurun_out/c14/ab.txt
done; done
