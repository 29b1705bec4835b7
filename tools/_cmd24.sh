mkdir -p gpurun_out/c24
for rep in 1 2; do
for cfg in "ZPP_AUX_STREAM=1 ZPP_EARLY_OPT=1" "ZPP_AUX_STREAM=0 ZPP_EARLY_OPT=1" "ZPP_AUX_STREAM=1 ZPP_EARLY_OPT=0"; do
  env $cfg timeout 600 python bench.py --no-cpu > gpurun_out/c24/b.json 2> gpurun_out/c24/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/c24/b.json').read().strip().splitlines()[-1]); print('$cfg', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['power_w'], d['roofline']['achieved'], d['loss'])" | tee -a gpurun_out/c24/ab.txt
done; done
