#!/bin/bash
# Evidence for profiles/: kernel breakdown of one full GPT-6.2B step, the ncu launch list of
# one step, and ncu --set full captures of the top kernels.  Run under gpurun (one GPU).
set -x
mkdir -p gpurun_out/prof
python tools/profile_step.py > gpurun_out/prof/breakdown.txt 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/prof/launches_step32.csv python tools/profile_step.py --ncu > gpurun_out/prof/ncu_list.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_tcgen05 -s 8 -c 8 \
    -o gpurun_out/prof/gemm_full python tools/profile_step.py --layers 2 --ncu > gpurun_out/prof/ncu_gemm.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:attn_ -c 4 \
    -o gpurun_out/prof/attn_full python tools/profile_step.py --layers 2 --ncu > gpurun_out/prof/ncu_attn.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"adamw|colred|layernorm" -c 6 \
    -o gpurun_out/prof/hbm_full python tools/profile_step.py --layers 2 --ncu > gpurun_out/prof/ncu_hbm.log 2>&1
ls -la gpurun_out/prof
