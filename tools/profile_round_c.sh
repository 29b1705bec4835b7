#!/bin/bash
# r01c evidence for profiles/: launch list of one full GPT-6.2B step (ncu, cold/serialised),
# ncu --set full of the attention kernels (fwd2, dkdv, dq) and of the adamw / embedding kernels.
mkdir -p gpurun_out/prof_c
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/prof_c/launches_step32.csv python tools/profile_step.py --ncu > gpurun_out/prof_c/ncu_list.log 2>&1
echo "launch list rc=$?"
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"attn_" -c 6 \
    -o gpurun_out/prof_c/attn_full python tools/profile_step.py --layers 2 --ncu > gpurun_out/prof_c/ncu_attn.log 2>&1
echo "attn full rc=$?"
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"adamw|embed_bwd|layernorm_bwd" -c 5 \
    -o gpurun_out/prof_c/misc_full python tools/profile_step.py --layers 2 --ncu > gpurun_out/prof_c/ncu_misc.log 2>&1
echo "misc full rc=$?"
ls -la gpurun_out/prof_c
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:gemm_tcgen05 --csv \
    --clock-control none --profile-from-start off --log-file gpurun_out/prof_c/gemm_traffic.csv \
    python tools/profile_step.py --layers 2 --ncu --gemm-shapes gpurun_out/prof_c/gemm_shapes.csv > gpurun_out/prof_c/ncu_gemm_traffic.log 2>&1
echo "gemm traffic rc=$?"
python tools/gemm_traffic.py gpurun_out/prof_c/gemm_traffic.csv gpurun_out/prof_c/gemm_shapes.csv gpurun_out/prof_c/gemm_traffic.json
timeout 300 python tools/profile_step.py > gpurun_out/prof_c/breakdown.txt 2>&1; head -30 gpurun_out/prof_c/breakdown.txt
