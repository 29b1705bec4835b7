mkdir -p gpurun_out/c33
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_tcgen05 -s 2 -c 12 \
    -o gpurun_out/c33/gemm_full python tools/profile_step.py --layers 2 --ncu > gpurun_out/c33/ncu_gemm.log 2>&1
echo "gemm full rc=$?"; tail -3 gpurun_out/c33/ncu_gemm.log
ls -la gpurun_out/c33
