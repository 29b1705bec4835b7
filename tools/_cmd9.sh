mkdir -p gpurun_out/c9
ncu --set full --import-source on --clock-control none -k regex:"attn_bwd_d|attn_fwd_tc" -c 3 -o gpurun_out/c9/attn_split python tools/attn_one.py > gpurun_out/c9/ncu.log 2>&1
echo rc=$?
