mkdir -p gpurun_out/c7
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off -k regex:gemm_tcgen05 --csv --log-file gpurun_out/c7/gemm_dram.csv python tools/profile_step.py --layers 2 --ncu --gemm-shapes gpurun_out/c7/gemm_shapes.csv > gpurun_out/c7/ncu.log 2>&1
echo ncu rc=$?
wc -l gpurun_out/c7/gemm_shapes.csv
