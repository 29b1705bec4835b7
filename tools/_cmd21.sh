mkdir -p gpurun_out/c21
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x > gpurun_out/c21/k.log 2>&1; echo ktests rc=$?; tail -2 gpurun_out/c21/k.log
timeout 120 python tools/attn_bench.py 1 2048 32 128 2>&1 | tee gpurun_out/c21/attn_bench.txt
timeout 120 python tools/attn_bench.py 2 2048 32 128 2>&1 | tee -a gpurun_out/c21/attn_bench.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:gemm_tcgen05 --csv \
    --clock-control none --profile-from-start off --log-file gpurun_out/c21/gemm_traffic.csv \
    python tools/profile_step.py --layers 2 --ncu --gemm-shapes gpurun_out/c21/gemm_shapes.csv > gpurun_out/c21/ncu_gemm_traffic.log 2>&1
python tools/gemm_traffic.py gpurun_out/c21/gemm_traffic.csv gpurun_out/c21/gemm_shapes.csv gpurun_out/c21/gemm_traffic.json
for i in 1 2; do
timeout 600 python bench.py --no-cpu > gpurun_out/c21/bench$i.json 2> gpurun_out/c21/bench$i.err
python -c "
import json; d=json.loads(open('gpurun_out/c21/bench$i.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['clocks'], d['roofline'], d['loss'])"
done
