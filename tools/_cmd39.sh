mkdir -p gpurun_out/c39
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c39/pytest_attn.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/c39/pytest_attn.log
for i in 1 2; do timeout 300 python tools/attn_bench.py 2 2048 32 128 >> gpurun_out/c39/attn_bench.txt 2>&1; done; cat gpurun_out/c39/attn_bench.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:attn_delta -c 3 --csv python tools/attn_bench.py 2 2048 32 128 > gpurun_out/c39/ncu_delta.csv 2>&1; echo ncu rc=$?
timeout 600 python bench.py > gpurun_out/c39/bench.json 2> gpurun_out/c39/bench.err; echo bench rc=$?; cut -c1-200 gpurun_out/c39/bench.json
