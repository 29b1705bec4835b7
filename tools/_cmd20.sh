mkdir -p gpurun_out/c20
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "norm or embed or attention" > gpurun_out/c20/k.log 2>&1; echo ktests rc=$?; tail -2 gpurun_out/c20/k.log
timeout 120 python tools/hbm_bench.py > gpurun_out/c20/hbm_bench.txt 2>&1; cat gpurun_out/c20/hbm_bench.txt
timeout 900 python bench.py > gpurun_out/c20/bench.json 2> gpurun_out/c20/bench.err; echo bench rc=$?; cut -c1-300 gpurun_out/c20/bench.json; tail -2 gpurun_out/c20/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/c20/bench_ref.json 2> gpurun_out/c20/bench_ref.err; echo ref rc=$?; cut -c1-300 gpurun_out/c20/bench_ref.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c20/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/c20/smoke.log
bash tools/profile_round_c.sh
