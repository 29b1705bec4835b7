mkdir -p gpurun_out/c20
timeout 900 python bench.py > gpurun_out/c20/bench.json 2> gpurun_out/c20/bench.err; echo bench rc=$?; cut -c1-300 gpurun_out/c20/bench.json; tail -2 gpurun_out/c20/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/c20/bench_ref.json 2> gpurun_out/c20/bench_ref.err; echo ref rc=$?; cut -c1-300 gpurun_out/c20/bench_ref.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c20/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/c20/smoke.log
bash tools/profile_round_c.sh
