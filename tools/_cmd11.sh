mkdir -p gpurun_out/c11
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c11/pytest.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/c11/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c11/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/c11/smoke.log
timeout 900 python bench.py > gpurun_out/c11/bench.json 2> gpurun_out/c11/bench.err; echo bench rc=$?; cut -c1-600 gpurun_out/c11/bench.json; tail -5 gpurun_out/c11/bench.err
timeout 300 python tools/profile_step.py > gpurun_out/c11/breakdown.txt 2>&1; head -40 gpurun_out/c11/breakdown.txt
