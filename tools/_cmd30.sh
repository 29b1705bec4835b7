mkdir -p gpurun_out/c30
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c30/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c30/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c30/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/c30/smoke.log
timeout 900 python bench.py > gpurun_out/c30/bench.json 2> gpurun_out/c30/bench.err; echo bench rc=$?; cut -c1-250 gpurun_out/c30/bench.json
