mkdir -p gpurun_out/c42
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c42/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/c42/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c42/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/c42/smoke.log
timeout 600 python bench.py > gpurun_out/c42/bench.json 2> gpurun_out/c42/bench.err; echo bench rc=$?; tail -1 gpurun_out/c42/bench.json | cut -c1-200
