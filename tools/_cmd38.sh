mkdir -p gpurun_out/c38
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/c38/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/c38/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c38/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/c38/smoke.log
timeout 300 python tools/hbm_bench.py > gpurun_out/c38/hbm_bench.txt 2>&1
timeout 600 python bench.py > gpurun_out/c38/bench.json 2> gpurun_out/c38/bench.err; echo bench rc=$?; cut -c1-200 gpurun_out/c38/bench.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:layernorm_bwd_dx_pk -c 1 -o gpurun_out/c38/ln_bwd_pk python tools/hbm_bench.py > gpurun_out/c38/ncu.log 2>&1; echo ncu rc=$?
