mkdir -p gpurun_out/c10
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c10/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c10/pytest.log
timeout 600 python bench.py --no-cpu > gpurun_out/c10/bench_aux.json 2> gpurun_out/c10/bench_aux.err; echo rc=$?; cat gpurun_out/c10/bench_aux.json | cut -c1-400
ZPP_AUX_STREAM=0 timeout 600 python bench.py --no-cpu > gpurun_out/c10/bench_noaux.json 2>&1; cat gpurun_out/c10/bench_noaux.json | cut -c1-400
timeout 300 python tools/profile_step.py > gpurun_out/c10/breakdown.txt 2>&1; head -30 gpurun_out/c10/breakdown.txt
