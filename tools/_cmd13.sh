mkdir -p gpurun_out/c13
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/c13/attn_tests.log 2>&1; echo attn tests rc=$?; tail -5 gpurun_out/c13/attn_tests.log
timeout 120 python tools/attn_bench.py 2>&1 | tee gpurun_out/c13/attn_bench.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c13/pytest.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/c13/pytest.log
timeout 600 python bench.py --no-cpu > gpurun_out/c13/bench.json 2> gpurun_out/c13/bench.err; echo bench rc=$?; cut -c1-400 gpurun_out/c13/bench.json; tail -3 gpurun_out/c13/bench.err
ZPP_EARLY_OPT=0 timeout 600 python bench.py --no-cpu > gpurun_out/c13/bench_noearly.json 2> gpurun_out/c13/bench_noearly.err; echo bench rc=$?; cut -c1-300 gpurun_out/c13/bench_noearly.json
