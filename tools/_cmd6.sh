mkdir -p gpurun_out/c6
timeout 300 python tools/gemm_shapes_bench.py > gpurun_out/c6/gemm_shapes.log 2>&1; cat gpurun_out/c6/gemm_shapes.log
timeout 600 python bench.py > gpurun_out/c6/bench_n1.json 2> gpurun_out/c6/bench_n1.err; echo bench rc=$?; cat gpurun_out/c6/bench_n1.json
