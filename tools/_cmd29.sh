mkdir -p gpurun_out/c29
ZPP_GRAPH_DEBUG=1 ZPP_CUDA_GRAPH=1 timeout 600 python bench.py --no-cpu --steps 3 > gpurun_out/c29/b.json 2> gpurun_out/c29/b.err; echo rc=$?
cat gpurun_out/c29/b.json | cut -c1-300
grep -v "^ *$" gpurun_out/c29/b.err | grep -v "^  " | head -20
