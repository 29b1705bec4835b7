mkdir -p gpurun_out/c34
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
   --log-file gpurun_out/c34/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/c34/ncu_bench.log 2>&1
echo "ncu bench rc=$?"; tail -2 gpurun_out/c34/ncu_bench.log; ls -la gpurun_out/c34
