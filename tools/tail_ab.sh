mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py -m gpu -q --timeout 600 -k "early_optimizer or multi" > gpurun_out/tail_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/tail_tests.log
bash tools/run_matrix.sh r02_tail "4|--steps 10 --warmup 3" "4|--steps 10 --warmup 3 --rt overlap_tail=False" "2|--steps 10 --warmup 3" "2|--steps 10 --warmup 3 --rt overlap_tail=False" "4|--steps 10 --warmup 3"
