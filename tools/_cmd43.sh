mkdir -p gpurun_out/c43
timeout 1000 python -m pytest tests -m gpu -q > gpurun_out/c43/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/c43/pytest.log
