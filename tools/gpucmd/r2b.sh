mkdir -p gpurun_out/r2b
timeout 1200 python -m pytest tests/test_gpu_cli.py tests/test_gpu_blasorder.py -x -q -m "gpu" > gpurun_out/r2b/pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/r2b/pytest.log
