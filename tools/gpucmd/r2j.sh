mkdir -p gpurun_out/r2j
timeout 900 python -m pytest tests/test_gpu_dist_native.py tests/test_gpu_march.py tests/test_gpu_distributed.py -x -q > gpurun_out/r2j/pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/r2j/pytest.log
