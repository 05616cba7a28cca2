# r02b: reference-order degree decision -- new kernels + construction/solve parity tests
mkdir -p gpurun_out/r2b
timeout 1200 python -m pytest tests/test_gpu_blasorder.py tests/test_gpu_parity.py tests/test_gpu_cli.py -x -q -m "gpu and not slow" > gpurun_out/r2b/pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/r2b/pytest.log
