mkdir -p gpurun_out/r2ao
timeout 3000 python -m pytest tests/test_gpu_checked.py -x -q > gpurun_out/r2ao/pytest_checked.log 2>&1; echo "checked rc=$?"; tail -30 gpurun_out/r2ao/pytest_checked.log | cut -c1-300
