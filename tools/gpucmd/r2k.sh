mkdir -p gpurun_out/r2k
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2k/pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/r2k/pytest.log
