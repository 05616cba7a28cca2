python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 800 python -m pytest tests -q -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep -E "^E |^FAILED" gpurun_out/pytest_gpu.log | head -8
