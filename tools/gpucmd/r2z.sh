mkdir -p gpurun_out/r2z
timeout 1200 python bench.py > gpurun_out/r2z/bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/r2z/bench.log
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2z/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2z/pytest_gpu.log
