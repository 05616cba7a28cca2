mkdir -p gpurun_out/r2ax
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2ax/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2ax/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2ax/bench_cfg4.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/r2ax/bench_cfg4.log
