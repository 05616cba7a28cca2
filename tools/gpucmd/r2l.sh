mkdir -p gpurun_out/r2l
timeout 600 python -m pytest tests/test_gpu_roots.py -q -m gpu > gpurun_out/r2l/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2l/pytest.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2l/bench.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/r2l/bench.log
