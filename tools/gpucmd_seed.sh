mkdir -p gpurun_out/seed
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/seed/pytest.log 2>&1; tail -1 gpurun_out/seed/pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/seed/bench_cfg2.log 2>&1; tail -c 100 gpurun_out/seed/bench_cfg2.log
