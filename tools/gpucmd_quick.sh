timeout 800 python -m pytest tests -q -m "gpu" -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python tools/cgs2_bench.py > gpurun_out/cgs2_bench.log 2>&1; cat gpurun_out/cgs2_bench.log
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; tail -c 1800 gpurun_out/bench_q.log
