mkdir -p gpurun_out/ring
python tools/cgs2_bench.py --n 1000000,8000000 --k 13,25,40,51 --reps 10 > gpurun_out/ring/cgs2.jsonl 2>&1; grep -v gemv gpurun_out/ring/cgs2.jsonl
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ring/bench_cfg2.log 2>&1; tail -c 100 gpurun_out/ring/bench_cfg2.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ring/bench_cfg4.log 2>&1; tail -c 100 gpurun_out/ring/bench_cfg4.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/ring/pytest.log 2>&1; tail -1 gpurun_out/ring/pytest.log
