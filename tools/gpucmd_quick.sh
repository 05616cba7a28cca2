timeout 800 python -m pytest tests -q -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep -E "^E |^FAILED" gpurun_out/pytest_gpu.log | head -8
python tools/spmv_bench.py 2>&1 | grep plain | cut -c1-90
python bench.py --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; grep -o '"value": [0-9.]*, "unit": "s", "n_gpus\|"median": [0-9.]*\|"frac": [0-9.]*\|"achieved": [0-9.]*\|"degree_effective": [0-9]*\|"iterations": [0-9]*' gpurun_out/bench_q.log | tr '\n' ' '; echo
