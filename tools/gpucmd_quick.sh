timeout 800 python -m pytest tests -q -m "gpu" -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep -E "^E |^FAILED" gpurun_out/pytest_gpu.log | head -5
for p in 1 0; do PG_PDL=$p python bench.py --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; echo "PDL=$p"; grep -o '"value": [0-9.]*, "unit": "s", "n_gpus\|"median": [0-9.]*\|"frac": [0-9.]*' gpurun_out/bench_q.log | tr '\n' ' '; echo; done
python tools/timeline.py > gpurun_out/timeline.log 2>&1; grep -E "span_us|busy_us|idle_us" gpurun_out/timeline.log
