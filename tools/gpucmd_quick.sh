timeout 800 python -m pytest tests -q -m "gpu" -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep -E "^E " gpurun_out/pytest_gpu.log | head -5
for kv in 0 1; do
PG_SPMV_L2KEEP=$kv python bench.py --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; echo "L2KEEP=$kv"; grep -o '"value": [0-9.]*, "unit": "s", "n_gpus\|"median": [0-9.]*\|"max": [0-9.]*\|"frac": [0-9.]*' gpurun_out/bench_q.log | tr '\n' ' '; echo
done
PG_SPMV_L2KEEP=1 python tools/timeline.py > gpurun_out/timeline.log 2>&1; head -c 1500 gpurun_out/timeline.log
