timeout 800 python -m pytest tests -q -m "gpu" -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep -E "^E |^FAILED" gpurun_out/pytest_gpu.log | head -5
python tools/cgs2_bench.py > gpurun_out/cgs2_ring.log 2>&1; echo RING; grep -v gemv gpurun_out/cgs2_ring.log
PG_CGS2_CHUNK_KMAX=0 python tools/cgs2_bench.py > gpurun_out/cgs2_ring0.log 2>&1; echo RING-ALL-K; grep -E '"k": 10' gpurun_out/cgs2_ring0.log | grep -v gemv
python bench.py --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; grep -o '"value": [0-9.]*, "unit": "s", "n_gpus\|"median": [0-9.]*\|"frac": [0-9.]*' gpurun_out/bench_q.log | tr '\n' ' '; echo
