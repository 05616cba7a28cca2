timeout 900 python -m pytest tests -q -m "gpu" -k "spmv or poly" > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python tools/spmv_bench.py 2>&1 | grep plain | head -3 | cut -c1-90
