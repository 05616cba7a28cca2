timeout 900 python -m pytest tests -q -m "gpu" -k "spmv or poly or solve" > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log; grep -E "^E |^FAILED" gpurun_out/pytest_gpu.log | head -5
for bp in 3 4 6; do echo "== pipe bp$bp"; PG_SPMV_DICT_BLOCKS_PER_SM=$bp python tools/spmv_bench.py 2>&1 | grep plain | head -2 | cut -c1-90; done
echo "== nopipe"; PG_SPMV_DICT_PIPE=0 python tools/spmv_bench.py 2>&1 | grep plain | head -2 | cut -c1-90
