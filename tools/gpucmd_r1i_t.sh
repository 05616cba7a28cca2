# r01i: GPU tests + cfg4 pass after the row-pattern stage change
set -x
mkdir -p gpurun_out/r1i
timeout 900 python -m pytest tests -q -m "gpu" -x > gpurun_out/r1i/pytest_gpu_t.log 2>&1; tail -2 gpurun_out/r1i/pytest_gpu_t.log
python tools/spmv_bench.py --variants default --cases cfg4,cfg2 2>&1 | tail -2
