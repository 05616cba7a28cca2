# r01i A/B: windowed ring counters (no per-row-block division) vs HEAD
set -x
mkdir -p gpurun_out/r1i
for i in 1 2; do
PG_LIB_PATH=variants_tmp/base/libpgmres.so python tools/spmv_bench.py --variants default --cases cfg4 2>&1 | tail -1
python tools/spmv_bench.py --variants default --cases cfg4 2>&1 | tail -1
done
timeout 900 python -m pytest tests -q -m "gpu" -x > gpurun_out/r1i/pytest_gpu_ab.log 2>&1; tail -2 gpurun_out/r1i/pytest_gpu_ab.log
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1i/bench_cfg4.log 2>&1; tail -c 300 gpurun_out/r1i/bench_cfg4.log
