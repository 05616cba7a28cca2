# r01i A/B: warp-cooperative windowed producer vs single-lane producer (HEAD)
set -x
mkdir -p gpurun_out/r1i
for i in 1 2; do
PG_LIB_PATH=variants_tmp/base2/libpgmres.so python tools/spmv_bench.py --variants default --cases cfg4 2>&1 | tail -1
python tools/spmv_bench.py --variants default --cases cfg4 2>&1 | tail -1
done
timeout 900 python -m pytest tests -q -m "gpu" -x > gpurun_out/r1i/pytest_gpu_wp.log 2>&1; tail -2 gpurun_out/r1i/pytest_gpu_wp.log
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1i/bench_cfg4_wp.log 2>&1; tail -c 200 gpurun_out/r1i/bench_cfg4_wp.log
