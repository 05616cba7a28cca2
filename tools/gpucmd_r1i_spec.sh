# r01i A/B: pattern kernel with speculative master gathers vs without
set -x
mkdir -p gpurun_out/r1i
for i in 1 2 3; do
PG_LIB_PATH=variants_tmp/nospec/libpgmres.so python tools/spmv_bench.py --variants default --cases cfg2 2>&1 | tail -1
python tools/spmv_bench.py --variants default --cases cfg2 2>&1 | tail -1
done
timeout 900 python -m pytest tests -q -m "gpu" -x > gpurun_out/r1i/pytest_gpu_spec.log 2>&1; tail -2 gpurun_out/r1i/pytest_gpu_spec.log
python bench.py --no-cpu-baseline > gpurun_out/r1i/bench_cfg2_spec.log 2>&1; tail -c 300 gpurun_out/r1i/bench_cfg2_spec.log
PG_LIB_PATH=variants_tmp/nospec/libpgmres.so python bench.py --no-cpu-baseline > gpurun_out/r1i/bench_cfg2_nospec.log 2>&1; tail -c 300 gpurun_out/r1i/bench_cfg2_nospec.log
