# r01i A/B: row-pattern windowed stages of 1024 / 768 rows with two rows per row thread
set -x
mkdir -p gpurun_out/r1i
for i in 1 2; do
for v in "" variants_tmp/r1024/libpgmres.so variants_tmp/r768/libpgmres.so; do
PG_LIB_PATH=${v:-paper_1907_00072_b200/libpgmres.so} python tools/spmv_bench.py --variants default --cases cfg4 2>&1 | tail -1
done; done
PG_LIB_PATH=variants_tmp/r1024/libpgmres.so timeout 900 python -m pytest tests -q -m "gpu" -x > gpurun_out/r1i/pytest_gpu_r1024.log 2>&1; tail -2 gpurun_out/r1i/pytest_gpu_r1024.log
timeout 900 python -m pytest tests -q -m "gpu" -x > gpurun_out/r1i/pytest_gpu_def.log 2>&1; tail -2 gpurun_out/r1i/pytest_gpu_def.log
