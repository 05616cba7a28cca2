# r02f: march kernel v2 -- parity + pass timings (min-blocks variants, chunk sizes)
mkdir -p gpurun_out/r2f
timeout 900 python -m pytest tests/test_gpu_march.py -x -q > gpurun_out/r2f/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2f/pytest.log
cd tools
PG_SPMV_MARCH=0 timeout 300 python march_bench.py 2>&1 | tail -2
for z in 0 12 25; do PG_MARCH_Z=$z timeout 300 python march_bench.py 2>&1 | tail -2; done
for v in mb1 mb3; do PG_LIB_PATH=../variants_tmp/$v/libpgmres.so timeout 300 python march_bench.py 2>&1 | tail -2; done
