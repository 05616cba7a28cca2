mkdir -p gpurun_out/r2i
timeout 900 python -m pytest tests/test_gpu_march.py -x -q > gpurun_out/r2i/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2i/pytest.log
cd tools; timeout 300 python march_bench.py 2>&1 | tail -2
for v in d1 d2mb1; do PG_LIB_PATH=../variants_tmp/$v/libpgmres.so timeout 300 python march_bench.py 2>&1 | tail -2; done
