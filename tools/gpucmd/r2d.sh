# r02d: plane-marching kernel -- parity + pass timing vs the windowed kernel
mkdir -p gpurun_out/r2d
timeout 900 python -m pytest tests/test_gpu_march.py -x -q > gpurun_out/r2d/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2d/pytest.log
cd tools
PG_SPMV_MARCH=0 timeout 300 python march_bench.py 2>&1 | tail -2
for z in 0 8 25 50 100; do PG_MARCH_Z=$z timeout 300 python march_bench.py 2>&1 | tail -2; done
