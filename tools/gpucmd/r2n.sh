# r02n: plane-ring kernel: parity tests, pass timing vs the windowed kernel
mkdir -p gpurun_out/r2n
timeout 900 python -m pytest tests/test_gpu_planes.py -x -q > gpurun_out/r2n/pytest_planes.log 2>&1; echo "planes rc=$?"; tail -30 gpurun_out/r2n/pytest_planes.log
cd tools
for on in 0 1 2; do PG_SPMV_PLANES=$on timeout 300 python march_bench.py 2>&1 | tail -2; done
for q in 288 512; do PG_PLANE_Q=$q timeout 300 python march_bench.py 2>&1 | tail -2 | head -1; done
cd ..
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_march.py tests/test_gpu_chain.py -x -q > gpurun_out/r2n/pytest_more.log 2>&1; echo "more rc=$?"; tail -15 gpurun_out/r2n/pytest_more.log
