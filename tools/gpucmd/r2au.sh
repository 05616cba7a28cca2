mkdir -p gpurun_out/r2au
cd tools
for i in 1 2; do CASES=cfg4 timeout 300 python march_bench.py 2>&1 | tail -1; done
PG_PLANE_VEC=0 CASES=cfg4 timeout 300 python march_bench.py 2>&1 | tail -1
cd ..
timeout 1500 python -m pytest tests/test_gpu_planes.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2au/pytest_planes.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2au/pytest_planes.log
