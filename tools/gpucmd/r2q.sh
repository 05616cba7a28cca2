mkdir -p gpurun_out/r2q
timeout 900 python -m pytest tests/test_gpu_planes.py -x -q > gpurun_out/r2q/pytest_planes.log 2>&1; echo "planes rc=$?"; tail -3 gpurun_out/r2q/pytest_planes.log | cut -c1-300
cd tools
export CASES=cfg4
timeout 300 python march_bench.py 2>&1 | tail -1
for v in e1 e2 e3 e4 e5 e7 mb3; do echo "== $v"; PG_LIB_PATH=../variants_tmp/$v/libpgmres.so timeout 300 python march_bench.py 2>&1 | tail -1; done
for s in 2 3 4; do PG_PLANE_STAGES=$s timeout 300 python march_bench.py 2>&1 | tail -1; done
