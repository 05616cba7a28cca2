mkdir -p gpurun_out/r2ab
timeout 900 python -m pytest tests/test_gpu_planes.py -x -q > gpurun_out/r2ab/pytest_planes.log 2>&1; echo "planes rc=$?"; tail -3 gpurun_out/r2ab/pytest_planes.log | cut -c1-400
cd tools
export CASES=cfg4
timeout 150 python march_bench.py 2>&1 | tail -1
for v in u1 u6; do echo "== $v"; PG_LIB_PATH=../variants_tmp/$v/libpgmres.so timeout 150 python march_bench.py 2>&1 | tail -1; done
