mkdir -p gpurun_out/r2u
timeout 900 python -m pytest tests/test_gpu_planes.py -x -q > gpurun_out/r2u/pytest_planes.log 2>&1; echo "planes rc=$?"; tail -3 gpurun_out/r2u/pytest_planes.log | cut -c1-400
cd tools
export CASES=cfg4
timeout 200 python march_bench.py 2>&1 | tail -1
for v in rt256 rpt2 rt160; do echo "== $v"; PG_LIB_PATH=../variants_tmp/$v/libpgmres.so timeout 150 python march_bench.py 2>&1 | tail -1; done
for q in 640 768 896; do PG_PLANE_Q=$q timeout 150 python march_bench.py 2>&1 | tail -1; done
