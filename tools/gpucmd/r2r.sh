mkdir -p gpurun_out/r2r
cd tools
export CASES=cfg4
timeout 200 python march_bench.py 2>&1 | tail -1
for v in e1 e2 e8 e16 e24 mb3; do echo "== $v"; PG_LIB_PATH=../variants_tmp/$v/libpgmres.so timeout 150 python march_bench.py 2>&1 | tail -1; done
for s in 2 3; do PG_PLANE_STAGES=$s timeout 150 python march_bench.py 2>&1 | tail -1; done
