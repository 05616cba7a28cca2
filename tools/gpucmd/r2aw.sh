cd tools
for v in dev1; do for i in 1 2; do echo "== $v"; PG_LIB_PATH=../variants_tmp/$v/libpgmres.so CASES=cfg4 timeout 300 python march_bench.py 2>&1 | tail -1; done; done
for s in 3 4 5; do PG_PLANE_STAGES=$s PG_LIB_PATH=../variants_tmp/dev1/libpgmres.so CASES=cfg4 timeout 300 python march_bench.py 2>&1 | tail -1; done
