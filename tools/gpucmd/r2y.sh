cd tools
export CASES=cfg4
timeout 150 python march_bench.py 2>&1 | tail -1
for v in e32 e8 e40; do echo "== $v"; PG_LIB_PATH=../variants_tmp/$v/libpgmres.so timeout 150 python march_bench.py 2>&1 | tail -1; done
