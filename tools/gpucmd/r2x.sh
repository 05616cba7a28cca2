cd tools
export CASES=cfg4
for v in rpt4 rt256 rt192; do echo "== $v"; PG_LIB_PATH=../variants_tmp/$v/libpgmres.so timeout 150 python march_bench.py 2>&1 | tail -1; done
PG_PLANE_Q=896 PG_LIB_PATH=../variants_tmp/rpt4/libpgmres.so timeout 150 python march_bench.py 2>&1 | tail -1
PG_PLANE_Q=768 PG_LIB_PATH=../variants_tmp/rt192/libpgmres.so timeout 150 python march_bench.py 2>&1 | tail -1
for q in 512 576; do PG_PLANE_Q=$q timeout 150 python march_bench.py 2>&1 | tail -1; done
