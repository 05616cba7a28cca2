cd tools
for v in old pipe0; do echo "== $v"; PG_LIB_PATH=../variants_tmp/$v/libpgmres.so timeout 300 python cgs2_bench.py --n 8000000 --k 12,19,30,45 2>&1 | grep -E "phase3|gemv"; done
echo "== new"; timeout 300 python cgs2_bench.py --n 8000000,1000000 --k 12,19,30,45 2>&1 | grep -E "phase"
