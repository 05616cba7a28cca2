for d in mb4_u8 mb6_u8 mb8_u4 mb6_u4 mb4_u4 mb8_u2; do
echo "== $d"; PG_LIB_PATH=$PWD/variants_tmp/$d/libpgmres.so python tools/spmv_bench.py 2>&1 | grep plain | cut -c1-110
done
