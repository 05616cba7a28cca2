# r01i A/B: windowed row-pattern stages without the epilogue operands (deeper ring)
set -x
for i in 1 2; do
for v in "" variants_tmp/epi0/libpgmres.so variants_tmp/epi0r256/libpgmres.so; do
PG_LIB_PATH=${v:-paper_1907_00072_b200/libpgmres.so} python tools/spmv_bench.py --variants default --cases cfg4 2>&1 | tail -1
done; done
PG_LIB_PATH=variants_tmp/epi0/libpgmres.so timeout 600 python -m pytest tests -q -m "gpu" -x -k "win or cfg4 or chain or spmv or poly" 2>&1 | tail -2
