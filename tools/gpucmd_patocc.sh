mkdir -p gpurun_out/patocc
python tools/spmv_bench.py --variants default --cases cfg2 > gpurun_out/patocc/base.jsonl 2>&1; cut -c1-90 gpurun_out/patocc/base.jsonl
for v in pat5 pat6 pat8; do for bps in 4 5 6 8; do PG_SPMV_PAT_BLOCKS_PER_SM=$bps PG_LIB_PATH=variants_tmp/$v/libpgmres.so python tools/spmv_bench.py --variants default --cases cfg2 > gpurun_out/patocc/$v.$bps.jsonl 2>&1; echo "$v bps=$bps $(cut -c1-90 gpurun_out/patocc/$v.$bps.jsonl)"; done; done
