set -x
mkdir -p gpurun_out/winpat3
python tools/spmv_bench.py --variants default --cases cfg4 > gpurun_out/winpat3/spmv.jsonl 2>&1; cat gpurun_out/winpat3/spmv.jsonl
for v in tb3 tb2 mb3; do PG_LIB_PATH=variants_tmp/$v/libpgmres.so python tools/spmv_bench.py --variants default --cases cfg4 > gpurun_out/winpat3/spmv_$v.jsonl 2>&1; cat gpurun_out/winpat3/spmv_$v.jsonl; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"sell_win_kernel" -s 2 -c 1 -o gpurun_out/winpat3/prof_winpat_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/winpat3/ncu.log 2>&1; tail -1 gpurun_out/winpat3/ncu.log
