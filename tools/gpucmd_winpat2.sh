set -x
mkdir -p gpurun_out/winpat2
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"sell_win_kernel" -s 2 -c 1 -o gpurun_out/winpat2/prof_winpat_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/winpat2/ncu.log 2>&1; tail -2 gpurun_out/winpat2/ncu.log
