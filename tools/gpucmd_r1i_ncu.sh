# r01i: full ncu captures of the cfg4 windowed pattern pass (read raw here)
set -x
mkdir -p gpurun_out/r1i
ncu --set full --clock-control none --import-source on -k regex:"sell_win_kernel" -s 2 -c 1 -o gpurun_out/r1i/prof_win_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r1i/ncu_win.log 2>&1; tail -2 gpurun_out/r1i/ncu_win.log
