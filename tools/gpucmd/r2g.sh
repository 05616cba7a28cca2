mkdir -p gpurun_out/r2g
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sell_march" -s 3 -c 1 -o gpurun_out/r2g/march_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2g/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/r2g/ncu.log
