mkdir -p gpurun_out/r2o
PG_SPMV_PLANES=2 timeout 600 python tools/plane_debug.py > gpurun_out/r2o/debug.log 2>&1; echo "debug rc=$?"; head -120 gpurun_out/r2o/debug.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"plane_ring" -s 2 -c 1 -o gpurun_out/r2o/prof_plane_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2o/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r2o/ncu.log
