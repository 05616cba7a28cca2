# r02e: plane-marching kernel parity + ncu of one cfg4 march pass
mkdir -p gpurun_out/r2e
timeout 900 python -m pytest tests/test_gpu_march.py -x -q > gpurun_out/r2e/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2e/pytest.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sell_march" -s 3 -c 1 -o gpurun_out/r2e/march_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2e/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r2e/ncu.log
