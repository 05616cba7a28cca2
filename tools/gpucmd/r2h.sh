mkdir -p gpurun_out/r2h
timeout 900 python -m pytest tests/test_gpu_march.py -x -q > gpurun_out/r2h/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2h/pytest.log
cd tools; timeout 300 python march_bench.py 2>&1 | tail -2; cd ..
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sell_march" -s 3 -c 1 -o gpurun_out/r2h/march_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2h/ncu.log 2>&1; echo "ncu rc=$?"
