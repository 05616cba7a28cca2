mkdir -p gpurun_out/r2as
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"plane_ring" -s 2 -c 1 -o gpurun_out/r2as/prof_plane_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2as/ncu.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/r2as
cd tools; CASES=cfg4 timeout 200 python march_bench.py 2>&1 | tail -1; cd ..
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2as/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2as/pytest_gpu.log
