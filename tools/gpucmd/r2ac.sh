mkdir -p gpurun_out/r2ac
timeout 900 python -m pytest tests/test_gpu_planes.py -x -q > gpurun_out/r2ac/pytest_planes.log 2>&1; echo "planes rc=$?"; tail -2 gpurun_out/r2ac/pytest_planes.log | cut -c1-400
cd tools; CASES=cfg4 timeout 150 python march_bench.py 2>&1 | tail -1; cd ..
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"plane_ring" -s 2 -c 1 -o gpurun_out/r2ac/prof_plane_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2ac/ncu.log 2>&1; echo "ncu rc=$?"
timeout 1200 python bench.py > gpurun_out/r2ac/bench.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/r2ac/bench.log | cut -c1-600
