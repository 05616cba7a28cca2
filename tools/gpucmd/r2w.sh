mkdir -p gpurun_out/r2w
timeout 900 python -m pytest tests/test_gpu_planes.py -x -q > gpurun_out/r2w/pytest_planes.log 2>&1; echo "planes rc=$?"; tail -3 gpurun_out/r2w/pytest_planes.log | cut -c1-400
cd tools
export CASES=cfg4
timeout 200 python march_bench.py 2>&1 | tail -1
PG_PLANE_BOX=0 timeout 200 python march_bench.py 2>&1 | tail -1
cd ..
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"plane_ring" -s 2 -c 1 -o gpurun_out/r2w/prof_plane_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2w/ncu.log 2>&1; echo "ncu rc=$?"
