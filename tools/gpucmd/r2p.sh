mkdir -p gpurun_out/r2p
timeout 900 python -m pytest tests/test_gpu_planes.py -x -q > gpurun_out/r2p/pytest_planes.log 2>&1; echo "planes rc=$?"; tail -30 gpurun_out/r2p/pytest_planes.log | cut -c1-300
cd tools
for on in 1 2; do PG_SPMV_PLANES=$on timeout 300 python march_bench.py 2>&1 | tail -2; done
for q in 288 512 576; do PG_PLANE_Q=$q timeout 300 python march_bench.py 2>&1 | tail -2 | head -1; done
PG_PLANE_STAGES=3 timeout 300 python march_bench.py 2>&1 | tail -2 | head -1
cd ..
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"plane_ring" -s 2 -c 1 -o gpurun_out/r2p/prof_plane_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2p/ncu.log 2>&1; echo "ncu rc=$?"
