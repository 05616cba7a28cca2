mkdir -p gpurun_out/r2bn
timeout 2700 python -m pytest tests -q -m gpu -x > gpurun_out/r2bn/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2bn/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bn/smoke.log 2>&1; tail -1 gpurun_out/r2bn/smoke.log
timeout 900 python bench.py > gpurun_out/r2bn/bench_cfg4.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2bn/bench_cfg4.log | grep -o '"value": [0-9.]*\|"frac": [0-9.]*' | head -3 | paste -sd' '
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"plane_ring" -s 2 -c 1 -o gpurun_out/r2bn/prof_plane_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2bn/ncu.log 2>&1; echo "ncu rc=$?"
cd tools; CASES=cfg4 PINGPONG=1 timeout 300 python march_bench.py 2>&1 | tail -1 | grep -o '"us": [0-9.]*'; cd ..
