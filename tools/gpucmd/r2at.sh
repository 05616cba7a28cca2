mkdir -p gpurun_out/r2at
cd tools; CASES=cfg4 timeout 300 python march_bench.py 2>&1 | tail -3; cd ..
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2at/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2at/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2at/smoke.log 2>&1; tail -1 gpurun_out/r2at/smoke.log
timeout 900 python bench.py > gpurun_out/r2at/bench_cfg4.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/r2at/bench_cfg4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"plane_ring" -s 2 -c 1 -o gpurun_out/r2at/prof_plane_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2at/ncu.log 2>&1; echo "ncu rc=$?"
