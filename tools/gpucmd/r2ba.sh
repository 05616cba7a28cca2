mkdir -p gpurun_out/r2ba
cd tools; for i in 1 2; do CASES=cfg4 timeout 300 python march_bench.py 2>&1 | tail -1; done; cd ..
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2ba/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2ba/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ba/smoke.log 2>&1; tail -1 gpurun_out/r2ba/smoke.log
timeout 900 python bench.py > gpurun_out/r2ba/bench_cfg4.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/r2ba/bench_cfg4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"plane_ring" -s 2 -c 1 -o gpurun_out/r2ba/prof_plane_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2ba/ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 python tools/degree_sweep.py --out gpurun_out/r2ba/cfg5_degree_sweep.json > gpurun_out/r2ba/cfg5_sweep.log 2>&1; echo "sweep rc=$?"; tail -6 gpurun_out/r2ba/cfg5_sweep.log | cut -c1-300
