set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 800 python -m pytest tests -q -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench2.log 2>&1; tail -c 2500 gpurun_out/bench2.log
python tools/profile_solve.py > gpurun_out/prof_plain.log 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/profile_solve.py > gpurun_out/ncu_launch.log 2>&1; tail -3 gpurun_out/ncu_launch.log
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:sell_kernel -s 20 -c 2 -o gpurun_out/prof_poly python tools/profile_solve.py > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"tile_kernel|rows_kernel" -s 30 -c 3 -o gpurun_out/prof_cgs2 python tools/profile_solve.py > gpurun_out/ncu_full2.log 2>&1; tail -3 gpurun_out/ncu_full2.log
