mkdir -p gpurun_out/r2aa
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2aa/smoke.log 2>&1; tail -1 gpurun_out/r2aa/smoke.log
timeout 900 python bench.py --config 2 --no-cpu-baseline > gpurun_out/r2aa/bench_cfg2.log 2>&1; echo "cfg2 rc=$?"; tail -c 400 gpurun_out/r2aa/bench_cfg2.log
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2aa/bench_cfg3.log 2>&1; echo "cfg3 rc=$?"; tail -c 300 gpurun_out/r2aa/bench_cfg3.log
timeout 900 python bench.py --construction arnoldi --poly-form roots --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2aa/bench_cfg4_arnoldi.log 2>&1; echo "arn rc=$?"; tail -c 300 gpurun_out/r2aa/bench_cfg4_arnoldi.log
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2aa/launches_cfg4.csv python tools/profile_solve.py --config 4 > gpurun_out/r2aa/ncu_launch.log 2>&1; echo "ncu launch rc=$?"; tail -1 gpurun_out/r2aa/ncu_launch.log
python tools/timeline.py --config 4 --out gpurun_out/r2aa/timeline_cfg4.json > gpurun_out/r2aa/timeline.log 2>&1; echo "timeline rc=$?"; tail -3 gpurun_out/r2aa/timeline.log
