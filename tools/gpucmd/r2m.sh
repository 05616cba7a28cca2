# r02m: evidence at HEAD after the session restart: full GPU suite, smoke, default
# bench (cfg4), reference arm, sanitizer sweep, cfg4 launch list, ncu full captures
set -x
mkdir -p gpurun_out/r2m
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m/smoke.log 2>&1; tail -2 gpurun_out/r2m/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2m/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2m/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/r2m/bench.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/r2m/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2m/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 1200 gpurun_out/r2m/bench_ref.log
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2m/launches_cfg4.csv python tools/profile_solve.py --config 4 > gpurun_out/r2m/ncu_launch.log 2>&1; echo "ncu launch rc=$?"; tail -2 gpurun_out/r2m/ncu_launch.log
ncu --set full --clock-control none --import-source on -k regex:"sell_win_kernel" -s 2 -c 1 -o gpurun_out/r2m/prof_win_cfg4 python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r2m/ncu_full_win.log 2>&1; echo "ncu win rc=$?"
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"tile_kernel|rows_kernel" -s 30 -c 3 -o gpurun_out/r2m/prof_cgs2_cfg4 python tools/profile_solve.py --config 4 --max-iters 40 > gpurun_out/r2m/ncu_full_cgs2.log 2>&1; echo "ncu cgs2 rc=$?"
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 1200 $S --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py tests/test_gpu_ilu.py tests/test_gpu_march.py \
    -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/r2m/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r2m/san_$tool.log
done
