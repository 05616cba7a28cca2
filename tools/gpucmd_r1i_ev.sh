# round-1 evidence refresh r01i (windowed ring counters, row-pattern stages without
# epilogue operands): tests, bench lines (cfg2 headline with CPU baseline,
# reference arm, cfg4, cfg3, roots / arnoldi variants), launch list + ncu full
# of the dominant kernels, timeline
set -x
mkdir -p gpurun_out/r1i
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1i/smoke.log 2>&1; tail -2 gpurun_out/r1i/smoke.log
timeout 900 python -m pytest tests -q -m "gpu" > gpurun_out/r1i/pytest_gpu.log 2>&1; tail -3 gpurun_out/r1i/pytest_gpu.log
python bench.py > gpurun_out/r1i/bench_cfg2.log 2>&1; tail -c 600 gpurun_out/r1i/bench_cfg2.log
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r1i/bench_ref_cfg2.log 2>&1; tail -c 400 gpurun_out/r1i/bench_ref_cfg2.log
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1i/bench_cfg4.log 2>&1; tail -c 300 gpurun_out/r1i/bench_cfg4.log
python bench.py --poly-form roots --no-cpu-baseline > gpurun_out/r1i/bench_cfg2_roots.log 2>&1; tail -c 300 gpurun_out/r1i/bench_cfg2_roots.log
python bench.py --construction arnoldi --poly-form roots --no-cpu-baseline > gpurun_out/r1i/bench_cfg2_arnoldi.log 2>&1; tail -c 300 gpurun_out/r1i/bench_cfg2_arnoldi.log
python bench.py --config 4 --construction arnoldi --poly-form roots --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1i/bench_cfg4_arnoldi.log 2>&1; tail -c 300 gpurun_out/r1i/bench_cfg4_arnoldi.log
python tools/timeline.py --config 2 --out gpurun_out/r1i/timeline_cfg2.json > /dev/null 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1i/launches_cfg2.csv python tools/profile_solve.py > gpurun_out/r1i/ncu_launch.log 2>&1; tail -2 gpurun_out/r1i/ncu_launch.log
ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"sell_pat_kernel<\(int\)1" -s 40 -c 2 -o gpurun_out/r1i/prof_poly_cfg2 python tools/profile_solve.py > gpurun_out/r1i/ncu_full.log 2>&1; tail -2 gpurun_out/r1i/ncu_full.log
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"tile_kernel|rows_kernel" -s 30 -c 3 -o gpurun_out/r1i/prof_cgs2_cfg2 python tools/profile_solve.py > gpurun_out/r1i/ncu_full2.log 2>&1; tail -2 gpurun_out/r1i/ncu_full2.log
ncu --set full --clock-control none --import-source on -k regex:"sell_win_kernel" -s 2 -c 1 -o gpurun_out/r1i/prof_win_cfg4_ev python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r1i/ncu_full3.log 2>&1; tail -2 gpurun_out/r1i/ncu_full3.log
python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r1i/bench_cfg3.log 2>&1; tail -c 200 gpurun_out/r1i/bench_cfg3.log
