# round-1 evidence set: bench line (with CPU baseline), launch list + ncu full of the fused pass and CGS2, timeline
python bench.py > gpurun_out/bench_r01.log 2>&1; tail -c 3500 gpurun_out/bench_r01.log
python tools/timeline.py --out gpurun_out/timeline_r01.json > gpurun_out/timeline_r01.log 2>&1
python tools/profile_solve.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/profile_solve.py > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:sell_kernel -s 40 -c 3 -o gpurun_out/prof_poly python tools/profile_solve.py > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"tile_kernel|rows_kernel|chunk" -s 150 -c 3 -o gpurun_out/prof_cgs2 python tools/profile_solve.py > gpurun_out/ncu_full2.log 2>&1; tail -1 gpurun_out/ncu_full2.log
