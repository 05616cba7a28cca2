set -x
mkdir -p gpurun_out/launch
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch/launches_cfg2.csv python tools/profile_solve.py > gpurun_out/launch/ncu_launch.log 2>&1; tail -2 gpurun_out/launch/ncu_launch.log
