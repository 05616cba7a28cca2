mkdir -p gpurun_out/r2bp
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2bp/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2bp/ncu_bench.log 2>&1; echo "rc=$?"; wc -l gpurun_out/r2bp/launches_bench.csv
