mkdir -p gpurun_out/r2bh
timeout 900 python bench.py --gpus 2 --dist-backend gloo --config 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2bh/bench_cfg2_gloo2.log 2>&1; echo "gloo2 cfg2 rc=$?"; tail -1 gpurun_out/r2bh/bench_cfg2_gloo2.log | cut -c1-400
timeout 1200 python bench.py --gpus 2 --dist-backend gloo --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2bh/bench_cfg4_gloo2.log 2>&1; echo "gloo2 cfg4 rc=$?"; tail -1 gpurun_out/r2bh/bench_cfg4_gloo2.log | cut -c1-400
