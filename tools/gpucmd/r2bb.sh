mkdir -p gpurun_out/r2bb
# launch list of one warm cfg4 solve (serialised, cold-cache per-launch times: shares only)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2bb/launches.csv python tools/profile_solve.py --config 4 > gpurun_out/r2bb/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 600 python tools/timeline.py --config 4 --out gpurun_out/r2bb/timeline_cfg4.json > gpurun_out/r2bb/timeline.log 2>&1; echo "timeline rc=$?"; tail -2 gpurun_out/r2bb/timeline.log | cut -c1-300
# the driver's launch form at one rank, and the reference arm
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r2bb/bench_torchrun1.log 2>&1; echo "torchrun rc=$?"; tail -c 400 gpurun_out/r2bb/bench_torchrun1.log
timeout 1500 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2bb/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 700 gpurun_out/r2bb/bench_ref.log
