nproc; python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo rc=$?; tail -c 1500 gpurun_out/bench_ref.log
