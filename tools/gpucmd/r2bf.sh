mkdir -p gpurun_out/r2bf
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2bf/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2bf/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bf/smoke.log 2>&1; tail -1 gpurun_out/r2bf/smoke.log
timeout 900 python bench.py > gpurun_out/r2bf/bench_cfg4.log 2>&1; echo "bench rc=$?"; tail -c 300 gpurun_out/r2bf/bench_cfg4.log
timeout 900 python bench.py --impl reference > gpurun_out/r2bf/bench_ref_cfg4.log 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/r2bf/bench_ref_cfg4.log
for c in 2 5 3; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2bf/bench_cfg$c.log 2>&1; echo "cfg$c rc=$?"; tail -1 gpurun_out/r2bf/bench_cfg$c.log | cut -c1-200; done
