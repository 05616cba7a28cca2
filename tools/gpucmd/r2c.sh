# r02c: full GPU suite + default bench (cfg4) + 2-rank gloo bench through --gpus
mkdir -p gpurun_out/r2c
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r2c/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2c/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c/smoke.log 2>&1; tail -1 gpurun_out/r2c/smoke.log
timeout 1200 python bench.py > gpurun_out/r2c/bench.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/r2c/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2c/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 800 gpurun_out/r2c/bench_ref.log
timeout 900 python bench.py --gpus 2 --dist-backend gloo --config 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2c/bench_gloo2.log 2>&1; echo "gloo2 rc=$?"; tail -c 600 gpurun_out/r2c/bench_gloo2.log
