# round-1 re-entry check r01i: smoke, GPU tests, default bench line
set -x
mkdir -p gpurun_out/r1i
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1i/smoke.log 2>&1; tail -2 gpurun_out/r1i/smoke.log
timeout 1200 python -m pytest tests -q -m "gpu" -x > gpurun_out/r1i/pytest_gpu.log 2>&1; tail -3 gpurun_out/r1i/pytest_gpu.log
python bench.py > gpurun_out/r1i/bench_cfg2.log 2>&1; tail -c 600 gpurun_out/r1i/bench_cfg2.log
