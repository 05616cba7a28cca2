# re-entry validation: smoke, GPU tests, headline bench
set -x
mkdir -p gpurun_out/r1e
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1e/smoke.log 2>&1; tail -2 gpurun_out/r1e/smoke.log
timeout 900 python -m pytest tests -q -m "gpu" > gpurun_out/r1e/pytest_gpu.log 2>&1; tail -3 gpurun_out/r1e/pytest_gpu.log
python bench.py > gpurun_out/r1e/bench_cfg2.log 2>&1; tail -c 600 gpurun_out/r1e/bench_cfg2.log
