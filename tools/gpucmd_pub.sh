set -x
mkdir -p gpurun_out/pub
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pub/pytest.log 2>&1; tail -2 gpurun_out/pub/pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/pub/bench_cfg2.log 2>&1; tail -c 150 gpurun_out/pub/bench_cfg2.log
PG_PUBLISH=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/pub/bench_cfg2_nopub.log 2>&1; tail -c 150 gpurun_out/pub/bench_cfg2_nopub.log
python tools/timeline.py --out gpurun_out/pub/timeline_cfg2.json > /dev/null 2>&1
