set -x
mkdir -p gpurun_out/master2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py -x -q > gpurun_out/master2/pytest.log 2>&1; tail -2 gpurun_out/master2/pytest.log
python tools/spmv_bench.py --variants default --cases cfg4,cfg2,cfg5 > gpurun_out/master2/spmv.jsonl 2>&1; cut -c1-120 gpurun_out/master2/spmv.jsonl
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/master2/bench_cfg4.log 2>&1; tail -c 200 gpurun_out/master2/bench_cfg4.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/master2/bench_cfg2.log 2>&1; tail -c 200 gpurun_out/master2/bench_cfg2.log
