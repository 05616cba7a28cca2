set -x
mkdir -p gpurun_out/master
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py -x -q > gpurun_out/master/pytest.log 2>&1; tail -3 gpurun_out/master/pytest.log
python tools/spmv_bench.py --variants default,nopat --cases cfg4,cfg2 > gpurun_out/master/spmv.jsonl 2>&1; cat gpurun_out/master/spmv.jsonl
PG_SPMV_MASTER=0 python tools/spmv_bench.py --variants default --cases cfg4,cfg2 > gpurun_out/master/spmv_nomaster.jsonl 2>&1; cat gpurun_out/master/spmv_nomaster.jsonl
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/master/bench_cfg4.log 2>&1; tail -c 200 gpurun_out/master/bench_cfg4.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/master/bench_cfg2.log 2>&1; tail -c 200 gpurun_out/master/bench_cfg2.log
