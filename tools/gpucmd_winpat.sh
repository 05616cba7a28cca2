set -x
mkdir -p gpurun_out/winpat
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py -x -q > gpurun_out/winpat/pytest.log 2>&1; tail -3 gpurun_out/winpat/pytest.log
python tools/spmv_bench.py --variants default,nopat --cases cfg4,cfg2 > gpurun_out/winpat/spmv.jsonl 2>&1; cat gpurun_out/winpat/spmv.jsonl
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/winpat/bench_cfg4.log 2>&1; tail -c 400 gpurun_out/winpat/bench_cfg4.log
PG_SPMV_WINPAT=0 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/winpat/bench_cfg4_pair.log 2>&1; tail -c 200 gpurun_out/winpat/bench_cfg4_pair.log
