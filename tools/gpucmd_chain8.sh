mkdir -p gpurun_out/chain8
timeout 600 python -m pytest tests/test_gpu_chain.py -x -q > gpurun_out/chain8/pytest.log 2>&1; tail -2 gpurun_out/chain8/pytest.log
python tools/chain_bench.py --tag master --settings "chain=0;chain=1,ts=1;chain=1,ts=2;chain=1,ts=4;chain=1,ts=8" > gpurun_out/chain8/master.jsonl 2>&1; cat gpurun_out/chain8/master.jsonl
