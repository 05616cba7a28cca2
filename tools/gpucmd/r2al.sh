mkdir -p gpurun_out/r2al
cd tools
for env in "PG_CGS2_TMA=0" "PG_CGS2_TMA=1"; do echo "== $env"; env $env timeout 300 python cgs2_bench.py --n 8000000,1000000 --k 8,12,19,25,30,45 2>&1 | grep -E "phase" > ../gpurun_out/r2al/cgs2_$env.jsonl; cat ../gpurun_out/r2al/cgs2_$env.jsonl | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['n']//1000000}M/k{json.loads(l)['k']}/{json.loads(l)['kernel'][-1]}:{json.loads(l)['us']:.0f}\" for l in sys.stdin))"; done
cd ..
timeout 1200 python bench.py > gpurun_out/r2al/bench.log 2>&1; echo "bench rc=$?"; tail -c 300 gpurun_out/r2al/bench.log
timeout 900 python bench.py --config 2 --no-cpu-baseline > gpurun_out/r2al/bench_cfg2.log 2>&1; echo "cfg2 rc=$?"
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2al/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2al/pytest_gpu.log
