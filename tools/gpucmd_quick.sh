for cfgs in "off 500" "smi 500" "smi 250"; do
set -- $cfgs
PG_BENCH_CLOCKS=$1 PG_BENCH_CLOCKS_MS=$2 python bench.py --no-cpu-baseline --steps 40 > gpurun_out/bench_x.log 2>&1
echo "== $cfgs"; grep -o '"value": [0-9.]*, "unit": "s", "n_gpus\|"median": [0-9.]*\|"max": [0-9.]*\|"samples": [0-9]*' gpurun_out/bench_x.log | tr '\n' ' '; echo
done
