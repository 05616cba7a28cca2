mkdir -p gpurun_out/cgsweep
for c in 1 2 3 4; do PG_TILE_CTAS_P1=$c PG_TILE_CTAS_P2=$c python tools/cgs2_bench.py --n 1000000,8000000 --k 16,20,25,30,35,40,45,51 --reps 10 > gpurun_out/cgsweep/c$c.jsonl 2>&1; done
grep -h phase1 gpurun_out/cgsweep/c*.jsonl | head -3
