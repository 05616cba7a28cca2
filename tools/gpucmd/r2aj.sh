cd tools
PG_TMA_DEBUG=1 timeout 300 python cgs2_bench.py --n 1000000 --k 12 --reps 1 2>&1 | head -5
