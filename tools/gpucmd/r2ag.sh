cd tools; timeout 300 python cgs2_bench.py --n 8000000,1000000 --k 12,19,30,45 2>&1 | grep -E "phase2"
