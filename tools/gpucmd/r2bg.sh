for t in 0 1; do echo "== PG_CGS2_TMA3=$t"; PG_CGS2_TMA3=$t timeout 600 python tools/cgs2_bench.py --n 8000000,1000000 --k 13,19,25,33,40,45 2>&1 | grep phase3 | cut -c1-120; done
echo "== one CTA per SM"; PG_TILE_CTAS_P3=1 timeout 600 python tools/cgs2_bench.py --n 8000000 --k 13,19,25 2>&1 | grep phase3 | cut -c1-120
timeout 900 python -m pytest tests/test_gpu_cgs2_tma.py -q -m gpu -x 2>&1 | tail -3
