cd tools
for env in "PG_CGS2_TMA=1" "PG_TILE_CTAS_P1=1 PG_TILE_CTAS_P2=1" "PG_TILE_CTAS_P1=2 PG_TILE_CTAS_P2=2" "PG_TILE_CTAS_P1=3 PG_TILE_CTAS_P2=3" "PG_TILE_CTAS_P1=4 PG_TILE_CTAS_P2=4" "PG_TILE_ROWS=128" "PG_TILE_ROWS=256"; do echo "== $env"; env $env timeout 300 python cgs2_bench.py --n 8000000,1000000 --k 12,19,25,30,45 2>&1 | grep -E "phase1|phase2" | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['n']//1000000}M/k{json.loads(l)['k']}/{json.loads(l)['kernel'][-1]}:{json.loads(l)['us']:.0f}\" for l in sys.stdin))"; done
