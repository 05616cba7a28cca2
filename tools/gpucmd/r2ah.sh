cd tools
for env in "PG_CGS2_UPD=0" "PG_CGS2_UPD=1" "PG_UPD_ROWS=128" "PG_UPD_CTAS=1" "PG_UPD_CTAS=3" "PG_UPD_ROWS=128 PG_UPD_CTAS=1"; do echo "== $env"; env $env timeout 300 python cgs2_bench.py --n 8000000,1000000 --k 12,19,30,45 2>&1 | grep -E "phase2" | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['n']//1000000}M/k{json.loads(l)['k']}:{json.loads(l)['us']}\" for l in sys.stdin))"; done
cd ..
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "icgs or cfg1 or small" > /tmp/pt.log 2>&1; echo "parity rc=$?"; tail -3 /tmp/pt.log
