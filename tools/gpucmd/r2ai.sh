cd tools
for env in "PG_CGS2_TMA=0" "PG_CGS2_TMA=1"; do echo "== $env"; env $env timeout 300 python cgs2_bench.py --n 8000000,1000000 --k 12,19,25,30,45 2>&1 | grep -E "phase1|phase2" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(f\"{d['n']//1000000}M k{d['k']} {d['kernel']}: {d['us']} us {d['gbs']} GB/s\")"; done
cd ..
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > /tmp/pt.log 2>&1; echo "parity rc=$?"; tail -3 /tmp/pt.log
