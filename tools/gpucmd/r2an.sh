timeout 900 python tools/e2e_probe.py --config 4 --reps 3 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_integration.py tests/test_gpu_distributed.py -x -q > /tmp/pt.log 2>&1; echo "tests rc=$?"; tail -3 /tmp/pt.log
