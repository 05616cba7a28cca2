timeout 900 python -m pytest tests/test_gpu_blasorder.py -q -m gpu -x -k "history" 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
