cd tools
echo "== old"; PG_LIB_PATH=../variants_tmp/old/libpgmres.so python vec_bench.py
echo "== new"; python vec_bench.py
cd ..
timeout 900 python -m pytest tests/test_gpu_cgs2_tma.py tests/test_gpu_parity.py -x -q > /tmp/pt.log 2>&1; echo "tests rc=$?"; tail -15 /tmp/pt.log | cut -c1-300
