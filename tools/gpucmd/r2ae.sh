mkdir -p gpurun_out/r2ae
cd tools; timeout 300 python cgs2_bench.py --n 8000000,1000000 --k 8,12,19,30,45 2>&1 | grep -E "phase" > ../gpurun_out/r2ae/cgs2.log; cat ../gpurun_out/r2ae/cgs2.log; cd ..
timeout 1200 python bench.py > gpurun_out/r2ae/bench.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/r2ae/bench.log
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2ae/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2ae/pytest_gpu.log
