# r02a: sanitizer sweep over the small GPU tests + current cfg4 bench baseline
mkdir -p gpurun_out/r2a
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 900 $S --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py tests/test_gpu_ilu.py tests/test_gpu_roots.py \
    -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/r2a/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r2a/san_$tool.log
done
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2a/bench_cfg4.log 2>&1; tail -c 600 gpurun_out/r2a/bench_cfg4.log
