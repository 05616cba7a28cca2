# r01i final: GPU tests + smoke + cfg4 / cfg2 bench lines + ncu of the 1024-row windowed pass
set -x
mkdir -p gpurun_out/r1i
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1i/smoke_fin.log 2>&1; tail -1 gpurun_out/r1i/smoke_fin.log
timeout 900 python -m pytest tests -q -m "gpu" > gpurun_out/r1i/pytest_gpu_fin.log 2>&1; tail -2 gpurun_out/r1i/pytest_gpu_fin.log
python tools/spmv_bench.py --variants default --cases cfg4 2>&1 | tail -1
python bench.py > gpurun_out/r1i/bench_cfg2_fin.log 2>&1; tail -c 200 gpurun_out/r1i/bench_cfg2_fin.log
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1i/bench_cfg4_fin.log 2>&1; tail -c 200 gpurun_out/r1i/bench_cfg4_fin.log
python bench.py --config 4 --construction arnoldi --poly-form roots --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1i/bench_cfg4_arnoldi_fin.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sell_win_kernel" -s 2 -c 1 -o gpurun_out/r1i/prof_win_cfg4_fin python tools/spmv_one.py --config 4 --grid 200 > gpurun_out/r1i/ncu_fin.log 2>&1; tail -1 gpurun_out/r1i/ncu_fin.log
