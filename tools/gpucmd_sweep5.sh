mkdir -p gpurun_out/sweep5
timeout 1200 python tools/degree_sweep.py --out gpurun_out/sweep5/cfg5_degree_sweep.json > gpurun_out/sweep5/policy.log 2>&1; tail -2 gpurun_out/sweep5/policy.log
timeout 1200 python tools/degree_sweep.py --construction arnoldi --out gpurun_out/sweep5/cfg5_degree_sweep_arnoldi.json > gpurun_out/sweep5/arnoldi.log 2>&1; tail -2 gpurun_out/sweep5/arnoldi.log
