# the dominant kernel (fused polynomial pass, kPoly) of a cfg2 solve
mkdir -p gpurun_out/r1e
ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"sell_pat_kernel<\(int\)1" -s 40 -c 2 -o gpurun_out/r1e/prof_polyk1_cfg2 python tools/profile_solve.py > gpurun_out/r1e/ncu_full4.log 2>&1; tail -2 gpurun_out/r1e/ncu_full4.log
