mkdir -p gpurun_out/r2af
cd tools
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tile_kernel<\(int\)2" -s 2 -c 1 -o ../gpurun_out/r2af/prof_p2_k45 python cgs2_bench.py --n 8000000 --k 45 --reps 3 > ../gpurun_out/r2af/ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tile_kernel<\(int\)1" -s 2 -c 1 -o ../gpurun_out/r2af/prof_p1_k45 python cgs2_bench.py --n 8000000 --k 45 --reps 3 > ../gpurun_out/r2af/ncu1.log 2>&1; echo "ncu rc=$?"
