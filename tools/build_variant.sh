#!/bin/bash
# Build an A/B variant of libpgmres.so with extra nvcc defines into variants_tmp/.
#   tools/build_variant.sh NAME -DPG_WIN_STAGES=2 ...
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/variants_tmp/$name
mkdir -p "$out"
nccl=$(python -c "from paper_1907_00072_b200._build import _nccl_include; print(_nccl_include())")
flags="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden,-ffp-contract=off -I $root/include -I $nccl"
for f in $(python -c "from paper_1907_00072_b200._build import SOURCES; print(' '.join(x[:-3] for x in SOURCES))"); do
  nvcc $flags "$@" -c "$root/paper_1907_00072_b200/csrc/$f.cu" -o "$out/$f.o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libpgmres.so" "$out"/*.o -ldl
rm -f "$out"/*.o
echo "$out/libpgmres.so"
