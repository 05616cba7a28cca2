// FP64 pipe microbenchmark (B200): dependent-issue latency and per-scheduler
// throughput of separately rounded DADD / DMUL chains, as the plane-ring
// kernel issues them.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_pipe fp64_pipe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C, bool MUL>
__global__ void chains(double* out, int iters, long long* cyc) {
  double a[C];
#pragma unroll
  for (int c = 0; c < C; ++c) a[c] = 1.0 + threadIdx.x * 1e-9 + c;
  const double k = 1.0000001;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < C; ++c) a[c] = MUL ? __dmul_rn(a[c], k) : __dadd_rn(a[c], k);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int C, bool MUL>
void run(int warps, double* out, long long* cyc) {
  const int iters = 2000;
  chains<C, MUL><<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  chains<C, MUL><<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_dep = (double)h / (iters * 8.0);          // cycles per dependent step
  const double per_inst_smsp = (double)h / (iters * 8.0 * C * ((warps + 3) / 4));  // per warp-inst on the busiest scheduler
  printf("%s warps/SM=%2d chains/thread=%d  cycles per dependent op %.1f  cycles per warp-inst per scheduler %.2f\n",
         MUL ? "DMUL" : "DADD", warps, C, per_dep, per_inst_smsp);
}

// FP64 chains interleaved with independent integer work (R integer ops per
// FP64 op): do the non-FP64 instructions hide under the FP64 pipe's 2-cycle
// occupancy, or does an FP64 instruction hold the dispatch port for 2 cycles?
template <int C, int R>
__global__ void mixed(double* out, int iters, long long* cyc) {
  double a[C];
  unsigned x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) { a[c] = 1.0 + threadIdx.x * 1e-9 + c; x[c] = threadIdx.x + c; }
  const double k = 1.0000001;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        a[c] = __dadd_rn(a[c], k);
#pragma unroll
        for (int r = 0; r < R; ++r) x[c] = x[c] * 1664525u + 1013904223u + r;
      }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += a[c] + x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int C, int R>
void runm(int warps, double* out, long long* cyc) {
  const int iters = 2000;
  mixed<C, R><<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  mixed<C, R><<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("mixed warps/SM=%2d chains=%d int-ops per DADD=%d  cycles per (DADD + ints) per scheduler %.2f\n",
         warps, C, R, (double)h / (iters * 8.0 * C * ((warps + 3) / 4)));
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 8);
  for (int w : {1, 4, 8, 16, 20, 32}) {
    run<1, false>(w, out, cyc);
    run<2, false>(w, out, cyc);
    run<6, false>(w, out, cyc);
    run<12, false>(w, out, cyc);
  }
  run<1, true>(1, out, cyc);
  run<6, true>(20, out, cyc);
  for (int w : {4, 20}) {
    runm<6, 0>(w, out, cyc);
    runm<6, 1>(w, out, cyc);
    runm<6, 2>(w, out, cyc);
    runm<6, 3>(w, out, cyc);
  }
  return 0;
}
