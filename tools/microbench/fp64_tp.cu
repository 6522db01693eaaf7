// FP64 throughput / shuffle latency probe on B200: W warps per CTA each issue the solve tile's
// FMA pattern (8 row chains x 4 + 4 column chains x 8 = 64 DFMA per lane) and the 10-step
// double transpose-reduction; cycles per repetition, one CTA per SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int reps, int mode) {
  const int lane = threadIdx.x & 31;
  double a[8][4], wc[4], racc[8], cacc[4];
  for (int i = 0; i < 8; ++i) for (int c = 0; c < 4; ++c) a[i][c] = 1.0 + 1e-9 * (i * 4 + c + lane);
  for (int c = 0; c < 4; ++c) wc[c] = 1.0 - 1e-9 * c;
  double acc = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (mode & 1) {
      for (int c = 0; c < 4; ++c) cacc[c] = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const double wr = wc[kk & 3] + acc * 1e-30;
        racc[kk] = a[kk][0] * wc[0];
#pragma unroll
        for (int c = 1; c < 4; ++c) racc[kk] = fma(a[kk][c], wc[c], racc[kk]);
#pragma unroll
        for (int c = 0; c < 4; ++c) cacc[c] = fma(a[kk][c], wr, cacc[c]);
      }
    } else {
      for (int kk = 0; kk < 8; ++kk) racc[kk] = acc + kk;
      for (int c = 0; c < 4; ++c) cacc[c] = acc - c;
    }
    if (mode & 2) {
      const bool b2 = lane & 4, b1 = lane & 2, b0 = lane & 1, b4 = lane & 16, b3 = lane & 8;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) { const double s = b2 ? racc[kk] : racc[kk + 4]; racc[kk] = (b2 ? racc[kk + 4] : racc[kk]) + __shfl_xor_sync(~0u, s, 4); }
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) { const double s = b1 ? racc[kk] : racc[kk + 2]; racc[kk] = (b1 ? racc[kk + 2] : racc[kk]) + __shfl_xor_sync(~0u, s, 2); }
      { const double s = b0 ? racc[0] : racc[1]; racc[0] = (b0 ? racc[1] : racc[0]) + __shfl_xor_sync(~0u, s, 1); }
#pragma unroll
      for (int c = 0; c < 2; ++c) { const double s = b4 ? cacc[c] : cacc[c + 2]; cacc[c] = (b4 ? cacc[c + 2] : cacc[c]) + __shfl_xor_sync(~0u, s, 16); }
      { const double s = b3 ? cacc[0] : cacc[1]; cacc[0] = (b3 ? cacc[1] : cacc[0]) + __shfl_xor_sync(~0u, s, 8); }
    }
    acc += racc[0] + cacc[0];
  }
  long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0) cyc[threadIdx.x >> 5] = (t1 - t0) / reps;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 32 * 8);
  for (int mode : {1, 2, 3})
    for (int w : {1, 4, 14, 16}) {
      k<<<148, 32 * w>>>(out, cyc, 1000, mode);
      long long c[32]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      printf("mode %d (1 fma, 2 shfl, 3 both) warps %2d: %lld cycles/rep (warp 0)\n", mode, w, c[0]);
    }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
