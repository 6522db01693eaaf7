// DMMA (mma.sync m8n8k4 f64) throughput on B200: W warps per CTA, each a 32x32 tile as 4x4
// accumulator blocks (the factor's rupd_tile_mma pattern without memory), K = 32 per rep.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__global__ void k(double* out, long long* cyc, int reps) {
  const int lane = threadIdx.x & 31;
  double acc[4][4][2];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double a[4], b[4];
  for (int i = 0; i < 4; ++i) a[i] = 1.0 + 1e-9 * (lane + i), b[i] = 1.0 - 1e-9 * (lane + i);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
  }
  long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0) cyc[threadIdx.x >> 5] = (t1 - t0) / reps;
  double s = 0; for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 32 * 8);
  for (int w : {1, 2, 4, 8, 16}) {
    k<<<148, 32 * w>>>(out, cyc, 200);
    long long c[32]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double fma = 128.0 * 256 * w;  // per CTA per rep
    printf("warps %2d: %lld cycles per 32x32x32 tile per warp -> %.1f FMA/clk/SM\n", w, c[0], fma / c[0]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
