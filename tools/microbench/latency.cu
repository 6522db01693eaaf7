// Latency probes on B200: __syncthreads at 512 threads, dependent DFMA chain, FP64 rsqrt
// variants, shared-memory load-to-use, L2 load-to-use.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, const double* g, long long* cyc) {
  __shared__ double sm[1024];
  const int tid = threadIdx.x;
  sm[tid] = tid * 1.0; __syncthreads();
  long long t0, t1; double x = 1.0 + tid * 1e-9, y = 1.000001;
  // 1. syncthreads
  t0 = clock64(); for (int i = 0; i < 1000; ++i) __syncthreads(); t1 = clock64();
  if (tid == 0) cyc[0] = (t1 - t0) / 1000;
  // 2. dependent DFMA
  t0 = clock64(); for (int i = 0; i < 1000; ++i) x = fma(x, y, 1e-12); t1 = clock64();
  if (tid == 0) cyc[1] = (t1 - t0) / 1000;
  // 3. rsqrt double library
  t0 = clock64(); for (int i = 0; i < 100; ++i) x = rsqrt(x) + 1.0; t1 = clock64();
  if (tid == 0) cyc[2] = (t1 - t0) / 100;
  // 4. sqrt double
  t0 = clock64(); for (int i = 0; i < 100; ++i) x = sqrt(x) + 1.0; t1 = clock64();
  if (tid == 0) cyc[3] = (t1 - t0) / 100;
  // 5. double division
  t0 = clock64(); for (int i = 0; i < 100; ++i) x = 1.0 / x + 1.0; t1 = clock64();
  if (tid == 0) cyc[4] = (t1 - t0) / 100;
  // 6. smem dependent load chain
  int idx = tid & 1023;
  t0 = clock64(); for (int i = 0; i < 1000; ++i) idx = (int)sm[idx] & 1023; t1 = clock64();
  if (tid == 0) cyc[5] = (t1 - t0) / 1000;
  // 7. global (L2-resident) dependent chain
  long long gi = tid;
  t0 = clock64(); for (int i = 0; i < 100; ++i) gi = (long long)g[gi] ; t1 = clock64();
  if (tid == 0) cyc[6] = (t1 - t0) / 100;
  // 8. rsqrtf seed + 2 Newton
  t0 = clock64(); for (int i = 0; i < 100; ++i) { double r = (double)rsqrtf((float)x); const double h=0.5*x; r = r*fma(-h*r,r,1.5); r = r*fma(-h*r,r,1.5); x = r + 1.0; } t1 = clock64();
  if (tid == 0) cyc[7] = (t1 - t0) / 100;
  // 9. shfl double chain
  t0 = clock64(); for (int i = 0; i < 1000; ++i) x = __shfl_sync(0xffffffff, x, (tid + 1) & 31) + 1e-9; t1 = clock64();
  if (tid == 0) cyc[8] = (t1 - t0) / 1000;
  out[tid] = x + gi + idx;
}
int main() {
  double *out, *g; long long* cyc; cudaMalloc(&out, 8192); cudaMalloc(&g, 1 << 20); cudaMalloc(&cyc, 128);
  double h[1 << 17]; for (int i = 0; i < (1 << 17); ++i) h[i] = (i * 7919 + 13) % (1 << 17); cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int th : {32, 256, 512, 1024}) {
    k<<<1, th>>>(out, g, cyc); long long c[9]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("threads %4d: sync %lld  dfma %lld  rsqrt %lld  sqrt %lld  div %lld  lds %lld  ldg(L2) %lld  fast_rsqrt %lld  shfl %lld cycles\n", th, c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7], c[8]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
