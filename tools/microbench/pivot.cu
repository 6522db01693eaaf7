// Latency of the factor kernel's one-warp pivot (pivot.cuh) in isolation, and its result
// against a host Cholesky inverse.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -maxrregcount=128 -I../../paper_1508_02977_b200/csrc -o pivot pivot.cu
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>
#include "pivot.cuh"

// BUSY: warps 2..15 run independent DFMA chains (the factor's trailing-tile load on the FP64
// pipe) until the pivot warps finish, to show what contention does to the pivot chain
template <int NB, int PAIR, int BUSY = 0>
__global__ void k(const double* D, int kd, double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double LR[NB * (NB + 1)];
  __shared__ __align__(16) double Li[NB * ffb::li_stride<NB>()];
  __shared__ double ir[NB];
  __shared__ int progress;
  __shared__ volatile int done;
  int bad = 1 << 30;
  if (threadIdx.x == 0) progress = 0, done = 0;
  __syncthreads();
  if (BUSY && threadIdx.x >= 64) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-12 * (threadIdx.x + i);
    while (!done) {
      if (BUSY == 1) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
          for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999999999, 1e-9);
      } else {  // DMMA m8n8k4 chains (4 accumulators)
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
          for (int i = 0; i < 8; i += 2)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(a[i]), "+d"(a[i + 1]) : "d"(1e-9), "d"(0.5));
      }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.0) out[0] = s;
    return;
  }
  if (threadIdx.x < (PAIR ? 64 : 32)) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (PAIR)
        ffb::pivot_pair<NB>(D, kd, 0, NB, LR, Li, ir, bad, 0, &progress, r + 1, nullptr);
      else
        ffb::pivot_warp<NB>(D, kd, 0, NB, LR, Li, ir, bad, 0, nullptr);
      asm volatile("bar.sync 1, %0;" ::"r"(PAIR ? 64 : 32));
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps, done = 1;
    for (int i = threadIdx.x; i < NB * NB; i += 32) out[i] = Li[(i / NB) * ffb::li_stride<NB>() + i % NB];
  }
}

template <int NB, int PAIR, int BUSY = 0>
void run(const double* D, int kd, const double* h) {
  double* out;
  long long* cyc;
  cudaMallocManaged(&out, NB * NB * 8);
  cudaMallocManaged(&cyc, 8);
  k<NB, PAIR, BUSY><<<1, 512>>>(D, kd, out, cyc, 20);
  cudaDeviceSynchronize();
  // host: L = chol(A), check Li L = I
  double L[32][32] = {};
  for (int j = 0; j < NB; ++j) {
    double s = h[j * kd + j];
    for (int q = 0; q < j; ++q) s -= L[j][q] * L[j][q];
    L[j][j] = std::sqrt(s);
    for (int i = j + 1; i < NB; ++i) {
      double t = h[i * kd + j];
      for (int q = 0; q < j; ++q) t -= L[i][q] * L[j][q];
      L[i][j] = t / L[j][j];
    }
  }
  double err = 0;
  for (int i = 0; i < NB; ++i)
    for (int j = 0; j < NB; ++j) {
      double s = 0;
      for (int q = 0; q < NB; ++q) s += out[i * NB + q] * L[q][j];
      err = std::fmax(err, std::fabs(s - (i == j)));
    }
  printf("NB%d %s%s %lld cyc, |Li L - I| = %.2e (%s)\n", NB, PAIR ? "pivot_pair" : "pivot_warp", BUSY == 1 ? " +14 DFMA warps" : (BUSY == 2 ? " +14 DMMA warps" : ""), *cyc, err,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int kd = 64;
  static double h[kd * kd];
  for (int i = 0; i < kd; ++i)
    for (int j = 0; j < kd; ++j) h[i * kd + j] = (i == j) ? 40.0 : 1.0 / (1 + i + j);
  double* D;
  cudaMalloc(&D, sizeof(h));
  cudaMemcpy(D, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int it = 0; it < 2; ++it) {
    run<32, 0>(D, kd, h);
    run<32, 1>(D, kd, h);
    run<16, 0>(D, kd, h);
    run<16, 1>(D, kd, h);
    run<32, 1, 1>(D, kd, h);
    run<32, 1, 2>(D, kd, h);
    run<32, 0, 1>(D, kd, h);
    run<32, 0, 2>(D, kd, h);
  }
}
