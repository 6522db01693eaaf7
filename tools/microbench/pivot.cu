// Latency of the factor kernel's one-warp pivot (pivot.cuh) in isolation, and its result
// against a host Cholesky inverse.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1508_02977_b200/csrc -o pivot pivot.cu
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>
#include "pivot.cuh"

template <int NB, int PAIR>
__global__ void k(const double* D, int kd, double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double LR[NB * (NB + 1)];
  __shared__ __align__(16) double Li[NB * (NB + 2)];
  __shared__ double ir[NB];
  __shared__ int progress;
  int bad = 1 << 30;
  if (threadIdx.x == 0) progress = 0;
  __syncthreads();
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
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
    for (int i = threadIdx.x; i < NB * NB; i += 32) out[i] = Li[(i / NB) * (NB + 2) + i % NB];
  }
}

template <int NB, int PAIR>
void run(const double* D, int kd, const double* h) {
  double* out;
  long long* cyc;
  cudaMallocManaged(&out, NB * NB * 8);
  cudaMallocManaged(&cyc, 8);
  k<NB, PAIR><<<1, 512>>>(D, kd, out, cyc, 20);
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
  printf("NB%d %s %lld cyc, |Li L - I| = %.2e (%s)\n", NB, PAIR ? "pivot_pair" : "pivot_warp", *cyc, err,
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
  }
}
