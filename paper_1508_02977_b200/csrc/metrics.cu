// Flow-error metrics against a .flo ground truth as a device reduction:
// compute_metrics (src/metrics.cpp:75-100). Per pixel with valid truth (|u|, |v| <= 1e9,
// metrics.cpp:17-19): angular error acos of the clamped (u, v, 1) cosine and the endpoint
// error, in the reference's operation order (--fmad=false); the sums are reduced in a fixed
// tree order (deterministic; equal to the reference's serial sums to rounding).
#include "ffb_internal.cuh"

#include <cmath>

namespace ffb {

namespace {

constexpr int kMT = 256;

__global__ void __launch_bounds__(kMT)
    k_metrics(const double* __restrict__ u1, const double* __restrict__ u2,
              const float* __restrict__ tu, const float* __restrict__ tv, long long n,
              double* __restrict__ part, unsigned* __restrict__ counter,
              double* __restrict__ out) {
  double sa = 0.0, se = 0.0, cnt = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * kMT + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * kMT) {
    const float ue = tu[i], ve = tv[i];
    if (!(fabs(static_cast<double>(ue)) <= 1e9 && fabs(static_cast<double>(ve)) <= 1e9)) continue;
    const double u = u1[i], v = u2[i];
    const double num = u * ue + v * ve + 1.0;
    const double den = sqrt((u * u + v * v + 1.0) *
                            (static_cast<double>(ue) * ue + static_cast<double>(ve) * ve + 1.0));
    double c = num / den;
    c = fmin(1.0, fmax(-1.0, c));
    sa += acos(c);
    const double du = u - ue, dv = v - ve;
    se += sqrt(du * du + dv * dv);
    cnt += 1.0;
  }
  __shared__ double sm[3][kMT / 32];
  for (int off = 16; off; off >>= 1) {
    sa += __shfl_xor_sync(~0u, sa, off);
    se += __shfl_xor_sync(~0u, se, off);
    cnt += __shfl_xor_sync(~0u, cnt, off);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sm[0][warp] = sa, sm[1][warp] = se, sm[2][warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, e = 0.0, k = 0.0;
    for (int w = 0; w < kMT / 32; ++w) a += sm[0][w], e += sm[1][w], k += sm[2][w];
    part[3 * blockIdx.x] = a, part[3 * blockIdx.x + 1] = e, part[3 * blockIdx.x + 2] = k;
    __threadfence();
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      double A = 0.0, E = 0.0, K = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) {
        A += __ldcg(part + 3 * b);
        E += __ldcg(part + 3 * b + 1);
        K += __ldcg(part + 3 * b + 2);
      }
      out[0] = A, out[1] = E, out[2] = K;
      *counter = 0;
    }
  }
}

}  // namespace

// out[0..2] = (sum of angular errors [rad], sum of endpoint errors, valid pixels)
void flow_metrics(const double* u1, const double* u2, const float* tu, const float* tv,
                  long long n, double* part, unsigned* counter, double* out, cudaStream_t st) {
  k_metrics<<<kRedBlocks, kMT, 0, st>>>(u1, u2, tu, tv, n, part, counter, out);
  FFB_LAUNCHED();
}

}  // namespace ffb
