// Pivot block of the factor kernel's blocked symmetric sweep (band.cu, K5): the Cholesky
// factor L of the nbk x nbk diagonal block A_KK and its inverse Li = L^-1, by one warp.
//
// Lane j owns column j in registers. The columns rotate down one row per elimination step
// (c[t] holds row k + t at step k), so every register index is static while the k loop stays
// rolled — a few hundred instructions, which matters because the pivot runs beside the other
// warps' work once per sweep step and must not evict their code. Column k of L is broadcast
// through shared memory, stored rotated (LR[k][t] = L[k + t][k]) so that every lane reads it
// with aligned 16-byte broadcast loads; shuffles would cost two SHFL per double on the
// (shared) MIO pipe. The forward substitution for Li reuses the same rows.
#pragma once

#include <type_traits>

namespace ffb {

// row stride of the L^-1 tiles: even (rows stay 16-byte aligned for paired loads) and
// = 4 mod 16 doubles, so the DMMA fragment loads — lanes (g, t4) reading Li[(g + ..) LDL + t4 + ..]
// as 64-bit loads served per half-warp — put the half-warp's 4 rows on disjoint 32-byte bank
// groups (NB + 2 had rows 16 bytes apart: ncu counted 6.3e9 excessive shared wavefronts per
// c4 factorisation, all on these loads)
template <int NB>
__host__ __device__ constexpr int li_stride() {
  return NB + 4;
}

// a usable pivot: positive and finite (false for NaN)
__device__ __forceinline__ bool pivot_ok(double d) { return d > 0.0 && d <= 1.7976931348623157e308; }

// 1/sqrt(x) for a positive normal x without branches: the hardware approximation refined by
// two Newton steps y <- y + y (1/2 - x/2 y^2), each doubling the correct bits
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  e = fma(-h * y, y, 0.5);
  return fma(y, e, y);
}

// src: the block's lower triangle with leading dimension ld (global D or a shared tile,
// which may alias LR); k0: its first row, for the breakdown index.
template <int NB>
__device__ __noinline__ void pivot_warp(const double* src, long long ld, int k0, int nbk,
                                        double* LR, double* Li, double* ir, int& first_bad,
                                        int bad_base, double* LiT) {
  static_assert(NB % 2 == 0 && NB <= 32, "pivot block");
  const int lane = threadIdx.x & 31;
  double c[NB];
#pragma unroll
  for (int t = 0; t < NB; ++t) {
    const int a = max(t, lane), b = min(t, lane);
    c[t] = (lane < nbk && t < nbk) ? src[a * ld + b] : (t == lane ? 1.0 : 0.0);
  }
  __syncwarp();
  int fb = first_bad;
#pragma unroll 1
  for (int k = 0; k < NB; ++k) {
    double dkk = __shfl_sync(~0u, c[0], k);
    const bool bad = !pivot_ok(dkk);
    fb = (bad && k < nbk) ? min(fb, bad_base + k0 + k) : fb;
    dkk = bad ? 1.0 : dkk;
    const double r = rsqrt_nr(dkk);
    const double l = (lane == k) ? dkk * r : c[0] * r;  // L[lane][k] for lane >= k
    double* row = LR + k * NB;                           // row[t] = L[k + t][k]
    if (lane >= k && lane < NB) row[lane - k] = l;
    if (lane == k) ir[k] = r;
    __syncwarp();
    // trailing update of column `lane`, rotated: c[t-1] = c[t] - L[k+t][k] L[lane][k]
    // (rows k + t >= NB read stale entries of `row`: they only ever feed rows >= NB)
    c[0] = c[1] - row[1] * l;
#pragma unroll
    for (int t = 2; t < NB; t += 2) {
      const double2 v = *reinterpret_cast<const double2*>(row + t);
      c[t - 1] = c[t] - v.x * l;
      c[t] = c[t + 1] - v.y * l;
    }
    c[NB - 1] = 0.0;
  }
  first_bad = fb;
  // column `lane` of L^-1: y_k = cur_k / L[k][k], cur_i -= L[i][k] y_k (i > k), rotated
#pragma unroll
  for (int t = 0; t < NB; ++t) c[t] = (t == lane) ? 1.0 : 0.0;
#pragma unroll 1
  for (int k = 0; k < NB; ++k) {
    const double y = c[0] * ir[k];
    if (lane < NB) {
      Li[k * li_stride<NB>() + lane] = y;
      if (LiT) LiT[lane * li_stride<NB>() + k] = y;
    }
    const double* row = LR + k * NB;
    c[0] = c[1] - row[1] * y;
#pragma unroll
    for (int t = 2; t < NB; t += 2) {
      const double2 v = *reinterpret_cast<const double2*>(row + t);
      c[t - 1] = c[t] - v.x * y;
      c[t] = c[t + 1] - v.y * y;
    }
    c[NB - 1] = 0.0;
  }
  __syncwarp();
}

// The same factorisation by two warps of the CTA (called by both; role = warp & 1): the
// Cholesky warp publishes each finished column of L through `progress` (a shared counter,
// value tag * 64 + k + 1 once column k is in LR, unique per call so it never needs a reset)
// and the substitution warp builds L^-1 one step behind it, so the two serial chains
// overlap instead of running back to back.
__device__ __forceinline__ int ld_acquire_shared(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];"
               : "=r"(v)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p)))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_shared(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(p))),
               "r"(v)
               : "memory");
}

// The elimination steps in kPivStages stages of NB / kPivStages steps: step k touches the
// rotated entries t < NB - k only, so stage s runs with width NB - s NB / kPivStages (FP64
// instructions are what the pivot warps compete for with the tile warps' DMMA).
#ifndef FFB_PIVS
#define FFB_PIVS 8
#endif
constexpr int kPivStages = FFB_PIVS;
template <int NB, int S = 0, class F>
__device__ __forceinline__ void pivot_stages(F& step) {
  constexpr int n = NB / kPivStages, W = NB - S * n;
  static_assert(NB % kPivStages == 0 && W % 2 == 0, "pivot stage widths");
#pragma unroll 1
  for (int k = S * n; k < (S + 1) * n; ++k) step(k, std::integral_constant<int, W>());
  if constexpr (S + 1 < kPivStages) pivot_stages<NB, S + 1>(step);
}

template <int NB>
__device__ __noinline__ void pivot_pair(const double* src, long long ld, int k0, int nbk,
                                        double* LR, double* Li, double* ir, int& first_bad,
                                        int bad_base, int* progress, int tag, double* LiT) {
  static_assert(NB % 2 == 0 && NB <= 32, "pivot block");
  const int lane = threadIdx.x & 31;
  double c[NB];
  if ((threadIdx.x >> 5) % 2 == 0) {  // Cholesky
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const int a = max(t, lane), b = min(t, lane);
      c[t] = (lane < nbk && t < nbk) ? src[a * ld + b] : (t == lane ? 1.0 : 0.0);
    }
    __syncwarp();
    int fb = first_bad;
    // software-pipelined: the next pivot (lane k+1's updated diagonal, c[1] - l^2 with its
    // own l) and its rsqrt are formed before this step's column update is issued
    double dkk = __shfl_sync(~0u, c[0], 0);
    if (!(dkk > 0.0) || !isfinite(dkk)) {
      if (0 < nbk) fb = min(fb, bad_base + k0);
      dkk = 1.0;
    }
    double r = rsqrt(dkk);
    // step k touches rotated entries t < NB - k only (rows k + t < NB): see pivot_stages
    auto step = [&](int k, auto width) {
      constexpr int WD = decltype(width)::value;
      const double l = (lane == k) ? dkk * r : c[0] * r;
      const double dn0 = __shfl_sync(~0u, c[1] - l * l, (k + 1) & 31);
      double* row = LR + k * NB;
      if (lane >= k && lane < NB) row[lane - k] = l;
      if (lane == k) ir[k] = r;
      __syncwarp();
      if (lane == 0) st_release_shared(progress, tag * 64 + k + 1);
      // branch-free pivot check and rsqrt: the step stays one basic block, so the scheduler
      // interleaves the Newton steps with the column update below instead of the warp
      // stalling on each of them in turn (the library rsqrt branches to a slow path)
      const bool bad = k + 1 < NB && !pivot_ok(dn0);
      fb = (bad && k + 1 < nbk) ? min(fb, bad_base + k0 + k + 1) : fb;
      const double dn = bad ? 1.0 : dn0;
      const double rn = rsqrt_nr(dn);
      c[0] = c[1] - row[1] * l;
#pragma unroll
      for (int t = 2; t < WD; t += 2) {
        const double2 v = *reinterpret_cast<const double2*>(row + t);
        c[t - 1] = c[t] - v.x * l;
        c[t] = c[t + 1] - v.y * l;
      }
      c[WD - 1] = 0.0;
      dkk = dn;
      r = rn;
    };
    pivot_stages<NB>(step);
    first_bad = fb;
  } else {  // forward substitution for L^-1, one column of L behind
#pragma unroll
    for (int t = 0; t < NB; ++t) c[t] = (t == lane) ? 1.0 : 0.0;
    auto step = [&](int k, auto width) {
      constexpr int WD = decltype(width)::value;
      while (ld_acquire_shared(progress) < tag * 64 + k + 1) {
      }
      __syncwarp();
      const double y = c[0] * ir[k];
      if (lane < NB) {
        Li[k * li_stride<NB>() + lane] = y;
        if (LiT) LiT[lane * li_stride<NB>() + k] = y;
      }
      const double* row = LR + k * NB;
      c[0] = c[1] - row[1] * y;
#pragma unroll
      for (int t = 2; t < WD; t += 2) {
        const double2 v = *reinterpret_cast<const double2*>(row + t);
        c[t - 1] = c[t] - v.x * y;
        c[t] = c[t + 1] - v.y * y;
      }
      c[WD - 1] = 0.0;
    };
    pivot_stages<NB>(step);
  }
  __syncwarp();
}

}  // namespace ffb
