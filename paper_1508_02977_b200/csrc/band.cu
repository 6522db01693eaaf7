// K5/K6: exact subdomain solves of the additive-Schwarz preconditioner — a block LDL^T
// factorization over grid lines, factor and solve batched over all subdomains.
//
// Replaces the reference's per-part SparseCholesky (src/linsolve.cpp:107-273: RCM,
// elimination tree, up-looking level-scheduled factorization, two triangular sweeps) that
// schwarz_solve drives per subdomain (src/schwarz.cpp:236-248). We use the structure of the
// pixel grid instead of a general sparse symbolic phase: the free rectangle of subdomain i
// is ordered line by line along its long (slow) side, each line holding its S vertices x nc
// components (kd = nc*S unknowns, fast axis = short side). A_i is then block tridiagonal:
// dense-banded diagonal blocks A_ll (nodal 3x3 blocks + fast-axis couplings) and DIAGONAL
// off-diagonal blocks B_l (the slow-axis edge weights, component-wise). Its exact block
// LDL^T factorization is
//     D_0 = A_00,   D_l = A_ll - B_l D_{l-1}^{-1} B_l,          Dinv_l = D_l^{-1},
// and A_i^{-1} r is two sweeps of one dense symmetric GEMV per line:
//     forward   y_l = Dinv_l (r_l - B_l y_{l-1})
//     backward  x_l = y_l - Dinv_l (B_{l+1} x_{l+1}),   x_{L-1} = y_{L-1}.
// Only Dinv_l is stored (packed lower triangle, kd(kd+1)/2 per line): half the storage and
// half the bytes per application of a banded Cholesky factor of the same matrix (which must
// hold the filled-in B_l L^-T blocks), and the only sequential dependency is line to line.
//
// Factor (K5, k_line_factor: a 4- or 8-CTA cluster per (subdomain, chain) of the twisted
// factorisation): per line, build D_l in place in the packed factor storage (L2-resident while
// it is swept) and invert it with a blocked symmetric sweep (Gauss-Jordan for SPD):
//     pivot block K (two warps, in registers, one step ahead): Lc = chol(A_KK), Li = Lc^-1,
//     Z = A_RK Li^T, A_RR -= Z Z^T (32x32 warp tiles on the FP64 tensor cores, DMMA m8n8k4),
//     A_RK <- Z Li, A_KK <- -Li^T Li,
// which leaves -D^{-1}; the flops equal a banded Cholesky's (n kd^2 / 2 FMAs).
// Solve (K6), three kernels by regime, every sum in a fixed order (deterministic):
//   k_line_solve_tile — narrow lines (c1, c2), latency regime: one 32x32 register tile per warp
//     across a cluster, operands and partial sums over distributed shared memory;
//   k_line_solve_rt   — lines up to 448 unknowns (c3, c4), bandwidth regime: the packed rows
//     stream through a shared-memory ring (cp.async.bulk + mbarrier) in whole 16-row groups and
//     are multiplied as 16x32 register tiles; one CTA per chain (persistent task queue when
//     chains > SMs) or a 2-/4-CTA cluster per chain; optional single-precision factor copy;
//   k_line_solve      — wider lines (c5) and 8-CTA clusters: the same ring with row batches,
//     each warp taking whole rows (row dots + per-lane column partials).
#include "ffb_internal.cuh"

#include <mutex>
#include "pivot.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

namespace ffb {

#ifdef FFB_PROFILE
__device__ unsigned long long g_prof[64];
#define PROF_DECL unsigned long long prof_t = clock64(), prof_acc[16] = {0};
#define PROF_MARK(i)                                   \
  do {                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0) {         \
      const unsigned long long t_ = clock64();         \
      prof_acc[i] += t_ - prof_t;                      \
      prof_t = t_;                                     \
    }                                                  \
  } while (0)
#define PROF_FLUSH(base)                                                  \
  do {                                                                    \
    if (blockIdx.x == 0 && threadIdx.x == 0)                              \
      for (int i_ = 0; i_ < 16; ++i_) g_prof[(base) + i_] += prof_acc[i_]; \
  } while (0)
// per-warp event timeline of CTA 0 for forward line steps 8..23 (tile solve kernel)
__device__ unsigned long long g_tl[16][16][8];
#define TL_MARK(i)                                                                   \
  do {                                                                               \
    if (blockIdx.x == 0 && phase == 0 && t >= 8 && t < 24 && (threadIdx.x & 31) == 0) \
      g_tl[t - 8][threadIdx.x >> 5][i] = clock64();                                  \
  } while (0)
// per-warp event timeline of CTA 0 for the sweep steps of line 10 (factor kernel)
__device__ unsigned long long g_ftl[16][16][8];
#define FTL_MARK(i)                                                                    \
  do {                                                                                 \
    if (blockIdx.x == 0 && bad_base == 10 * kd && step < 16 && (threadIdx.x & 31) == 0) \
      g_ftl[step][threadIdx.x >> 5][i] = clock64();                                    \
  } while (0)
#else
#define FTL_MARK(i) \
  do {              \
  } while (0)
#define TL_MARK(i) \
  do {             \
  } while (0)
#define PROF_DECL
#define PROF_MARK(i) \
  do {               \
  } while (0)
#define PROF_FLUSH(base) \
  do {                   \
  } while (0)
#endif

namespace {

// ----------------------------------------------------------------- packed row layout
// Row r of a line's lower triangle holds columns 0..r, padded to an even length so every
// row starts 16-byte aligned: rows 2m and 2m+1 both have length 2m+2.
__host__ __device__ __forceinline__ long long prow_off(int r) {
  const long long m = r >> 1;
  return (r & 1) ? 2 * m * (m + 1) + 2 * m + 2 : 2 * m * (m + 1);
}

// the same offset in 32-bit arithmetic (a line holds < 2^31 entries)
__device__ __forceinline__ int prow_off32(int r) {
  const int m = r >> 1;
  return 2 * m * (m + 1) + (r & 1) * (2 * m + 2);
}

// global interleaved index of local unknown j of line l
__device__ __forceinline__ long long gidx(const SubInfo& s, int l, int j, int W, int nc) {
  const int a = j / nc, c = j - a * nc;
  const int lx = s.xfast ? a : l, ly = s.xfast ? l : a;
  return (static_cast<long long>(s.fy0 + ly) * W + (s.fx0 + lx)) * nc + c;
}

// slow-axis coupling B_l between unknown j of line l and of line l-1 (l >= 1)
__device__ __forceinline__ double bcoef(const SubInfo& s, const double* __restrict__ coef,
                                        size_t N, int W, int nc, int l, int j) {
  const int a = j / nc, c = j - a * nc;
  const int k = c < 2 ? 0 : 1;
  const int lx = s.xfast ? a : l, ly = s.xfast ? l : a;
  const size_t v = static_cast<size_t>(s.fy0 + ly) * W + (s.fx0 + lx);
  return s.xfast ? coef[(8 + k) * N + v - W] : coef[(6 + k) * N + v - 1];
}

// entry (i, j), j <= i, of the intra-line block A_ll
__device__ __forceinline__ double aline(const SubInfo& s, const double* __restrict__ coef,
                                        size_t N, int W, int nc, int l, int i, int j) {
  const int ai = i / nc, ci = i - ai * nc;
  const int aj = j / nc, cj = j - aj * nc;
  const int lx = s.xfast ? ai : l, ly = s.xfast ? l : ai;
  const size_t v = static_cast<size_t>(s.fy0 + ly) * W + (s.fx0 + lx);
  if (ai == aj) {
    // m planes: 0 m11, 1 m12, 2 m13, 3 m22, 4 m23, 5 m33
    const int sum = ci + cj;
    const int plane = ci == cj ? (ci == 0 ? 0 : (ci == 1 ? 3 : 5)) : (sum == 1 ? 1 : (sum == 2 ? 2 : 4));
    return coef[plane * N + v];
  }
  if (aj == ai - 1 && ci == cj) {
    const int k = ci < 2 ? 0 : 1;
    return s.xfast ? coef[(6 + k) * N + v - 1] : coef[(8 + k) * N + v - W];
  }
  return 0.0;
}

// ----------------------------------------------------------------- cluster helpers
// Every subdomain is owned by one thread-block cluster of C CTAs (C = 1, 2, 4 or 8, chosen
// so that ~128 SMs take part); CTAs exchange partial results through distributed shared
// memory and order their global-memory work with cluster barriers.
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// barrier over the whole cluster with release/acquire ordering of shared and global memory
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
// the same barrier in two halves (arrive early, wait late)
__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of `p` (a shared-memory variable of this CTA) in CTA `rank` of the cluster
template <class T>
__device__ __forceinline__ T* cl_map(T* p, unsigned rank) {
  size_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(p), "r"(rank));
  return reinterpret_cast<T*>(out);
}

// rows [row_lo(c), row_lo(c+1)) of a packed lower triangle of size kd: equal shares of the
// kd(kd+1)/2 entries (cumulative work ~ i^2/2)
// Cost model: a row costs its entries plus rc (its batch setup and reduction share), so the
// CTA holding the many short leading rows is not the cluster's straggler.
__device__ __forceinline__ int row_lo(int c, int C, int kd, int rc = 0) {
  if (c <= 0) return 0;
  if (c >= C) return kd;
  const double a = rc + 0.5;
  const double total = 0.5 * kd * kd + a * kd;  // F(r) = r^2/2 + a r
  const double target = total * c / C;
  int r = static_cast<int>(-a + sqrt(a * a + 2.0 * target) + 0.5);
  return min(max(r, c), kd - (C - c));
}

// ----------------------------------------------------------------- twisted chains
// Lines 0..m-1 are factored top-down (chain 0), lines L-1..m+1 bottom-up (chain 1), and the
// middle line m closes both:
//   chain 0:  D_l = A_ll - B_l D_{l-1}^-1 B_l,        chain 1:  E_l = A_ll - B_{l+1} E_{l+1}^-1 B_{l+1}
//   middle:   T = A_mm - B_m D_{m-1}^-1 B_m - B_{m+1} E_{m+1}^-1 B_{m+1}
// A_i^-1 r then runs forward from both ends to the middle and backward from the middle out,
// halving the sequential depth of both the factorization and the solve.

// ----------------------------------------------------------------- K5 factor
constexpr int kFT = 512;  // factor threads per CTA (16 warps)
constexpr int kFW = kFT / 32;

// A_RR -= Z Z^T on the 32x32 tile (TU, TV) of the lower triangle (rows/columns of K
// excluded): 4x8 thread tiles (rows ub0+16q+2ui+{0,1}, columns vb0+8q+2vi+{0,1}:
// conflict-free double2 reads of Z)
__device__ __forceinline__ void rupd_tile(double* __restrict__ D, int kd, int kdp,
                                          const double* __restrict__ Z, int nbk, int k0, int k1,
                                          int TU, int TV, int lane) {
  const int ui = lane & 7, vi = lane >> 3;
  const int ub0 = 32 * TU + 2 * ui, vb0 = 32 * TV + 2 * vi;
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // the tile's read-modify-write targets -> L1
    const int u = ub0 + 16 * (i >> 1) + (i & 1);
    if (u < kd && (vi & 1) == 0)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(D + prow_off32(u) + 32 * TV + 8 * vi));
  }
  double acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
#pragma unroll 2
  for (int c = 0; c < nbk; ++c) {
    const double* zc = Z + c * kdp;
    double a[4], b[8];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const double2 x = *reinterpret_cast<const double2*>(zc + ub0 + 16 * q);
      a[2 * q] = x.x, a[2 * q + 1] = x.y;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 y = *reinterpret_cast<const double2*>(zc + vb0 + 8 * q);
      b[2 * q] = y.x, b[2 * q + 1] = y.y;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
  }
  // read-modify-write in 16-byte pairs (see rupd_tile_mma)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int u = ub0 + 16 * (i >> 1) + (i & 1);
    if (u >= kd || (u >= k0 && u < k1)) continue;
    double* rowp = D + prow_off32(u);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int v = vb0 + 8 * m;
      if (v <= u && (v < k0 || v >= k1)) {
        double2* pp = reinterpret_cast<double2*>(rowp + v);
        double2 x = *pp;
        x.x -= acc[i][2 * m];
        x.y -= acc[i][2 * m + 1];
        *pp = x;
      }
    }
  }
}

// P (stride NB+1, lower) <- A_K'K' - Z_K' Z_K'^T for the next pivot block K' = [k1, k1+nb1)
// (k1 a multiple of 32): the 32x32 tile of rupd_tile, read from D but written to P only.
// Split over 4 warps (part = warp 0..3): rows 8 part .. 8 part + 7, lane -> 2 rows x 4 cols.
template <int NB>
__device__ __forceinline__ void kk_update(const double* __restrict__ D, int kd, int kdp,
                                          const double* __restrict__ Z, int nbk, int k1,
                                          int nb1, double* P, int lane, int part) {
  const int ui = lane & 3, vi = lane >> 2;
  const int u0 = 8 * part + 2 * ui, v0 = 4 * vi;
  double acc[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  if (v0 <= u0 + 1) {
#pragma unroll 4
    for (int c = 0; c < nbk; ++c) {
      const double* zc = Z + c * kdp + k1;
      const double2 a = *reinterpret_cast<const double2*>(zc + u0);
      const double2 b0 = *reinterpret_cast<const double2*>(zc + v0);
      const double2 b1 = *reinterpret_cast<const double2*>(zc + v0 + 2);
      const double b[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[0][j] = fma(a.x, b[j], acc[0][j]);
        acc[1][j] = fma(a.y, b[j], acc[1][j]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int u = u0 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int v = v0 + j;
      if (v <= u && u < nb1)
        P[u * (NB + 1) + v] = D[prow_off32(k1 + u) + k1 + v] - acc[i][j];
    }
  }
}

// kk_update on the FP64 tensor cores (NB = 32; defined after dmma_8x8x4)
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b);
__device__ __forceinline__ void kk_update_mma(const double* __restrict__ D, int zs,
                                              const double* __restrict__ Z, int nbk, int k1,
                                              int nb1, double* P, int lane, int part) {
  // row block `part` (rows 8 part .. 8 part + 7 of K'), column blocks 0..part; the A_K'K'
  // entries are loaded first so their latency hides behind the products
  const int g = lane >> 2, t = lane & 3;
  const int u = 8 * part + g;
  double d0[4][2];
#pragma unroll
  for (int nb = 0; nb < 4; ++nb)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int v = 8 * nb + 2 * t + h;
      d0[nb][h] = (nb <= part && v <= u && u < nb1) ? D[prow_off32(k1 + u) + k1 + v] : 0.0;
    }
  // even and odd k-steps in separate accumulators: two dependent DMMA chains of 4 instead of
  // one of 8 (a warp has at most 4 blocks, too few to hide the DMMA latency otherwise)
  double acc[2][4][2];
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) acc[e][nb][0] = acc[e][nb][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    if (4 * ks >= nbk) break;
    const double* zc = Z + (4 * ks + t) * zs + k1;  // A[m][k] = Z[k][k1+m], B[k][n] = Z[k][k1+n]
    const double a = zc[8 * part + g];
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
      if (nb <= part) dmma_8x8x4(acc[ks & 1][nb], a, zc[8 * nb + g]);
  }
#pragma unroll
  for (int nb = 0; nb < 4; ++nb)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int v = 8 * nb + 2 * t + h;
      if (nb <= part && v <= u && u < nb1)
        P[u * 33 + v] = d0[nb][h] - (acc[0][nb][h] + acc[1][nb][h]);
    }
}

// A_RK <- Z L^-1 on rows r0..r0+31 (rows of K skipped): out[u][c] = sum_c2 Z[c2][u] Li[c2][c],
// written to D[u][k0 + c] (u > k0) or its transpose D[k0 + c][u] (u < k0). Lane: 4 rows x 4
// columns per pass, NB/16 passes (register budget of the factor kernel).
template <int NB>
__device__ __forceinline__ void tile_ark(double* __restrict__ D, int kd, int kdp,
                                         const double* Z, const double* Li, int r0, int k0,
                                         int k1, int lane) {
  constexpr int LDL = li_stride<NB>();
  const int ui = lane & 7, vi = lane >> 3;
  const int nbk = k1 - k0;
#pragma unroll 1
  for (int pass = 0; pass < NB / 16; ++pass) {
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    const int cb = 16 * pass + 2 * vi;  // columns cb, cb+1, cb+8, cb+9
#pragma unroll 4
    for (int c2 = 0; c2 < NB; ++c2) {
      double a[4], b[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double2 x = *reinterpret_cast<const double2*>(Z + c2 * kdp + r0 + 2 * ui + 16 * h);
        a[2 * h] = x.x, a[2 * h + 1] = x.y;
        const double2 y = *reinterpret_cast<const double2*>(Li + c2 * LDL + cb + 8 * h);
        b[2 * h] = y.x, b[2 * h + 1] = y.y;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    // 16-byte stores: column pairs (c, c + 1) of a row below K, row pairs (u, u + 1) of the
    // transposed block above K (u even, k0 even)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int u = r0 + 2 * ui + 16 * (i >> 1) + (i & 1);
      if (u >= kd || (u >= k0 && u < k1) || u < k0) continue;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int c = cb + 8 * m;
        if (c + 1 < nbk)
          *reinterpret_cast<double2*>(D + prow_off32(u) + k0 + c) =
              make_double2(acc[i][2 * m], acc[i][2 * m + 1]);
        else if (c < nbk)
          D[prow_off32(u) + k0 + c] = acc[i][2 * m];
      }
    }
#pragma unroll
    for (int m = 0; m < 2; ++m) {  // rows u = r0 + 2 ui + 16 m and u + 1 above K
      const int u = r0 + 2 * ui + 16 * m;
      if (u >= k0) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = cb + 8 * (j >> 1) + (j & 1);
        if (c >= nbk) continue;
        *reinterpret_cast<double2*>(D + prow_off32(k0 + c) + u) =
            make_double2(acc[2 * m][j], acc[2 * m + 1][j]);
      }
    }
  }
}

// A_KK <- -L^-T L^-1 (lower triangle), one warp (4 rows x 4 columns per lane and pass)
template <int NB>
__device__ __forceinline__ void tile_akk(double* __restrict__ D, int kd, const double* Li, int k0,
                                         int nbk, int lane) {
  constexpr int LDL = li_stride<NB>();
  const int ui = lane & 7, vi = lane >> 3;
#pragma unroll 1
  for (int pass = 0; pass < NB / 16; ++pass) {
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    const int cb = 16 * pass + 2 * vi;
    for (int m = 0; m < nbk; ++m) {
      double a[4], b[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double2 x = *reinterpret_cast<const double2*>(Li + m * LDL + 2 * ui + 16 * h);
        a[2 * h] = x.x, a[2 * h + 1] = x.y;
        const double2 y = *reinterpret_cast<const double2*>(Li + m * LDL + cb + 8 * h);
        b[2 * h] = y.x, b[2 * h + 1] = y.y;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = 2 * ui + 16 * (i >> 1) + (i & 1);
      if (r >= nbk) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = cb + 8 * (j >> 1) + (j & 1);
        if (c <= r) D[prow_off32(k0 + r) + k0 + c] = -acc[i][j];
      }
    }
  }
}

// The same tile update on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64): a warp holds
// the 32x32 tile as 4x4 accumulator blocks of 8x8 (2 doubles per lane each); per k-step of 4
// pivot columns it loads one A fragment per row block and one B fragment per column block
// (8 shared-memory loads for 16 MMAs = 4096 FMAs), a quarter of the operand traffic of the
// 4x8 FFMA register tile, which is shared-memory bound on wide lines.
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void rupd_tile_mma(double* __restrict__ D, int kd, int kdp,
                                              const double* __restrict__ Z, int nbk, int k0,
                                              int k1, int TU, int TV, int lane) {
  const int g = lane >> 2, t = lane & 3;  // fragment row/col group, thread in group
  const int u0 = 32 * TU, v0 = 32 * TV;
  const bool diag = TU == TV;
#ifndef FFB_ACCX
#define FFB_ACCX 1
#endif
  // The tile's entries are the accumulators' initial values (FFB_ACCX): D - Z Z^T is formed as
  // D + (-Z) Z^T in the DMMA chain itself, so all 16 pair loads of the tile are in flight at
  // once before the first product — one exposed L2 round trip per tile instead of one per
  // RG row blocks after the products (the RG = 1 / 2 / 4 sweep, profiles/r2_factor_knobs.txt,
  // shows how much of a tile is that latency) — and no second register set for them.
  // 16-byte pairs (v even; K is 32-aligned, so a pair is wholly inside or outside it). The
  // pair at v = u of an even row u also rewrites the row's pad, which nothing reads during the
  // sweep and pack_line zeroes at its end.
  double acc[4][4][2];
  unsigned onmask = 0;
  auto pair_ptr = [&](int i, int j) {
    return reinterpret_cast<double2*>(D + prow_off32(u0 + 8 * i + g) + v0 + 8 * j + 2 * t);
  };
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int u = u0 + 8 * i + g;
    const bool row_on = u < kd && !(u >= k0 && u < k1);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int v = v0 + 8 * j + 2 * t;
      const bool on = row_on && !(diag && j > i) && v <= u && (v < k0 || v >= k1);
      onmask |= on ? 1u << (4 * i + j) : 0u;
      double2 x = make_double2(0.0, 0.0);
      if (FFB_ACCX && on) x = *pair_ptr(i, j);
      acc[i][j][0] = x.x, acc[i][j][1] = x.y;
    }
  }
#pragma unroll 2
  for (int c0 = 0; c0 < nbk; c0 += 4) {
    const double* zc = Z + (c0 + t) * kdp;  // A[m][k] = Z[c0+k][u0+m], B[k][n] = Z[c0+k][v0+n]
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = zc[u0 + 8 * i + g];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = diag ? a[j] : zc[v0 + 8 * j + g];
    if (FFB_ACCX) {
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = -a[i];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (!diag || j <= i) dmma_8x8x4(acc[i][j], a[i], b[j]);
  }
  if (FFB_ACCX) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (onmask >> (4 * i + j) & 1u) *pair_ptr(i, j) = make_double2(acc[i][j][0], acc[i][j][1]);
    return;
  }
  // FFB_ACCX = 0: read-modify-write after the products, RG row blocks of loads before their
  // stores (written load-store per pair, the compiler keeps the order — the stores may alias
  // the next loads — and the tile pays one L2 round trip per pair).
#ifndef FFB_RG
#define FFB_RG 2
#endif
  constexpr int RG = FFB_RG;
#pragma unroll
  for (int i0 = 0; i0 < 4; i0 += RG) {
    double2 x[RG][4];
#pragma unroll
    for (int ii = 0; ii < RG; ++ii)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        x[ii][j] = (onmask >> (4 * (i0 + ii) + j) & 1u) ? *pair_ptr(i0 + ii, j) : make_double2(0.0, 0.0);
#pragma unroll
    for (int ii = 0; ii < RG; ++ii)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (onmask >> (4 * (i0 + ii) + j) & 1u)
          *pair_ptr(i0 + ii, j) = make_double2(x[ii][j].x - acc[i0 + ii][j][0], x[ii][j].y - acc[i0 + ii][j][1]);
  }
}

// tile_ark on the FP64 tensor cores (NB = 32): out[u][c] = sum_c2 Z[c2][u] Li[c2][c] as 4x4
// DMMA blocks, A[m][k] = Z[c0+k][r0+m], B[k][n] = Li[c0+k][n]; column block j needs only the
// k-steps from its diagonal on (Li is lower triangular). Besides a quarter of the issue
// slots of the FFMA tile, it keeps the FP64 FFMA pipe free for the pivot warps' chain.
__device__ __forceinline__ void tile_ark_mma(double* __restrict__ D, int kd, int zs,
                                             const double* Z, const double* Li, int r0, int k0,
                                             int k1, int lane) {
  constexpr int LDL = li_stride<32>();
  const int g = lane >> 2, t = lane & 3;
  const int nbk = k1 - k0;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 2
  for (int ks = 0; ks < 8; ++ks) {
    const double* zc = Z + (4 * ks + t) * zs + r0;
    const double* lc = Li + (4 * ks + t) * LDL;
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = zc[8 * i + g];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = lc[8 * j + g];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (ks >= 2 * j) dmma_8x8x4(acc[i][j], a[i], b[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int u = r0 + 8 * i + g;
    if (u >= kd || (u >= k0 && u < k1)) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = 8 * j + 2 * t;
      if (u >= k1) {  // row u below K: columns (c, c + 1) of its K segment, 16-byte store
        if (c + 1 < nbk)
          *reinterpret_cast<double2*>(D + prow_off32(u) + k0 + c) =
              make_double2(acc[i][j][0], acc[i][j][1]);
        else if (c < nbk)
          D[prow_off32(u) + k0 + c] = acc[i][j][0];
      } else {  // row u above K: stored transposed, in rows k0 + c and k0 + c + 1
        if (c < nbk) D[prow_off32(k0 + c) + u] = acc[i][j][0];
        if (c + 1 < nbk) D[prow_off32(k0 + c + 1) + u] = acc[i][j][1];
      }
    }
  }
}

#ifndef FFB_ARK_MMA
#define FFB_ARK_MMA 1
#endif
template <int NB>
__device__ __forceinline__ void ark_tile(bool use_mma, double* __restrict__ D, int kd, int zs,
                                         const double* Z, const double* Li, int r0, int k0,
                                         int k1, int lane) {
  if constexpr (NB == 32 && FFB_ARK_MMA) {
    if (use_mma) return tile_ark_mma(D, kd, zs, Z, Li, r0, k0, k1, lane);
  }
  tile_ark<NB>(D, kd, zs, Z, Li, r0, k0, k1, lane);
}

// P (stride NB+1) <- the nbk x nbk diagonal block at (k, k) of the packed line D (lower)
template <int NB>
__device__ __forceinline__ void load_block(const double* __restrict__ D, int k, int nbk,
                                           double* P, int lane) {
  double v[NB];
#pragma unroll
  for (int a = 0; a < NB; ++a)  // all loads in flight before the first store
    v[a] = (a < nbk && lane <= a) ? D[prow_off32(k + a) + k + lane] : 0.0;
#pragma unroll
  for (int a = 0; a < NB; ++a)
    if (a < nbk && lane <= a) P[a * (NB + 1) + lane] = v[a];
  __syncwarp();
}

// In-place inversion of the SPD line matrix D (its packed lower triangle, rows at prow_off, in
// the line's own factor storage) by the blocked symmetric sweep; leaves -D^{-1} there.
// The next step's pivot block is factored by warp 0 while the other 15 warps write the
// current step's A_RK and A_KK (tile updates from a dynamic queue).
// Shared memory: P (NB x NB+1), Li[2] (double-buffered), ir (NB), the tile counter, Z.
template <int NB>
__device__ void sweep_invert(double* __restrict__ D, int kd, int kdp, double* P, double* Li2,
                             double* ir, int* cnt, double* Z, int& first_bad, int bad_base,
                             int la, int q, int C) {
  const bool use_mma = la & 2;  // tile updates on the FP64 tensor cores
  la &= 1;
  // Z row stride: kdp + 4 doubles. A 64-bit shared load is served per half-warp (16 lanes,
  // 128 B); a DMMA fragment load's half-warp touches 4 pivot-column rows x 32 B, which this
  // stride puts on 4 distinct 32-byte bank groups (one wavefront; kdp + 8 took two — ncu
  // r1f_factor_c2: 2x the ideal wavefronts), and the Z stores' rows 2 apart on two (was four).
  const int zs = kdp + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int LDL = li_stride<NB>();
  constexpr int LS = NB * LDL;
  PROF_DECL
  if (tid == 0) cnt[0] = 0, cnt[3] = 0;
  if (warp == 0) {
    load_block<NB>(D, 0, min(NB, kd), P, lane);
    pivot_warp<NB>(P, NB + 1, 0, min(NB, kd), P, Li2, ir, first_bad, bad_base, nullptr);
  }
  const bool la_reg = NB == 32 && la;  // look-ahead on a private copy of the next pivot block
  int pv_tag = 0;                      // pivot_pair progress tags (warps 0-3)
  if (tid == 0) cnt[2] = 0;
  const int nt = (kd + 31) / 32;
  const int ntiles = nt * (nt + 1) / 2;
  int step = 0;
  for (int k0 = 0; k0 < kd; k0 += NB, ++step) {
    const int nbk = min(NB, kd - k0);
    const int k1 = k0 + nbk;
    const double* Li = Li2 + (step & 1) * LS;
    double* Lnext = Li2 + ((step + 1) & 1) * LS;
    __syncthreads();
    if (tid == 0) {  // the queues of the next step (idle since the sync)
      cnt[(step + 1) & 1] = 0;
      cnt[3 + ((step + 1) & 1)] = 0;
    }
    PROF_MARK(1); FTL_MARK(0);
#ifndef FFB_KKPF
#define FFB_KKPF 1
#endif
    if (FFB_KKPF && la_reg && warp < 4 && k1 < kd && lane < 16) {
      // the next pivot block A_K'K' is final since the previous step (its tile is the
      // look-ahead's private copy now): pull its rows into L1 while Z is formed, so the
      // look-ahead update after the Z barrier does not wait a full L2 round trip for them
      const int u = 8 * warp + (lane >> 1);
      if (u < min(NB, kd - k1)) {
        const double* pf = D + prow_off32(k1 + u) + k1 + 16 * (lane & 1);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(pf));
      }
    }
    // ---- Z = A_RK Li^T
    if constexpr (NB == 32) {
      // on the FP64 tensor cores: rows in blocks of 8 (K is 8-aligned, so a block is wholly
      // inside or outside it), D[8x8] += A[8x4] B[4x8] with A = the panel, B = Li^T; column
      // block nb only needs the k-steps up to its diagonal (Li is lower triangular)
      const int g = lane >> 2, t4 = lane & 3;
      // the next row block's panel loads are issued before this block's products
      double an[8];
      auto load_panel = [&](int rb) {
        const int i = 8 * rb + g;
        const bool live = 8 * rb < kdp && i < kd && (i < k0 || i >= k1);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const int c2 = 4 * ks + t4;
          an[ks] = (live && c2 < nbk) ? (i > k0 ? D[prow_off32(i) + k0 + c2] : D[prow_off32(k0 + c2) + i])
                                      : 0.0;
        }
      };
      // la_reg on a cluster: the row blocks are split between groups of FFB_ZSPLIT CTAs, and
      // each block is stored into the Z of every CTA of its group (distributed shared memory;
      // the cluster barrier after the Z phase orders it, the previous step's final one frees
      // the buffers). The panel loads are the cost (one L2 round trip per row block); 2-way
      // beats 4-way, where the remote stores (~20 B/clk per SM) take what the loads saved.
#ifndef FFB_ZSPLIT
#define FFB_ZSPLIT 2
#endif
      const int zs_n = la_reg ? min(C, FFB_ZSPLIT) : 1;  // CTAs sharing the Z row blocks
      const int zs_base = q - q % zs_n;
      const int rb0 = (q % zs_n) * kFW + warp, rstep = kFW * zs_n;
      load_panel(rb0);
      for (int rb = rb0; 8 * rb < kdp; rb += rstep) {
        double a[8];
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) a[ks] = an[ks];
        load_panel(rb + rstep);
        // two accumulator chains per column block (even / odd k-steps; see kk_update_mma)
        double acc[4][2], acc1[4][2];
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          acc[nb][0] = acc[nb][1] = acc1[nb][0] = acc1[nb][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            if (ks <= 2 * nb + 1)
              dmma_8x8x4((ks & 1) ? acc1[nb] : acc[nb], a[ks], Li[(8 * nb + g) * LDL + 4 * ks + t4]);
          acc[nb][0] += acc1[nb][0];
          acc[nb][1] += acc1[nb][1];
        }
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
          for (int h = 0; h < 2; ++h) Z[(8 * nb + 2 * t4 + h) * zs + 8 * rb + g] = acc[nb][h];
#pragma unroll 1
        for (int r = 1; r < zs_n; ++r) {
          double* Zr = cl_map(Z, static_cast<unsigned>(zs_base + (q % zs_n + r) % zs_n));
#pragma unroll
          for (int nb = 0; nb < 4; ++nb)
#pragma unroll
            for (int h = 0; h < 2; ++h) Zr[(8 * nb + 2 * t4 + h) * zs + 8 * rb + g] = acc[nb][h];
        }
        if (warp >= 4 && rb == rb0) FTL_MARK(3);  // first row block stored
      }
      if (warp >= 4) FTL_MARK(2);  // Z loop done (before the barrier)
    } else {
    // thread per row: all loads issued first, 32 independent chains
    for (int i = tid; i < kdp; i += kFT) {
      const bool live = i < kd && (i < k0 || i >= k1);
      double a[NB];
      if (live && i > k0) {
        // row i's segment of the panel: 16-byte loads (rows start 16-byte aligned, k0 even)
        const double2* row = reinterpret_cast<const double2*>(D + prow_off32(i) + k0);
#pragma unroll
        for (int c = 0; c < NB; c += 2) {
          const double2 v = c < nbk ? row[c / 2] : make_double2(0.0, 0.0);
          a[c] = v.x;
          a[c + 1] = c + 1 < nbk ? v.y : 0.0;
        }
      } else {
#pragma unroll
        for (int c = 0; c < NB; ++c) a[c] = (live && c < nbk) ? D[prow_off32(k0 + c) + i] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int c2 = 0; c2 <= c; ++c2) acc = fma(a[c2], Li[c * LDL + c2], acc);
        Z[c * zs + i] = acc;
      }
    }
    }
    // la_reg: A_RK is overwritten during this step's tile phase, so every CTA's Z must be
    // done first (cluster barrier); otherwise a CTA barrier suffices here
    if (la_reg && C > 1) cl_sync(); else __syncthreads();
    PROF_MARK(2); FTL_MARK(1);
    // ---- A_RR -= Z Z^T, 32x32 tiles from a shared queue (tiles q, q + C, ... of the
    // cluster's CTA q). Look-ahead (la, single CTA): warp 0 first finishes the tile holding
    // the next pivot block and factors that block meanwhile.
    const int nx = (la && k1 < kd) ? k1 / 32 : -1;
    const int special = nx >= 0 ? nx * (nx + 1) / 2 + nx : -1;
    if (la_reg && warp < 4 && special >= 0) {
      // NB = 32: tile (nx, nx) is exactly the next pivot block K', needed by nothing but the
      // pivot (A_KK is overwritten at its own step). Every CTA of the cluster updates a
      // private copy in P (warps 0-3) and factors it (warp 0); nobody writes the tile back,
      // so there is no ordering against the other CTAs' updates.
      if constexpr (NB == 32)
        kk_update_mma(D, zs, Z, nbk, k1, min(NB, kd - k1), P, lane, warp);
      else
        kk_update<NB>(D, kd, zs, Z, nbk, k1, min(NB, kd - k1), P, lane, warp);
      asm volatile("bar.sync 2, 128;" ::: "memory");
      PROF_MARK(6); FTL_MARK(2);
      if (warp < 2)
        pivot_pair<NB>(P, NB + 1, k1, min(NB, kd - k1), P, Lnext, ir, first_bad, bad_base,
                       cnt + 2, ++pv_tag, nullptr);
      else
        ++pv_tag;
      PROF_MARK(5); FTL_MARK(3);
    } else if (warp == 0 && special >= 0) {
      {
        rupd_tile(D, kd, zs, Z, nbk, k0, k1, nx, nx, lane);
        __syncwarp();
        load_block<NB>(D, k1, min(NB, kd - k1), P, lane);
        pivot_warp<NB>(P, NB + 1, k1, min(NB, kd - k1), P, Lnext, ir, first_bad, bad_base,
                       nullptr);
      }
      PROF_MARK(5);
    }
    if (la_reg) {
      // A_RK <- Z L^-1 (row tiles q, q + C, ... of the cluster) and A_KK, concurrently with the
      // trailing updates: they touch only the columns of K, which the tiles exclude
      if (q == C - 1 && warp == kFW - 1) tile_akk<NB>(D, kd, Li, k0, nbk, lane);
#ifdef FFB_PROFILE
      long long ftl_t0 = clock64(), ftl_n = 0;
#endif
      for (;;) {
        int T = 0;
        if (lane == 0) T = q + C * atomicAdd(cnt + 3 + (step & 1), 1);
        T = __shfl_sync(~0u, T, 0);
        if (32 * T >= kd) break;
        ark_tile<NB>(use_mma, D, kd, zs, Z, Li, 32 * T, k0, k1, lane);
#ifdef FFB_PROFILE
        ++ftl_n;
#endif
      }
#ifdef FFB_PROFILE
      if (blockIdx.x == 0 && bad_base == 10 * kd && step < 16 && lane == 0)
        g_ftl[step][warp][6] = (clock64() - ftl_t0) * 16 + ftl_n;
#endif
    }
#ifdef FFB_PROFILE
    long long ftl_t1 = clock64(), ftl_m = 0;
#endif
    for (;;) {
      int idx = 0;
      if (lane == 0) idx = q + C * atomicAdd(cnt + (step & 1), 1);
      idx = __shfl_sync(~0u, idx, 0);
      if (idx >= ntiles) break;
      if (idx == special) continue;
      // tile row from the triangular index: single-precision estimate, exact integer fix-up
      // (a double sqrt here stalled the queue loop: 5% of the kernel's warp stall samples)
      int TU = static_cast<int>((sqrtf(8.0f * static_cast<float>(idx) + 1.0f) - 1.0f) * 0.5f);
      while (TU * (TU + 1) / 2 > idx) --TU;
      while ((TU + 1) * (TU + 2) / 2 <= idx) ++TU;
      if (use_mma)
        rupd_tile_mma(D, kd, zs, Z, nbk, k0, k1, TU, idx - TU * (TU + 1) / 2, lane);
      else
        rupd_tile(D, kd, zs, Z, nbk, k0, k1, TU, idx - TU * (TU + 1) / 2, lane);
#ifdef FFB_PROFILE
      ++ftl_m;
#endif
    }
#ifdef FFB_PROFILE
    if (blockIdx.x == 0 && bad_base == 10 * kd && step < 16 && lane == 0)
      g_ftl[step][warp][7] = (clock64() - ftl_t1) * 16 + ftl_m;
#endif
    // all tile updates (and, across the cluster, all reads of A_RK for Z) are done
    if (!la_reg) {
      if (C > 1) cl_sync(); else __syncthreads();
    }
    PROF_MARK(3); FTL_MARK(4);
    if (la_reg) {
      // A_RK, A_KK done in the tile phase
    } else if (!la && warp == 0) {
      // the next pivot block is final now: factor it while the other warps write A_RK, A_KK
      if (k1 < kd)
        load_block<NB>(D, k1, min(NB, kd - k1), P, lane),
            pivot_warp<NB>(P, NB + 1, k1, min(NB, kd - k1), P, Lnext, ir, first_bad, bad_base,
                           nullptr);
      PROF_MARK(5);
    } else {
      // ---- A_RK <- Z Li ; A_KK <- -Li^T Li, as 32x32 tiles (4x8 per lane): row tiles
      // q, q + C, ... of the cluster over this CTA's participating warps; A_KK by one warp
      const int w0 = la ? 0 : 1, nw = kFW - w0, wi = warp - w0;
      for (int T = q + C * wi; 32 * T < kd; T += C * nw) {
        ark_tile<NB>(use_mma, D, kd, zs, Z, Li, 32 * T, k0, k1, lane);
      }
      if (q == C - 1 && warp == kFW - 1) tile_akk<NB>(D, kd, Li, k0, nbk, lane);
    }
    PROF_MARK(7);
    if (C > 1) cl_sync();  // A_RK, A_KK written cluster-wide before the next Z / pack
    PROF_MARK(4); FTL_MARK(5);
  }
  __syncthreads();
  PROF_FLUSH(32);
}

// D <- A_ll - sum over the given neighbour lines of B (inv_nb) B  (lower triangle)
__device__ void build_line(const SubInfo& s, const double* __restrict__ coef, size_t N, int W,
                           int nc, int l, int nb0, int bl0, int nb1, int bl1,
                           const double* __restrict__ F, double* __restrict__ D, int q,
                           int C) {
  // neighbour nbX (line index or -1) with coupling taken at line blX (bcoef(blX): between
  // lines blX and blX-1). CTA q of the cluster builds rows kFW q + (kFW C) k + warp, which
  // read only the same rows of the neighbour inverses (packed by this CTA: pack_line uses
  // the same split).
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kd = s.kd;
  for (int i = warp + kFW * q; i < kd; i += kFW * C) {
    const double b0i = nb0 >= 0 ? bcoef(s, coef, N, W, nc, bl0, i) : 0.0;
    const double b1i = nb1 >= 0 ? bcoef(s, coef, N, W, nc, bl1, i) : 0.0;
    const long long oi = prow_off(i);
    for (int j = lane; j <= i; j += 32) {
      double v = aline(s, coef, N, W, nc, l, i, j);
      if (nb0 >= 0)
        v -= b0i * bcoef(s, coef, N, W, nc, bl0, j) * F[static_cast<long long>(nb0) * s.line_sz + oi + j];
      if (nb1 >= 0)
        v -= b1i * bcoef(s, coef, N, W, nc, bl1, j) * F[static_cast<long long>(nb1) * s.line_sz + oi + j];
      D[oi + j] = v;
    }
  }
  __syncthreads();
}

// ---- tile-major line layout (the register-tiled solve streams whole tiles) ----------------
// A line's lower triangle as 32x32 tiles (I, J), I >= J, row-major; tile row I has
// h = min(32, kd - 32 I) rows. An off-diagonal tile stores its h rows of 32 entries, a
// diagonal tile its packed lower triangle (local row r: r + 1 entries padded to even, at
// prow_off(r)). Same number of doubles as the packed row layout (tile_line_size == prow_off).
__host__ __device__ __forceinline__ int tile_h(int I, int kd) { return min(32, kd - 32 * I); }
__host__ __device__ __forceinline__ long long tile_row_off(int I, int kd) {
  // tile rows before I are full (h = 32): I off-diagonal tiles of 1024 + one diagonal of 544
  (void)kd;
  return 1024LL * I * (I - 1) / 2 + 544LL * I;
}
__host__ __device__ __forceinline__ long long tile_off(int I, int J, int kd) {
  return tile_row_off(I, kd) + 32LL * tile_h(I, kd) * J;
}
__host__ __device__ __forceinline__ int tile_size(int I, int J, int kd) {
  const int h = tile_h(I, kd);
  return I == J ? static_cast<int>(prow_off(h)) : 32 * h;
}

// the sweep leaves -D^-1 in place in the packed line: negate it, zero the pads of even rows
// (Ft: the tile-major copy the register-tiled solve streams, written in the same pass with the
// diagonal halved — see k_line_solve_tile; nullptr when that solve is not used)
__device__ __noinline__ void pack_line(const SubInfo& s, int l, double* F, int q, int C, double* Ft) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kd = s.kd;
  double* Fl = F + static_cast<long long>(l) * s.line_sz;
  double* Tl = Ft ? Ft + s.fac_off + static_cast<long long>(l) * s.line_sz : nullptr;
  for (int i = warp + kFW * q; i < kd; i += kFW * C) {
    const int o = prow_off32(i);
    const int I = i >> 5, r = i & 31;
    for (int j = lane; j <= i; j += 32) {
      const double v = -Fl[o + j];
      Fl[o + j] = v;
      if (Tl) {
        const int J = j >> 5;
        const long long d = tile_off(I, J, kd) + (I == J ? prow_off32(r) + (j & 31) : 32 * r + (j & 31));
        Tl[d] = j == i ? 0.5 * v : v;
      }
    }
    if ((i & 1) == 0 && lane == 0) {
      Fl[o + i + 1] = 0.0;
      if (Tl) Tl[tile_off(I, I, kd) + prow_off32(r) + r + 1] = 0.0;
    }
  }
  __syncthreads();
}

// one thread-block cluster of C CTAs per (subdomain, chain): chain 0 lines 0..m-1 downward,
// chain 1 lines L-1..m+1 upward; mid = 1 launches one cluster per subdomain for the middle
// line. The CTAs of a cluster share the line matrix D (global scratch, L2-resident): each
// builds and packs its share of the rows, takes every C-th tile of the trailing updates and
// its share of the A_RK rows, and factors the pivot blocks redundantly (no exchange).
template <int NB>
__global__ void __launch_bounds__(kFT, 1)
    k_line_factor(const SubInfo* __restrict__ subs, const double* __restrict__ coef, size_t N,
                  int W, int nc, double* __restrict__ fac, double* __restrict__ fac_t,
                  double* __restrict__ scratch,
                  long long scratch_stride, int kdp, int mid, int* __restrict__ bad,
                  const int2* __restrict__ changed, int la) {
  const int C = static_cast<int>(cl_size()), q = static_cast<int>(cl_rank());
  const int cid = blockIdx.x / C;
  const int sub = mid ? cid : cid >> 1;
  const int chain = mid ? 0 : cid & 1;
  const SubInfo s = subs[sub];
  const int tid = threadIdx.x;
  const int kd = s.kd, L = s.L, m = s.m;
  // lines [lo, hi] of this subdomain whose operator changed since the last factorisation
  // (all of them on a full refactorisation): chain 0 restarts at lo, chain 1 at hi, and the
  // untouched prefix of each chain keeps its inverses (D_l depends on lines <= l only)
  const int2 chg = changed ? changed[sub] : make_int2(0, L - 1);
  if (chg.x > chg.y) return;  // nothing changed in this subdomain
  double* F = fac + s.fac_off;  // each line is built, inverted and negated in place
  extern __shared__ __align__(16) double fsm[];
  constexpr int LDL = li_stride<NB>();
  double* P = fsm;                      // NB x (NB+1)
  double* Li = P + NB * (NB + 1);       // 2 x NB x LDL (double-buffered L^-1)
  double* ir = Li + 2 * NB * LDL;       // NB
  int* cnt = reinterpret_cast<int*>(ir + NB);
  double* Z = ir + 2 * NB;              // NB x kdp
  for (int e = tid; e < NB * (kdp + 8); e += kFT) Z[e] = 0.0;
  int first_bad = 0x7fffffff;
  PROF_DECL
  if (mid) {
    double* D = F + static_cast<long long>(m) * s.line_sz;
    build_line(s, coef, N, W, nc, m, m > 0 ? m - 1 : -1, m, m < L - 1 ? m + 1 : -1, m + 1, F, D,
               q, C);
    if (C > 1) cl_sync();
    PROF_MARK(0);
    sweep_invert<NB>(D, kd, kdp, P, Li, ir, cnt, Z, first_bad, m * kd, la, q, C);
    pack_line(s, m, F, q, C, fac_t);
  } else {
    const int nlines = chain == 0 ? m : L - 1 - m;
    const int t0 = chain == 0 ? chg.x : L - 1 - chg.y;
    for (int t = max(t0, 0); t < nlines; ++t) {
      const int l = chain == 0 ? t : L - 1 - t;
      const int prev = t == 0 ? -1 : (chain == 0 ? l - 1 : l + 1);
      const int bl = chain == 0 ? l : l + 1;  // coupling between l and prev
      double* D = F + static_cast<long long>(l) * s.line_sz;
      build_line(s, coef, N, W, nc, l, prev, bl, -1, 0, F, D, q, C);
      if (C > 1) cl_sync();
      PROF_MARK(0);
      sweep_invert<NB>(D, kd, kdp, P, Li, ir, cnt, Z, first_bad, l * kd, la, q, C);
      pack_line(s, l, F, q, C, fac_t);
      PROF_MARK(5);
    }
  }
  PROF_FLUSH(0);
  if (tid == 0 && q == 0 && first_bad != 0x7fffffff) atomicMin(bad + sub, first_bad);
}

// ----------------------------------------------------------------- K6 solve
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Waits are bounded: a wait that has not completed after ~2e11 cycles (about 100 s — four
// orders of magnitude beyond the longest legitimate one) traps, so a protocol error ends the
// process with a CUDA error instead of hanging it (the fast path, a completed phase on the
// first try, does not read the clock).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      ".reg .s64 t0, t1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE_%=;\n"
      "mov.u64 t0, %%clock64;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE_%=;\n"
      "mov.u64 t1, %%clock64;\n"
      "sub.s64 t1, t1, t0;\n"
      "setp.lt.s64 P1, t1, 200000000000;\n"
      "@P1 bra WAIT_%=;\n"
      "trap;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)  // suspend-time hint: sleep in the wait instead of polling
      : "memory");
}

__device__ __forceinline__ double2 lds_f64x2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// two consecutive entries of a staged factor row as doubles (FT = double: one 16-byte load;
// float, the opt-in single-precision factor copy: one 8-byte load, widened)
template <class FT>
__device__ __forceinline__ double2 lds_pair(uint32_t addr);
template <>
__device__ __forceinline__ double2 lds_pair<double>(uint32_t addr) {
  return lds_f64x2(addr);
}
template <>
__device__ __forceinline__ double2 lds_pair<float>(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
}

// R per-lane partial sums (R = 4 or 8 rows) -> lane ends with the warp total of row
// lane / (32 / R): halving exchanges (16, 8[, 4]) then a butterfly over the rest
template <int R>
__device__ __forceinline__ double transpose_reduce(double (&acc)[R], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8;
  if constexpr (R == 2) {  // one halving exchange, then a butterfly over 16 lanes
    const double send = b4 ? acc[0] : acc[1];
    double t = (b4 ? acc[1] : acc[0]) + __shfl_xor_sync(0xffffffffu, send, 16);
    t += __shfl_xor_sync(0xffffffffu, t, 8);
    t += __shfl_xor_sync(0xffffffffu, t, 4);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    return t;
  }
#pragma unroll
  for (int k = 0; k < R / 2; ++k) {
    const double send = b4 ? acc[k] : acc[k + R / 2];
    const double keep = b4 ? acc[k + R / 2] : acc[k];
    acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < R / 4; ++k) {
    const double send = b3 ? acc[k] : acc[k + R / 4];
    const double keep = b3 ? acc[k + R / 4] : acc[k];
    acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double t = acc[0];
  if (R == 8) {
    const bool b2 = lane & 4;
    const double send = b2 ? acc[0] : acc[1];
    const double keep = b2 ? acc[1] : acc[0];
    t = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  } else {
    t += __shfl_xor_sync(0xffffffffu, t, 4);
  }
  t += __shfl_xor_sync(0xffffffffu, t, 2);
  t += __shfl_xor_sync(0xffffffffu, t, 1);
  return t;
}

#ifndef FFB_SOLVE_WARPS
#define FFB_SOLVE_WARPS 16
#endif
constexpr int kSW = FFB_SOLVE_WARPS;  // solve warps per CTA: kSW - 1 compute + 1 producer
constexpr int kSolveHdr = 1024;  // mbarriers (0..239), task slots (240..255), cluster row table
// development probe (FFB_SOLVE_DBG): 1 skip the row arithmetic, 2 skip the line exchange,
// 4 skip the bulk copies. Results are wrong with any bit set; timing decomposition only.
__device__ int g_solve_dbg = 0;
constexpr int kST = kSW * 32;
constexpr int kCW = kSW - 1;
constexpr int kCT = kCW * 32;
constexpr int kCS = (kCW + 1) / 2;  // column-partial slots (the compute warps reduced in two rounds)

// Row chunking of a CTA's rows [rlo, rhi) of one line: the longest run of rows starting at
// r0 whose packed size fits `cap` doubles (at least one row). Identical on every thread.
__device__ __forceinline__ int chunk_end(int r0, int rhi, long long cap) {
  const long long base = prow_off(r0);
  int r1 = r0 + 1;
  {
    const double t = static_cast<double>(base + cap);
    const int m = static_cast<int>((sqrt(1.0 + 2.0 * t) - 1.0) * 0.5);  // 2m(m+1) <= t
    if (2 * m > r1) r1 = 2 * m;
  }
  if (r1 > rhi) r1 = rhi;
  while (r1 > r0 + 1 && prow_off(r1) - base > cap) --r1;
  while (r1 < rhi && prow_off(r1 + 1) - base <= cap) ++r1;
  return r1;
}

// The same chunk end from a starting guess (the previous chunk's row count): 32-bit and
// without the square root, the loops settle in a step or two because consecutive chunks of a
// line differ by about a row. The result does not depend on the guess (the largest run that
// fits, at least one row). Per chunk on every compute thread, the square-root version cost
// the 4-CTA-cluster solve of c5 ~20% more instructions (ncu r2ab: 1.60e9 vs 1.34e9).
__device__ __forceinline__ int chunk_end_from(int r0, int rhi, int cap, int guess) {
  const int base = prow_off32(r0);
  int r1 = min(r0 + max(guess, 1), rhi);
  while (r1 > r0 + 1 && prow_off32(r1) - base > cap) --r1;
  while (r1 < rhi && prow_off32(r1 + 1) - base <= cap) ++r1;
  return r1;
}

// Lines visited by (phase, chain): forward 0: 0..m-1, forward 1: L-1..m+1; backward: the
// middle m first, then m-1..0 / m+1..L-1. The middle is solved by every chain with a forward
// part (a chain without one — an unbalanced split, m = 0 or m = L-1 — does nothing) and
// written by mid_writer(s).
__device__ __forceinline__ int chain_len(int phase, int chain, const SubInfo& s) {
  const int len0 = s.m, len1 = s.L - 1 - s.m;
  const int len = chain == 0 ? len0 : len1;
  if (phase == 0) return len;
  if (len > 0) return len + 1;
  return (chain == 0 && len1 == 0) ? 1 : 0;  // L == 1: chain 0 solves the single line
}
__device__ __forceinline__ int mid_writer(const SubInfo& s) { return (s.m > 0 || s.L == 1) ? 0 : 1; }
__device__ __forceinline__ int chain_line(int phase, int chain, const SubInfo& s, int t) {
  if (phase == 0) return chain == 0 ? t : s.L - 1 - t;
  return chain == 0 ? s.m - t : s.m + t;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// persistent queue: a backward task waits for its subdomain's forward chains (bounded, as above)
__device__ __forceinline__ void wait_forward_done(const int* p, int need) {
  if (ld_acquire_gpu(p) >= need) return;
  const long long t0 = clock64();
  while (ld_acquire_gpu(p) < need) {
    __nanosleep(100);
    if (clock64() - t0 > 200000000000LL) __trap();
  }
}

// wait with cluster-scope acquire: pairs with remote release-arrivals from the other CTAs
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      ".reg .s64 t0, t1;\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONEC_%=;\n"
      "mov.u64 t0, %%clock64;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONEC_%=;\n"
      "mov.u64 t1, %%clock64;\n"
      "sub.s64 t1, t1, t0;\n"
      "setp.lt.s64 P1, t1, 200000000000;\n"
      "@P1 bra WAITC_%=;\n"
      "trap;\n"
      "DONEC_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// asynchronous store of one double into CTA `rank`'s shared memory at the offset of `dst`,
// completing 8 transaction bytes on that CTA's mbarrier at the offset of `bar`
__device__ __forceinline__ void st_async_remote(double* dst, double v, uint64_t* bar,
                                                unsigned rank) {
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(dst)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra),
               "d"(v), "r"(rb)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// barrier among the compute warps only (the producer warp streams on independently)
__device__ __forceinline__ void compute_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kCT) : "memory");
}

// One sweep (phase 0 forward / 1 backward) of both chains of every subdomain: cluster of C
// CTAs per (subdomain, chain); each line's packed rows are split over the cluster (equal
// entry counts) and the symmetric products combined through distributed shared memory.
// Warp 15 is a producer that streams the CTA's share of every line through the shared-memory
// ring (cp.async.bulk, full/empty mbarriers) independently of the compute warps, so the bulk
// copy engine keeps running across the per-line reductions.
template <int MAXM, bool PERSIST>
__global__ void __launch_bounds__(kST, 1)
    k_line_solve(const SubInfo* __restrict__ subs, const double* __restrict__ fac,
                 const double* __restrict__ coef, size_t N, const double* __restrict__ r,
                 double* __restrict__ ylocal, double* __restrict__ zlocal, int W, int nc,
                 int stages, int cap, int kd_max, int rc, int phase_arg,
                 const int* __restrict__ flags,
                 const double* __restrict__ rlocal, int* __restrict__ qsync, int nsub_all) {
  if (flags && (flags[0] | flags[1])) return;  // PCG converged or failed (grid-uniform)
  const int C = static_cast<int>(cl_size()), crank = static_cast<int>(cl_rank());
  // Tasks (phase, subdomain, chain). One per cluster; or (PERSIST, one CTA per chain, one CTA
  // per SM) a dynamic queue of the whole application — the forward chains of every
  // subdomain, then the backward chains — so the chains fill the SMs without the partly
  // empty last round of a one-chain-per-CTA launch (c4: 512 chains on 148 SMs per sweep).
  // qsync[0] is the queue head, qsync[1 + sub] counts the finished forward chains of sub: a
  // backward task waits for them (release/acquire through global memory; the forward tasks
  // were all dequeued earlier, so they are running or done).
  const int ntask = PERSIST ? 4 * nsub_all : 1;
  auto decode = [&](int tk, int& ph, int& sub, int& chain) {
    if (!PERSIST) {
      const int cid = blockIdx.x / C;
      ph = phase_arg, sub = cid >> 1, chain = cid & 1;
      return;
    }
    ph = tk >= 2 * nsub_all ? 1 : 0;
    const int c2 = tk - ph * 2 * nsub_all;
    sub = c2 >> 1, chain = c2 & 1;
  };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + 8;
  const int dbg = g_solve_dbg;
  uint64_t* red_bar = empty + 8;  // [2]: partial sums for my rows have arrived (line parity)
  uint64_t* x_bar = red_bar + 2;  // [2]: the other CTAs' x of the line have arrived
  uint64_t* tbar = x_bar + 2;     // [4] PERSIST: task id k published by the producer
  uint64_t* tfree = tbar + 4;     // [4] PERSIST: the consumers have read task slot k
  int* task_ids = reinterpret_cast<int*>(smem_raw + 240);  // [4]
  double* stage0 = reinterpret_cast<double*>(smem_raw + kSolveHdr);
  // column-partial slots: one per compute warp, or 8 (two-round reduction) for wide lines
  // where the 7 kd doubles buy ring capacity (must match solve_plan)
  constexpr int ncs = MAXM >= 20 ? kCS : kCW;
  double* colpart = stage0 + static_cast<size_t>(stages) * cap;  // ncs x kd_max
  double* wv = colpart + static_cast<size_t>(ncs) * kd_max;      // kd_max
  double* yrow = wv + kd_max;                                    // kd_max (own rows)
  double* xbuf = yrow + kd_max;                                  // 2 x kd_max (line parity)
  double* red = xbuf + 2 * kd_max;                               // 2 x C x kd_max slots
  double* dcorr = red + 2 * static_cast<size_t>(C) * kd_max;     // kd_max: D_ii w_i
  if (tid == 0) {
    for (int q = 0; q < stages; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kCW);
    }
    // point-to-point line exchange between the cluster's CTAs (no cluster-wide barriers):
    // CTA o receives partial sums from CTAs o+1..C-1 and x from all others
    for (int q = 0; q < 2; ++q) {
      mbar_init(&red_bar[q], 1);  // armed with the expected bytes by this CTA each use
      mbar_init(&x_bar[q], 1);
    }
    for (int q = 0; q < 4; ++q) {
      mbar_init(&tbar[q], 1);
      mbar_init(&tfree[q], 1);
    }
    fence_barrier_init();
  }
  int* rlos = reinterpret_cast<int*>(smem_raw + 256);  // row_lo(c) for c = 0..C (C > 1)
  if (C > 1 && tid <= C) rlos[tid] = row_lo(tid, C, subs[(blockIdx.x / C) >> 1].kd, rc);
  // Everything after the header starts at zero: x of "line -1" (xbuf), and the slots the row
  // loop reads without a mask — the operand pair past an odd line width (wv[kd], multiplied by
  // a zeroed entry: a NaN pattern left in shared memory by an earlier kernel made 0 * NaN and
  // stalled the CG on NaN residuals, seen with kd 447 on 4-CTA clusters), the ring stages.
  {
    const int nz = stages * cap + (ncs + 5 + 2 * C) * kd_max;  // colpart wv yrow xbuf red dcorr
    for (int j = tid; j < nz; j += kST) stage0[j] = 0.0;
  }
  if (C > 1) cl_sync(); else __syncthreads();  // barriers initialised cluster-wide

  // ------------------------------------------------------------------ producer warp
  // Row chunks of a line: the CTA's rows [rlo, rhi) cut into runs whose packed rows fit one
  // ring stage (chunk_end), computed on the fly by the producer and the consumers alike.
  if (warp == kCW) {
    int q = 0;  // ring slots used so far (continues across tasks)
    int line_of[8];  // line of the chunk last placed in each stage
#pragma unroll
    for (int k = 0; k < 8; ++k) line_of[k] = -1;
    for (int kk = 0;; ++kk) {
      int tk = kk;
      if (PERSIST) {  // dequeue and publish the next task to the compute warps
        if (lane == 0) {
          if (kk >= 4) mbar_wait(&tfree[kk & 3], ((kk >> 2) - 1) & 1);
          tk = atomicAdd(qsync, 1);
          task_ids[kk & 3] = tk;
          mbar_arrive(&tbar[kk & 3]);
        }
        tk = __shfl_sync(0xffffffffu, tk, 0);
      }
      if (tk >= ntask) break;
      int phase, sub, chain;
      decode(tk, phase, sub, chain);
      const SubInfo s = subs[sub];
      const int kd = s.kd, nl = chain_len(phase, chain, s);
      const int rlo = row_lo(crank, C, kd, rc), rhi = row_lo(crank + 1, C, kd, rc);
      if (nl == 0 || rlo >= rhi) continue;
      const double* F = fac + s.fac_off;
      int t_i = 0, r_a = rlo;  // next chunk: line step t_i, first row r_a
      const int n_first = chunk_end(rlo, rhi, cap) - rlo;  // rows of a line's first chunk
      int n_prev = n_first;
      // place chunks in FIFO order; with C > 1 only while they belong to lines <= t_sync + 1
      // and the stage's previous occupant belongs to a line the consumers finish before
      // barrier t_sync (the gating is moot for one CTA per chain)
      const int t_sync = 1 << 30;
      while (t_i < nl) {
        if (C > 1 && t_i > t_sync + 1) break;
        const int st = q % stages;
        int prev_line = -1;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k == st) prev_line = line_of[k];
        if (C > 1 && prev_line > t_sync) break;
        if (q >= stages) mbar_wait(&empty[st], ((q / stages) - 1) & 1);
        const int l = chain_line(phase, chain, s, t_i);
        const int r_b = chunk_end_from(r_a, rhi, cap, n_prev);
        const int o0 = prow_off32(r_a), o1 = prow_off32(r_b);
        if (lane == 0) {
          if (dbg & 4) {
            mbar_arrive(&full[st]);
          } else {
            fence_proxy_async();
            mbar_expect_tx(&full[st], static_cast<uint32_t>((o1 - o0) * sizeof(double)));
            bulk_g2s(stage0 + static_cast<size_t>(st) * cap, F + static_cast<long long>(l) * s.line_sz + o0,
                     static_cast<uint32_t>((o1 - o0) * sizeof(double)), &full[st]);
          }
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k == st) line_of[k] = t_i;
        ++q;
        n_prev = r_b - r_a;
        r_a = r_b;
        if (r_a == rhi) r_a = rlo, n_prev = n_first, ++t_i;
      }
    }
    return;
  }

  // ------------------------------------------------------------------ compute warps
  int c_seq = 0;  // ring slots consumed (continues across tasks)
  PROF_DECL
  for (int kk = 0;; ++kk) {
  int tk = kk;
  if (PERSIST) {
    mbar_wait(&tbar[kk & 3], (kk >> 2) & 1);
    tk = task_ids[kk & 3];
    compute_bar();  // every compute thread has read the slot
    if (tid == 0) mbar_arrive(&tfree[kk & 3]);
  }
  if (tk >= ntask) break;
  int phase, sub, chain;
  decode(tk, phase, sub, chain);
  const SubInfo s = subs[sub];
  const int kd = s.kd, L = s.L, m = s.m;
  const int nl = chain_len(phase, chain, s);
  if (nl == 0) continue;  // cluster-uniform
  const int rlo = row_lo(crank, C, kd, rc), rhi = row_lo(crank + 1, C, kd, rc);
  const int n_first = rlo < rhi ? chunk_end(rlo, rhi, cap) - rlo : 0;
  double* yl = ylocal + s.vec_off;
  double* zl = zlocal + s.vec_off;
  const double* rl = rlocal ? rlocal + s.vec_off : nullptr;  // per-subdomain rhs (RAS mode)
  if (PERSIST && kk > 0) {  // x of "line -1" is zero for every task (one CTA per chain)
    for (int j = tid; j < 2 * kd_max; j += kCT) xbuf[j] = 0.0;
    compute_bar();
  }
  if (PERSIST && phase == 1) {  // both forward chains of this subdomain are done
    if (tid == 0) {
      const int need = (s.m > 0 ? 1 : 0) + (s.L - 1 - s.m > 0 ? 1 : 0);
      wait_forward_done(qsync + 1 + sub, need);
    }
    compute_bar();
  }
  // operand of line step t, prefetched into registers one step ahead. Forward:
  // w = r_l - b_prev o y_prev; backward middle: w = r_m - b_m y_{m-1} - b_{m+1} y_{m+1};
  // backward chain: w = b_next o x_next and x_l = y_l - Dinv_l w.
  constexpr int PS = 32 * MAXM > kCT ? 2 : 1;  // j = tid + kCT*q, kd <= PS*kCT
  double pf_r[PS], pf_b[PS], pf_y[PS];
  auto prefetch = [&](int t) {
#pragma unroll
    for (int q = 0; q < PS; ++q) {
      pf_r[q] = pf_b[q] = pf_y[q] = 0.0;
      if (t >= nl) continue;
      const int l = chain_line(phase, chain, s, t);
      const int j = tid + kCT * q;
      if (j < kd) {
        if (phase == 0) {
          pf_r[q] = rl ? rl[static_cast<long long>(l) * kd + j] : r[gidx(s, l, j, W, nc)];
          if (t > 0) pf_b[q] = bcoef(s, coef, N, W, nc, chain == 0 ? l : l + 1, j);
        } else if (t == 0) {  // middle line: both neighbours from the forward sweep
          double w = rl ? rl[static_cast<long long>(l) * kd + j] : r[gidx(s, l, j, W, nc)];
          if (m > 0) w -= bcoef(s, coef, N, W, nc, m, j) * __ldcg(yl + static_cast<long long>(m - 1) * kd + j);
          if (m < L - 1)
            w -= bcoef(s, coef, N, W, nc, m + 1, j) * __ldcg(yl + static_cast<long long>(m + 1) * kd + j);
          pf_r[q] = w;
        } else {
          pf_b[q] = bcoef(s, coef, N, W, nc, chain == 0 ? l + 1 : l, j);
        }
      }
      const int jo = rlo + tid + kCT * q;  // owned row
      if (phase == 1 && t > 0 && jo < rhi) pf_y[q] = __ldcg(yl + static_cast<long long>(l) * kd + jo);
    }
  };
  prefetch(0);
  for (int t = 0; t < nl; ++t) {
    const int l = chain_line(phase, chain, s, t);
    const int par = t & 1;
    const bool subtract = phase == 1 && t > 0;  // x_l = y_l - Dinv_l w
    const double* xprev = xbuf + (par ^ 1) * kd_max;  // x of line t-1 (zeros at t = 0)
    if (C > 1 && t > 0 && !(dbg & 2)) mbar_wait_cluster(&x_bar[par ^ 1], ((t - 1) >> 1) & 1);
    if (C > 1 && tid == 0 && !(dbg & 2)) {
      // this line's incoming bytes: partial sums for my rows from CTAs crank+1..C-1, and x
      // of every row I do not own
      const uint32_t mine = static_cast<uint32_t>(rhi - rlo);
      if (crank < C - 1) mbar_arrive_expect(&red_bar[par], 8u * mine * (C - 1 - crank));
      mbar_arrive_expect(&x_bar[par], 8u * (static_cast<uint32_t>(kd) - mine));
    }
    double cur_y[PS];
#pragma unroll
    for (int q = 0; q < PS; ++q) {
      const int j = tid + kCT * q;
      if (j < kd)
        wv[j] = (phase == 0) ? pf_r[q] - pf_b[q] * xprev[j]
                             : (t == 0 ? pf_r[q] : pf_b[q] * xprev[j]);
      cur_y[q] = pf_y[q];
    }
    if (!(dbg & 16)) prefetch(t + 1);
    compute_bar();
    PROF_MARK(0);
    // lane owns the column pairs j = 64 mm + 2 lane + {0, 1}: operand in registers for the
    // whole line, rows read as 16-byte pairs (row starts are 16-byte aligned)
    constexpr int M2 = (MAXM + 1) / 2;
#ifndef FFB_RB7
#define FFB_RB7 2
#endif
    // rows per batch and operand placement within the 128-register budget
    // (two rows per batch on lines wider than 256 unknowns: the column partials stay in
    // registers and the row loop issues fewer dead predicated loads; measured c3 4.61 -> 4.27
    // ms, c4 18.7 -> 17.7, c5 8.2 -> 5.3 per application)
    constexpr int RB = M2 <= 4 ? 8 : (M2 <= 7 ? FFB_RB7 : (M2 <= 10 ? 4 : 2));
    constexpr bool WREG = M2 <= 4 || (M2 <= 7 && RB == 4);
    double2 wreg[M2], cacc[M2];
#pragma unroll
    for (int mm = 0; mm < M2; ++mm) {
      const int j = 64 * mm + 2 * lane;
      wreg[mm].x = j < kd ? wv[j] : 0.0;
      wreg[mm].y = j + 1 < kd ? wv[j + 1] : 0.0;
      cacc[mm].x = cacc[mm].y = 0.0;
    }
    for (int r0 = rlo, r1 = rlo, n_prev = n_first; r0 < rhi; n_prev = r1 - r0, r0 = r1) {
      r1 = chunk_end_from(r0, rhi, cap, n_prev);
      const int st = c_seq % stages;
      mbar_wait(&full[st], (c_seq / stages) & 1);
      PROF_MARK(1);
      const double* Sb = stage0 + static_cast<size_t>(st) * cap - prow_off32(r0);
      // batches of R rows per warp (rows i0 + k kCW): R independent accumulation chains and
      // one transpose reduction per batch. Row i is read as its padded pairs (the pad is 0):
      // every lane loads unconditionally and masks by selection, so the R loads of a column
      // step issue back to back; the diagonal enters both the row dot and the column sums
      // and is taken out once through dcorr.
      const uint32_t sbase = smem_u32(Sb) + 16u * lane;
      for (int i0 = r0 + warp; i0 < r1 && !(dbg & 1); i0 += RB * kCW) {
        uint32_t ra[RB];
        double wi[RB], racc[RB];
        int np[RB];
        int npmax = 0;
#pragma unroll
        for (int k = 0; k < RB; ++k) {
          const int i = i0 + k * kCW;
          const bool ok = i < r1;
          ra[k] = sbase + 8u * static_cast<uint32_t>(prow_off32(ok ? i : r0));
          wi[k] = ok ? wv[i] : 0.0;
          np[k] = ok ? (i + 2) >> 1 : 0;  // pairs in the padded row
          npmax = max(npmax, np[k]);
          racc[k] = 0.0;
        }
#pragma unroll
        for (int mm = 0; mm < M2; ++mm) {
          if (32 * mm >= npmax) break;
          const int pidx = 32 * mm + lane;
          double2 v[RB];
#pragma unroll
          for (int k = 0; k < RB; ++k) v[k] = lds_f64x2(ra[k] + 512u * mm);
          const double2 w2 = WREG ? wreg[mm] : *reinterpret_cast<const double2*>(wv + 64 * mm + 2 * lane);
#pragma unroll
          for (int k = 0; k < RB; ++k) {
            const bool in = pidx < np[k];
            v[k].x = in ? v[k].x : 0.0;
            v[k].y = in ? v[k].y : 0.0;
            racc[k] = fma(v[k].x, w2.x, racc[k]);
            racc[k] = fma(v[k].y, w2.y, racc[k]);
          }
          double cx = cacc[mm].x, cy = cacc[mm].y, dx = 0.0, dy = 0.0;
#pragma unroll
          for (int k = 0; k < RB; k += 2) {
            cx = fma(v[k].x, wi[k], cx);
            cy = fma(v[k].y, wi[k], cy);
            dx = fma(v[k + 1].x, wi[k + 1], dx);
            dy = fma(v[k + 1].y, wi[k + 1], dy);
          }
          cacc[mm].x = cx + dx;
          cacc[mm].y = cy + dy;
        }
        if (lane < RB) {  // D_ii w_i of row k = lane
          const int i = i0 + lane * kCW;
          if (i < r1) dcorr[i] = Sb[prow_off32(i) + i] * wv[i];
        }
        // transpose reduction: lane ends with the total of row k(lane)
        const double tot = transpose_reduce<RB>(racc, lane);
        const int kk = lane / (32 / RB);
        const int i = i0 + kk * kCW;
        if ((lane & (32 / RB - 1)) == 0 && i < r1) yrow[i] = tot;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage
      PROF_MARK(2);
      ++c_seq;
    }
    // column partials of the 15 warps: one slot per warp (ncs = 15), or, for wide lines,
    // through 8 slots (fixed order): warps 8..14 hand theirs to warps 0..6, then warps 0..7
    // publish (each reuses the slot it just read) — 7 kd doubles more for the stage ring
    if constexpr (ncs == kCW) {
#pragma unroll
      for (int mm = 0; mm < M2; ++mm) {
        const int j = 64 * mm + 2 * lane;
        if (j < rhi) colpart[warp * kd_max + j] = cacc[mm].x;
        if (j + 1 < rhi) colpart[warp * kd_max + j + 1] = cacc[mm].y;
      }
    } else {
      if (warp >= kCS) {
#pragma unroll
        for (int mm = 0; mm < M2; ++mm) {
          const int j = 64 * mm + 2 * lane;
          if (j < rhi) colpart[(warp - kCS) * kd_max + j] = cacc[mm].x;
          if (j + 1 < rhi) colpart[(warp - kCS) * kd_max + j + 1] = cacc[mm].y;
        }
      }
      compute_bar();
      if (warp < kCS) {
#pragma unroll
        for (int mm = 0; mm < M2; ++mm) {
          const int j = 64 * mm + 2 * lane;
          if (warp + kCS < kCW) {
            if (j < rhi) cacc[mm].x += colpart[warp * kd_max + j];
            if (j + 1 < rhi) cacc[mm].y += colpart[warp * kd_max + j + 1];
          }
          if (j < rhi) colpart[warp * kd_max + j] = cacc[mm].x;
          if (j + 1 < rhi) colpart[warp * kd_max + j + 1] = cacc[mm].y;
        }
      }
    }
    compute_bar();
    PROF_MARK(3);
    // column partials of this CTA (+ its own row dots), reduced in a fixed slot order and
    // scattered to the CTA that owns each row
    int owner = 0;
    for (int j = tid; j < rhi && !(dbg & 8); j += kCT) {
      double tv = (j >= rlo) ? yrow[j] - dcorr[j] : 0.0;
      if constexpr (ncs == kCW) {
#pragma unroll 5
        for (int w = 0; w < kCW; ++w) tv += colpart[w * kd_max + j];
      } else {
#pragma unroll
        for (int w = 0; w < kCS; ++w) tv += colpart[w * kd_max + j];
      }
      while (owner + 1 < C && rlos[owner + 1] <= j) ++owner;
      double* slot = red + static_cast<size_t>(par * C + crank) * kd_max;
      if (owner == crank || (dbg & 2))
        slot[j] = tv;
      else
        st_async_remote(slot + j, tv, &red_bar[par], static_cast<unsigned>(owner));
    }
    compute_bar();
    if (C > 1 && !(dbg & 2) && crank < C - 1) mbar_wait_cluster(&red_bar[par], (t >> 1) & 1);
    PROF_MARK(4);
#pragma unroll
    for (int q = 0; q < PS; ++q) {
      const int j = rlo + tid + kCT * q;
      if (j >= rhi || (dbg & 8)) continue;
      double tv = 0.0;
      for (int c = crank; c < C; ++c) tv += red[static_cast<size_t>(par * C + c) * kd_max + j];
      const long long k = static_cast<long long>(l) * kd + j;
      double v;
      if (!subtract) {
        v = tv;
        if (phase == 0) {
          yl[k] = v;
          if (L == 1) zl[k] = v;
        } else if (chain == mid_writer(s)) {
          zl[k] = v;  // middle line, written once
        }
      } else {
        v = cur_y[q] - tv;
        zl[k] = v;
      }
      double* xo = xbuf + par * kd_max;
      xo[j] = v;
      for (int c = 0; c < C && !(dbg & 2); ++c)
        if (c != crank) st_async_remote(xo + j, v, &x_bar[par], static_cast<unsigned>(c));
    }
    compute_bar();
    PROF_MARK(5);
  }
  // every CTA receives x from all others at every line: waiting for the last line's
  // arrivals means no remote store into this CTA's shared memory is still in flight
  if (C > 1 && !(dbg & 2)) mbar_wait_cluster(&x_bar[(nl - 1) & 1], ((nl - 1) >> 1) & 1);
  if (C > 1 && (dbg & 2)) cl_sync();
  if (PERSIST && phase == 0) {  // publish this forward chain (y of its lines) to the queue
    __threadfence();
    compute_bar();
    if (tid == 0) atomicAdd(qsync + 1 + sub, 1);
  }
  }  // tasks
  PROF_FLUSH(16);
}

// ----------------------------------------------------------------- K5b, row-group tiles
// The ring kernel for one CTA per chain (c3, c4: lines of up to kRtMaxKd unknowns) with the
// arithmetic cut into tiles. The packed rows stream through the two-stage ring in runs of
// whole 16-row groups, and the lower triangle is processed as 16x32 tiles (group g, column
// block J <= g/2), tile k of a line going to compute warp k mod 15. A lane holds 4 rows x 2
// column pairs of a tile — 8 LDS.128 and 32 DFMA — and a 7-shuffle reduction gives the
// tile's 16 row partials (T w) and 32 column partials (T^T w, the upper half the packed rows
// leave out). Off-diagonal tiles need no masking at all. Each warp accumulates into its own
// kd slot in a fixed tile order; the line's product is the 15 slots summed in warp order
// (deterministic). Versus the row-batch loop of k_line_solve (every element masked, both
// partials carried per column pair) this issues ~3x fewer instructions per element.
constexpr int kRtMaxKd = 448;
static_assert(kRtMaxKd <= kCT, "one operand element per compute thread");

__device__ __forceinline__ int rt_first_tile(int g) {  // tiles of groups 0..g-1
  const int h = g >> 1;
  return (g & 1) ? (h + 1) * (h + 1) : h * (h + 1);
}
// end group of the ring chunk that starts at group g0: whole 16-row groups while they fit
__device__ __forceinline__ int rt_chunk_end(int g0, int ng, int kd, int cap) {
  const int base = prow_off32(16 * g0);
  int g1 = g0 + 1;
  while (g1 < ng && prow_off32(min(16 * (g1 + 1), kd)) - base <= cap) ++g1;
  return g1;
}

// first row group of CTA q of a C-CTA cluster: the line's ng groups cut into C runs of about
// equal tile counts (= equal bytes: a tile is 512 entries)
__device__ __forceinline__ int rt_group_lo(int q, int C, int ng) {
  if (q <= 0) return 0;
  if (q >= C) return ng;
  const int target = (rt_first_tile(ng) * q + C / 2) / C;
  int g = 0;
  while (g < ng && rt_first_tile(g) < target) ++g;
  return g;
}

// The chunk and tile schedule of a line depends only on (kd, cap): the compute warps keep it
// in two small tables in the shared-memory header, rebuilt when a task's kd differs from the
// previous one's (per chunk and per tile the schedule arithmetic cost ~100 and ~25
// instructions on every warp — 27% of the kernel's instructions, ncu r3c — against one
// shared-memory load now).
//   chunk c: {packed offset of its first row, T0 | T1 << 8 | (T0 mod kCW) << 16}
//   tile tau: group | column block << 5 | kind << 9 (rt_tile's KIND, 0..3)
constexpr int kRtTabChunks = 256;  // byte offset of the chunk table in the header (28 x 8 B)
constexpr int kRtTabTiles = 480;   // byte offset of the tile table (<= 210 x 2 B)
constexpr int kRtTabCount = 232;   // byte offset of the chunk count
constexpr int kRtXbar = 192;       // byte offset of the two line-exchange mbarriers (clusters)
static_assert(kRtTabChunks + 8 * ((kRtMaxKd + 15) / 16) <= kRtTabTiles, "chunk table");
static_assert(kRtTabTiles + 2 * (((kRtMaxKd + 15) / 16 + 1) / 2) * (((kRtMaxKd + 15) / 16) / 2 + 1) <=
                  kSolveHdr, "tile table");

// tile (rows R0..R0+15, columns C0..C0+31) of the chunk staged at shared address sb whose
// first row starts at packed offset soff; adds T w into yacc[rows] and T^T w (strictly
// lower part) into yacc[columns].
//   KIND 0: a full off-diagonal tile, nothing masked.
//   KIND 1: an off-diagonal tile of the line's last, partial row group.
//   KIND 2: the diagonal tile of an even group (R0 == C0): columns C0..C0+15 triangular
//           (j <= i), columns C0+16.. above the diagonal (not loaded).
//   KIND 3: the diagonal tile of an odd group (R0 == C0 + 16): columns C0..C0+15 full,
//           columns C0+16.. triangular.
// Rows past the line (KIND != 0): their loads are redirected to row 0 of the chunk (finite
// data), their operand is zero (so they add +-0 to the column sums) and their row sums are
// dropped. The triangular half's masks depend on the lane only through d = 4 rg - 2 cg:
// entry (a, c) is on or below the diagonal iff d + a - c >= 0. Operand slots past the line
// hold finite values (zero, or an earlier task's), which the zeroed entries cancel.
template <int KIND, class FT>
__device__ __forceinline__ void rt_tile(uint32_t sb, int soff, int R0, int C0, int kd,
                                        const double* __restrict__ wv, double* __restrict__ yacc,
                                        int lane) {
  constexpr bool DIAG = KIND >= 2;
  constexpr bool HALF1 = KIND != 2;  // columns C0+16.. hold entries of the lower triangle
  constexpr int TH = KIND == 2 ? 0 : 1;  // the triangular half of a diagonal tile
  const int rg = lane >> 3, cg = lane & 7;
  const int i0 = R0 + 4 * rg;  // even: rows i0, i0+1 have length i0+2, rows i0+2, i0+3 i0+4
  const int j0 = C0 + 2 * cg;
  int o[4];
  o[0] = prow_off32(i0) - soff + j0;
  o[1] = o[0] + i0 + 2;
  o[2] = o[1] + i0 + 2;
  o[3] = o[2] + i0 + 4;
  double2 t[4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int oa = (KIND != 0 && i0 + a >= kd) ? j0 : o[a];
    const uint32_t ad = sb + static_cast<uint32_t>(sizeof(FT)) * static_cast<uint32_t>(oa);
    t[a][0] = lds_pair<FT>(ad);
    t[a][1] = HALF1 ? lds_pair<FT>(ad + 16u * static_cast<uint32_t>(sizeof(FT))) : make_double2(0.0, 0.0);
  }
  const double2 wc0 = *reinterpret_cast<const double2*>(wv + j0);
  const double2 wc1 = HALF1 ? *reinterpret_cast<const double2*>(wv + j0 + 16) : make_double2(0.0, 0.0);
  const double2 wr01 = *reinterpret_cast<const double2*>(wv + i0);
  const double2 wr23 = *reinterpret_cast<const double2*>(wv + i0 + 2);
  double wr[4] = {wr01.x, wr01.y, wr23.x, wr23.y};
  double tc[4][4];  // column-part copy (a diagonal tile: without the diagonal)
  double tr[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    tr[a][0] = t[a][0].x, tr[a][1] = t[a][0].y, tr[a][2] = t[a][1].x, tr[a][3] = t[a][1].y;
#pragma unroll
    for (int c = 0; c < 4; ++c) tc[a][c] = tr[a][c];
  }
  if (KIND != 0) {
#pragma unroll
    for (int a = 0; a < 4; ++a) wr[a] = i0 + a < kd ? wr[a] : 0.0;
  }
  if (DIAG) {
    const int d = 4 * rg - 2 * cg;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tc[a][2 * TH + c] = d + a - c > 0 ? tr[a][2 * TH + c] : 0.0;
        tr[a][2 * TH + c] = d + a - c >= 0 ? tr[a][2 * TH + c] : 0.0;
      }
  }
  double rp[4], cp[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double v = tr[a][0] * wc0.x;
    v = fma(tr[a][1], wc0.y, v);
    if (HALF1) {
      v = fma(tr[a][2], wc1.x, v);
      v = fma(tr[a][3], wc1.y, v);
    }
    rp[a] = v;
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (!HALF1 && c >= 2) {
      cp[c] = 0.0;
      continue;
    }
    double v = tc[0][c] * wr[0];
    v = fma(tc[1][c], wr[1], v);
    v = fma(tc[2][c], wr[2], v);
    cp[c] = fma(tc[3][c], wr[3], v);
  }
  // rows: sum over the 8 lanes of the row group -> lanes 2k, 2k+1 hold row i0 + k
  const bool b2 = lane & 4, b1 = lane & 2;
  double k0 = (b2 ? rp[2] : rp[0]) + __shfl_xor_sync(0xffffffffu, b2 ? rp[0] : rp[2], 4);
  double k1 = (b2 ? rp[3] : rp[1]) + __shfl_xor_sync(0xffffffffu, b2 ? rp[1] : rp[3], 4);
  double u = (b1 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, b1 ? k0 : k1, 2);
  u += __shfl_xor_sync(0xffffffffu, u, 1);
  // columns: sum over the 4 row groups -> lane holds column j0 + 16 h + e
  const bool h = lane & 16, e = lane & 8;
  double q0 = (h ? cp[2] : cp[0]) + __shfl_xor_sync(0xffffffffu, h ? cp[0] : cp[2], 16);
  double q1 = (h ? cp[3] : cp[1]) + __shfl_xor_sync(0xffffffffu, h ? cp[1] : cp[3], 16);
  const double v = (e ? q1 : q0) + __shfl_xor_sync(0xffffffffu, e ? q0 : q1, 8);
  const int row = i0 + (cg >> 1);
  const int col = j0 + (h ? 16 : 0) + (e ? 1 : 0);
  if (!(lane & 1) && (KIND == 0 || row < kd)) yacc[row] += u;
  // a diagonal tile's rows and columns overlap: rows first, then columns
  if (DIAG) __syncwarp();
  if (!DIAG || col < kd) yacc[col] += v;
  __syncwarp();
}

// Clusters (C = 2 or 4 CTAs per chain, when a rank has fewer chains than SMs — multi-GPU
// shards): CTA q streams and multiplies only its run of row groups (rt_group_lo: equal bytes),
// so each SM ingests 1/C of the line; at the end of a line every CTA sends its kd partial sums
// to the others (st.async into their shared memory, one transaction barrier per line parity)
// and all of them add the C partials in CTA order, so every CTA holds the same x for the next
// line's operand; CTA 0 writes the results. One launch per sweep (no task queue).
// FT = float streams the single-precision copy of the line inverses (factor_to_f32: opt-in,
// half the bytes per application; the products and sums stay in double): fac then points at
// that copy, a line of it starts at fac32_off + l * ((line_sz + 3) & ~3) floats, and `cap`
// counts floats (twice the doubles the same stage holds).
template <bool PERSIST, class FT>
__global__ void __launch_bounds__(kST, 1)
    k_line_solve_rt(const SubInfo* __restrict__ subs, const FT* __restrict__ fac,
                    const double* __restrict__ coef, size_t N, const double* __restrict__ r,
                    double* __restrict__ ylocal, double* __restrict__ zlocal, int W, int nc,
                    int cap, int kd_max, int phase_arg, const int* __restrict__ flags,
                    const double* __restrict__ rlocal, int* __restrict__ qsync, int nsub_all) {
  if (flags && (flags[0] | flags[1])) return;  // PCG converged or failed (grid-uniform)
  constexpr int stages = 2;
  const int C = PERSIST ? 1 : static_cast<int>(cl_size());
  const int crank = PERSIST ? 0 : static_cast<int>(cl_rank());
  // tasks as in k_line_solve: one chain per cluster, or (PERSIST) the dynamic queue of both sweeps
  const int ntask = PERSIST ? 4 * nsub_all : 1;
  auto decode = [&](int tk, int& ph, int& sub, int& chain) {
    if (!PERSIST) {
      const int cid = static_cast<int>(blockIdx.x) / C;
      ph = phase_arg, sub = cid >> 1, chain = cid & 1;
      return;
    }
    ph = tk >= 2 * nsub_all ? 1 : 0;
    const int c2 = tk - ph * 2 * nsub_all;
    sub = c2 >> 1, chain = c2 & 1;
  };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + 8;
  uint64_t* tbar = empty + 8;  // [4] PERSIST: task id k published by the producer
  uint64_t* tfree = tbar + 4;  // [4] PERSIST: the consumers have read task slot k
  int* task_ids = reinterpret_cast<int*>(smem_raw + 240);  // [4]
  constexpr int kEls = 8 / static_cast<int>(sizeof(FT));  // factor entries per double of stage
  const int cap_d = cap / kEls;                           // a stage in doubles
  double* stage0 = reinterpret_cast<double*>(smem_raw + kSolveHdr);
  double* yacc = stage0 + static_cast<size_t>(stages) * cap_d;  // kCW x kd_max
  double* wv = yacc + static_cast<size_t>(kCW) * kd_max;         // kd_max
  double* xbuf = wv + kd_max;                                    // 2 x kd_max (line parity)
  double* xch = xbuf + 2 * kd_max;  // C > 1: 2 x C x kd_max partial sums (line parity, sender)
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem_raw + kRtXbar);  // [2] (line parity)
  int2* chunk_tab = reinterpret_cast<int2*>(smem_raw + kRtTabChunks);
  unsigned short* tile_tab = reinterpret_cast<unsigned short*>(smem_raw + kRtTabTiles);
  int* chunk_cnt = reinterpret_cast<int*>(smem_raw + kRtTabCount);
  if (tid == 0) {
    for (int q = 0; q < stages; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kCW);
    }
    for (int q = 0; q < 4; ++q) {
      mbar_init(&tbar[q], 1);
      mbar_init(&tfree[q], 1);
    }
    mbar_init(&xbar[0], 1);  // armed with the expected bytes by this CTA at every line
    mbar_init(&xbar[1], 1);
    fence_barrier_init();
  }
  // yacc, wv, xbuf start at zero — and so do the ring stages: a masked tile row reads a finite
  // stand-in from its stage (rt_tile), which must not be a NaN pattern of never-written memory
  for (int j = tid; j < stages * cap_d + (kCW + 3) * kd_max; j += kST) stage0[j] = 0.0;
  if (C > 1) cl_sync(); else __syncthreads();  // barriers initialised cluster-wide

  // ------------------------------------------------------------------ producer warp
  if (warp == kCW) {
    int q = 0;  // ring slots used so far (continues across tasks)
    for (int kk = 0;; ++kk) {
      int tk = kk;
      if (PERSIST) {
        if (lane == 0) {
          if (kk >= 4) mbar_wait(&tfree[kk & 3], ((kk >> 2) - 1) & 1);
          tk = atomicAdd(qsync, 1);
          task_ids[kk & 3] = tk;
          mbar_arrive(&tbar[kk & 3]);
        }
        tk = __shfl_sync(0xffffffffu, tk, 0);
      }
      if (tk >= ntask) break;
      int phase, sub, chain;
      decode(tk, phase, sub, chain);
      const SubInfo s = subs[sub];
      const int kd = s.kd, nl = chain_len(phase, chain, s), ng = (kd + 15) >> 4;
      const int glo = rt_group_lo(crank, C, ng), ghi = rt_group_lo(crank + 1, C, ng);
      const bool f32 = sizeof(FT) == 4;
      const FT* F = fac + (f32 ? s.fac32_off : s.fac_off);
      const long long lstride = f32 ? ((s.line_sz + 3) & ~3LL) : s.line_sz;
      for (int t = 0; t < nl; ++t) {
        const int l = chain_line(phase, chain, s, t);
        for (int g0 = glo, g1; g0 < ghi; g0 = g1, ++q) {
          g1 = rt_chunk_end(g0, ghi, kd, cap);
          const int st = q % stages;
          if (q >= stages) mbar_wait(&empty[st], ((q / stages) - 1) & 1);
          const int o0 = prow_off32(16 * g0), o1 = prow_off32(min(16 * g1, kd));
          // bulk copies move multiples of 16 bytes: a float chunk's tail rounds up into the
          // line's padding
          const uint32_t bytes = (static_cast<uint32_t>(o1 - o0) * static_cast<uint32_t>(sizeof(FT)) + 15u) & ~15u;
          if (lane == 0) {
            fence_proxy_async();
            mbar_expect_tx(&full[st], bytes);
            bulk_g2s(stage0 + static_cast<size_t>(st) * cap_d, F + static_cast<long long>(l) * lstride + o0,
                     bytes, &full[st]);
          }
          __syncwarp();
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ compute warps
  int c_seq = 0;    // ring slots consumed (continues across tasks)
  int tab_kd = -1;  // line width the schedule tables hold
  const uint32_t sb0 = smem_u32(stage0);
  for (int kk = 0;; ++kk) {
    int tk = kk;
    if (PERSIST) {
      mbar_wait(&tbar[kk & 3], (kk >> 2) & 1);
      tk = task_ids[kk & 3];
      compute_bar();  // every compute thread has read the slot
      if (tid == 0) mbar_arrive(&tfree[kk & 3]);
    }
    if (tk >= ntask) break;
    int phase, sub, chain;
    decode(tk, phase, sub, chain);
    const SubInfo s = subs[sub];
    const int kd = s.kd, L = s.L, m = s.m, ng = (kd + 15) >> 4;
    const int nl = chain_len(phase, chain, s);
    if (nl == 0) continue;
    double* yl = ylocal + s.vec_off;
    double* zl = zlocal + s.vec_off;
    const double* rl = rlocal ? rlocal + s.vec_off : nullptr;  // per-subdomain rhs (RAS mode)
    if (kd != tab_kd) {  // (re)build the schedule tables; every compute warp is past the last line
      tab_kd = kd;
      const int glo = rt_group_lo(crank, C, ng), ghi = rt_group_lo(crank + 1, C, ng);
      const int T_lo = rt_first_tile(glo), T_hi = rt_first_tile(ghi);
      for (int tau = T_lo + tid; tau < T_hi; tau += kCT) {
        int g = glo;
        while (rt_first_tile(g + 1) <= tau) ++g;
        const int J = tau - rt_first_tile(g), I = g >> 1;
        const int kind = J == I ? 2 + (g & 1) : (16 * (g + 1) > kd ? 1 : 0);
        tile_tab[tau] = static_cast<unsigned short>(g | (J << 5) | (kind << 9));
      }
      if (tid == 0) {
        int c = 0;
        for (int g0 = glo, g1; g0 < ghi; g0 = g1, ++c) {
          g1 = rt_chunk_end(g0, ghi, kd, cap);
          const int T0 = rt_first_tile(g0), T1 = rt_first_tile(g1);
          chunk_tab[c] = make_int2(prow_off32(16 * g0), T0 | (T1 << 8) | (((T0 - T_lo) % kCW) << 16));
        }
        *chunk_cnt = c;
      }
      compute_bar();
    }
    const int nchunk = *chunk_cnt;
    // thread tid owns unknown j = tid of every line: its vertex / component, the global index
    // of its residual entry and of its slow-axis coupling as base + line * stride
    long long g_base = 0, b_base = 0;
    int g_stride = 0, b_stride = 0;
    if (tid < kd) {
      const int a = tid / nc, cc = tid - a * nc;
      const long long v0 = static_cast<long long>(s.fy0 + (s.xfast ? 0 : a)) * W + s.fx0 + (s.xfast ? a : 0);
      g_base = v0 * nc + cc;
      g_stride = s.xfast ? W * nc : nc;
      b_base = static_cast<long long>((s.xfast ? 8 : 6) + (cc < 2 ? 0 : 1)) * static_cast<long long>(N) +
               v0 - (s.xfast ? W : 1);
      b_stride = s.xfast ? W : 1;
    }
    auto gix = [&](int l) { return g_base + static_cast<long long>(l) * g_stride; };
    auto bco = [&](int l) { return coef[b_base + static_cast<long long>(l) * b_stride]; };
    if (PERSIST && kk > 0) {  // x of "line -1" is zero for every task
      for (int j = tid; j < 2 * kd_max; j += kCT) xbuf[j] = 0.0;
      compute_bar();
    }
    if (PERSIST && phase == 1) {  // both forward chains of this subdomain are done
      if (tid == 0) {
        const int need = (s.m > 0 ? 1 : 0) + (s.L - 1 - s.m > 0 ? 1 : 0);
        wait_forward_done(qsync + 1 + sub, need);
      }
      compute_bar();
    }
    // operand of line step t (k_line_solve), prefetched one step ahead; thread tid owns j = tid
    double pf_r = 0.0, pf_b = 0.0, pf_y = 0.0;
    auto prefetch = [&](int t) {
      pf_r = pf_b = pf_y = 0.0;
      const int j = tid;
      if (t >= nl || j >= kd) return;
      const int l = chain_line(phase, chain, s, t);
      if (phase == 0) {
        pf_r = rl ? rl[static_cast<long long>(l) * kd + j] : r[gix(l)];
        if (t > 0) pf_b = bco(chain == 0 ? l : l + 1);
      } else if (t == 0) {
        double w = rl ? rl[static_cast<long long>(l) * kd + j] : r[gix(l)];
        if (m > 0) w -= bco(m) * __ldcg(yl + static_cast<long long>(m - 1) * kd + j);
        if (m < L - 1) w -= bco(m + 1) * __ldcg(yl + static_cast<long long>(m + 1) * kd + j);
        pf_r = w;
      } else {
        pf_b = bco(chain == 0 ? l + 1 : l);
        pf_y = __ldcg(yl + static_cast<long long>(l) * kd + j);
      }
    };
    prefetch(0);
    double* ya = yacc + static_cast<size_t>(warp) * kd_max;
    for (int t = 0; t < nl; ++t) {
      const int l = chain_line(phase, chain, s, t);
      const int par = t & 1;
      const bool subtract = phase == 1 && t > 0;  // x_l = y_l - Dinv_l w
      const double* xprev = xbuf + (par ^ 1) * kd_max;
      if (tid < kd)
        wv[tid] = (phase == 0) ? pf_r - pf_b * xprev[tid] : (t == 0 ? pf_r : pf_b * xprev[tid]);
      const double cur_y = pf_y;
      prefetch(t + 1);
      // this line's incoming partial sums: kd doubles from each of the other CTAs
      if (C > 1 && tid == 0) mbar_arrive_expect(&xbar[par], 8u * static_cast<uint32_t>(kd) * (C - 1));
      compute_bar();
      for (int c = 0; c < nchunk; ++c, ++c_seq) {
        const int2 ce = chunk_tab[c];
        const int soff = ce.x;
        const int T0 = ce.y & 255, T1 = (ce.y >> 8) & 255, T0m = ce.y >> 16;
        const int st = c_seq & 1;
        const uint32_t sb = sb0 + static_cast<uint32_t>(st) * static_cast<uint32_t>(cap_d) * 8u;
        int tau = T0 + warp - T0m + (warp < T0m ? kCW : 0);
        // every warp waits for the stage, tiles or not: a warp may not arrive on empty for the
        // stage's next use before the producer has refilled it
        mbar_wait(&full[st], (c_seq >> 1) & 1);
        for (; tau < T1; tau += kCW) {
          const int e = tile_tab[tau];
          const int R0 = (e & 31) << 4, C0 = ((e >> 5) & 15) << 5, kind = e >> 9;
          if (kind == 0)
            rt_tile<0, FT>(sb, soff, R0, C0, kd, wv, ya, lane);
          else if (kind == 1)
            rt_tile<1, FT>(sb, soff, R0, C0, kd, wv, ya, lane);
          else if (kind == 2)
            rt_tile<2, FT>(sb, soff, R0, C0, kd, wv, ya, lane);
          else
            rt_tile<3, FT>(sb, soff, R0, C0, kd, wv, ya, lane);
        }
        if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage
      }
      compute_bar();
      const int j = tid;
      if (j < kd) {
        double tv = 0.0;
#pragma unroll 5
        for (int w = 0; w < kCW; ++w) {
          tv += yacc[w * kd_max + j];
          yacc[w * kd_max + j] = 0.0;
        }
        if (C > 1) {
          // all-to-all of the CTAs' partial sums; the line's product is their sum in CTA order
          // on every CTA. A sender is at most one line ahead of a receiver (it needs the
          // receiver's partials of the line before), so the two parities never collide.
          double* mine = xch + static_cast<size_t>(par * C + crank) * kd_max + j;
          *mine = tv;
          for (int c = 0; c < C; ++c)
            if (c != crank) st_async_remote(mine, tv, &xbar[par], static_cast<unsigned>(c));
          mbar_wait_cluster(&xbar[par], (t >> 1) & 1);
          tv = 0.0;
          for (int c = 0; c < C; ++c) tv += xch[static_cast<size_t>(par * C + c) * kd_max + j];
        }
        const long long k = static_cast<long long>(l) * kd + j;
        const bool wr = crank == 0;
        double v;
        if (!subtract) {
          v = tv;
          if (phase == 0) {
            if (wr) yl[k] = v;
            if (wr && L == 1) zl[k] = v;
          } else if (wr && chain == mid_writer(s)) {
            zl[k] = v;  // middle line, written once
          }
        } else {
          v = cur_y - tv;
          if (wr) zl[k] = v;
        }
        xbuf[par * kd_max + j] = v;
      }
      compute_bar();
    }
    if (PERSIST && phase == 0) {  // publish this forward chain (y of its lines) to the queue
      __threadfence();
      compute_bar();
      if (tid == 0) atomicAdd(qsync + 1 + sub, 1);
    }
  }
}

// ----------------------------------------------------------------- K6, register-tiled
// Latency regime (lines whose packed triangle, split over the cluster, fits the register
// file: c1, c2). A line step of the sweep is a dependent chain — the operand of line t needs
// x of line t-1 — so what bounds it is the latency of one symmetric GEMV plus its reduction,
// not the bytes. Here the line's lower triangle is cut into 32x32 tiles (I, J), I >= J, one
// tile per warp across the cluster, and each warp holds its tile of the NEXT line in
// registers (8 rows x 4 columns per lane, loaded while the current line's exchange is in
// flight, the line after that prefetched into L2). The critical path per line is then:
// operand -> 64 register FMAs -> 10 shuffles -> one st.async of the row and the column
// partial to the owners of blocks I and J -> the owner sums its nt + 1 contributions in a fixed
// order -> st.async broadcast of x to every CTA of the cluster. One CTA barrier per line.
// Contribution k of output block I: the row partial of tile (I, k) for k <= I, the column
// partial of tile (k - 1, I) for k > I (the diagonal tile gives both, its diagonal counted
// once, in the row partial). Deterministic: every sum runs in a fixed order.
constexpr int kTileWarps = 16;
constexpr int kTileThreads = kTileWarps * 32;
constexpr int kTileMaxNt = 16;
constexpr int kTileMaxOwn = 2;  // blocks per dedicated owner warp

__device__ __forceinline__ void st_async_to(uint32_t dst_cluster, double v, uint32_t bar_cluster) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                   dst_cluster),
               "d"(v), "r"(bar_cluster)
               : "memory");
}
// mbarrier wait that fails loudly instead of hanging forever: traps after ~1e11 cycles
// (~50 s at 1.965 GHz) — far beyond any legitimate wait, including time-slicing or compute
// preemption by other tenants, so only a genuine deadlock ends there
__device__ __forceinline__ void mbar_wait_g(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      ".reg .s64 t0, t1;\n"
      "mov.u64 t0, %%clock64;\n"
      "WAITG_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONEG_%=;\n"
      "mov.u64 t1, %%clock64;\n"
      "sub.s64 t1, t1, t0;\n"
      "setp.lt.s64 P1, t1, 100000000000;\n"
      "@P1 bra WAITG_%=;\n"
      "trap;\n"
      "DONEG_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local, unsigned rank) {
  uint32_t r;
  // not volatile: a pure address translation, so the compiler may hoist it out of the line loop
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---- K6, register-tiled ---------------------------------------------------------------------
// Placement tables (built on the host by set_tile_tables) for cluster-size index ci (C = 1,
// 2, 4, 8) and nt tile rows:
//  c_tile_of[ci][nt][cta][slot]  tile number (row-major over I >= J) or 255; the tiles of a
//                                CTA fill slots (= warps) 0, 1, ... and, in that order, the
//                                CTA's share of each line in its shared-memory stage
//  c_nloc[ci][nt][I]             contributions to block I written by its own CTA
//  c_owner[ci][nt][I]            warp of CTA I % C that reduces block I: the warps above the
//                                CTA's tiles when there are any (at most kTileMaxOwn blocks
//                                each), else warp I / C
// A tile (I, J) goes to the CTA of block I or of block J, whichever holds fewer bytes, so at
// least one of its two partials stays local.
__constant__ unsigned char c_tile_of[4][kTileMaxNt + 1][8][kTileWarps];
__constant__ unsigned char c_nloc[4][kTileMaxNt + 1][kTileMaxNt];
__constant__ unsigned char c_owner[4][kTileMaxNt + 1][kTileMaxNt];

__global__ void __launch_bounds__(kTileThreads, 1)
    k_line_solve_tile(const SubInfo* __restrict__ subs, const double* __restrict__ fac_t,
                      const double* __restrict__ coef, size_t N, const double* __restrict__ r,
                      double* __restrict__ ylocal, double* __restrict__ zlocal, int W, int nc,
                      int kdp_max, int stage_doubles, int phase, const int* __restrict__ flags,
                      const double* __restrict__ rlocal) {
  if (flags && (flags[0] | flags[1])) return;  // PCG converged or failed (grid-uniform)
  const int C = static_cast<int>(cl_size()), crank = static_cast<int>(cl_rank());
  const int cid = blockIdx.x / C;
  const int sub = cid >> 1, chain = cid & 1;
  const SubInfo s = subs[sub];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kd = s.kd, L = s.L, m = s.m;
  const int nl = chain_len(phase, chain, s);
  if (nl == 0) return;  // cluster-uniform
  const int nt = (kd + 31) >> 5, kdp = nt * 32;
  const int ci = C == 1 ? 0 : (C == 2 ? 1 : (C == 4 ? 2 : 3));
  const double* F = fac_t + s.fac_off;
  double* yl = ylocal + s.vec_off;
  double* zl = zlocal + s.vec_off;
  const double* rl = rlocal ? rlocal + s.vec_off : nullptr;
  const int dbg = g_solve_dbg;  // development probe: 4 skip the stage copies

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* blk_bar = reinterpret_cast<uint64_t*>(smem_raw);  // [16] one per owned block
  // operand of line step t: wv[t & 1], landed on w_bar[t & 1]. Double-buffered: an owner whose
  // block gets no contribution from this CTA may send the next operand while this CTA still
  // waits for the current one.
  uint64_t* w_bar = blk_bar + kTileWarps;                      // [2]
  uint64_t* full = w_bar + 2;                                  // [2] line stages landed
  double* stage = reinterpret_cast<double*>(smem_raw + 256);   // 2 x stage_doubles
  double* wv = stage + 2 * static_cast<size_t>(stage_doubles);  // 2 x kdp_max: operands
  long long* op_r = reinterpret_cast<long long*>(wv + 2 * kdp_max);  // kdp_max: r index, line 0
  long long* op_b = op_r + kdp_max;  // kdp_max: coupling index (coef) at line 0
  double* slots = reinterpret_cast<double*>(op_b + kdp_max);  // [owned block][nt + 1][32]
  const int n_own = (nt - crank + C - 1) / C;  // blocks crank, crank + C, ... < nt
  // this CTA's tiles: my tile's place in the line (tile-major) and in the stage (slot order),
  // and the CTA's doubles per line
  int my_tau = 255, my_off = 0, my_src = 0, my_sz = 0, cta_doubles = 0;
  for (int q = 0; q < kTileWarps; ++q) {
    const int tq = c_tile_of[ci][nt][crank][q];
    if (tq == 255) break;
    int I = 0;
    while ((I + 1) * (I + 2) / 2 <= tq) ++I;
    const int J = tq - I * (I + 1) / 2, sz = tile_size(I, J, kd);
    if (q == warp) my_tau = tq, my_off = cta_doubles, my_src = static_cast<int>(tile_off(I, J, kd)), my_sz = sz;
    cta_doubles += sz;
  }
  // contributions / operand blocks written by warps of this CTA arrive (after plain shared
  // stores); those of other CTAs complete transaction bytes (st.async)
  if (tid == 0) {
    for (int q = 0; q < n_own; ++q) mbar_init(&blk_bar[q], 1 + c_nloc[ci][nt][q * C + crank]);
    mbar_init(&w_bar[0], 1 + n_own);
    mbar_init(&w_bar[1], 1 + n_own);
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_barrier_init();
  }
  const bool has_tile = my_tau != 255;
  int TI = 0, TJ = 0;
  if (has_tile) {
    while ((TI + 1) * (TI + 2) / 2 <= my_tau) ++TI;
    TJ = my_tau - TI * (TI + 1) / 2;
  }
  const bool diag = TI == TJ;
  const int th = has_tile ? tile_h(TI, kd) : 0;
  const int rg = lane >> 3, cg = lane & 7;
  const int i0 = 32 * TI + 8 * rg;   // my rows i0 .. i0 + 7
  const int jc0 = 32 * TJ + 2 * cg;  // my columns jc0, jc0 + 1, jc0 + 16, jc0 + 17
  // where my two partials go: row partial -> block TI (contribution TJ, row cg of group rg),
  // column partial -> block TJ (contribution TI + 1, column (rg & 2 ? 16 : 0) + 2 cg + (rg & 1))
  const int orow = TI % C, ocol = TJ % C;
  const int er = ((TI / C) * (nt + 1) + TJ) * 32 + 8 * rg + cg;
  const int ec = ((TJ / C) * (nt + 1) + TI + 1) * 32 + (rg & 2 ? 16 : 0) + 2 * cg + (rg & 1);
  const uint32_t slots_u = smem_u32(slots), blk_bar_u = smem_u32(blk_bar);
  const uint32_t er_remote = mapa_u32(slots_u + 8u * er, orow);
  const uint32_t er_bar = mapa_u32(blk_bar_u + 8u * (TI / C), orow);
  const uint32_t ec_remote = mapa_u32(slots_u + 8u * ec, ocol);
  const uint32_t ec_bar = mapa_u32(blk_bar_u + 8u * (TJ / C), ocol);
  // blocks this warp reduces (ob = index among the CTA's blocks), at most two, reduced together
  static_assert(kTileMaxOwn == 2, "owner slots are unrolled by hand");
  int ob0 = -1, ob1 = -1;
  for (int q = 0; q < n_own; ++q)
    if (c_owner[ci][nt][q * C + crank] == warp) {
      if (ob0 < 0) ob0 = q; else if (ob1 < 0) ob1 = q;
    }
  const bool owner = ob0 >= 0;
  const int io0 = 32 * (ob0 * C + crank) + lane, io1 = 32 * (ob1 * C + crank) + lane;  // my rows
  uint32_t blk_tx0 = 0, blk_tx1 = 0;  // remote bytes per line into my blocks
  if (ob0 >= 0) blk_tx0 = 256u * static_cast<uint32_t>(nt + 1 - c_nloc[ci][nt][ob0 * C + crank]);
  if (ob1 >= 0) blk_tx1 = 256u * static_cast<uint32_t>(nt + 1 - c_nloc[ci][nt][ob1 * C + crank]);
  const uint32_t w_tx = 256u * static_cast<uint32_t>(nt - n_own);
  // operand addressing of unknown j: r and the slow-axis coupling are affine in the line index
  // (gidx / bcoef with the division by nc hoisted; kept in shared memory)
  if (tid < kd) {
    const int a = tid / nc, c = tid - a * nc;
    op_r[tid] = (s.xfast ? (static_cast<long long>(s.fy0) * W + s.fx0 + a)
                         : (static_cast<long long>(s.fy0 + a) * W + s.fx0)) * nc + c;
    const int k = c < 2 ? 0 : 1;
    const long long v0 = s.xfast ? static_cast<long long>(s.fy0) * W + s.fx0 + a
                                 : static_cast<long long>(s.fy0 + a) * W + s.fx0;
    op_b[tid] = s.xfast ? (8 + k) * static_cast<long long>(N) + v0 - W
                        : (6 + k) * static_cast<long long>(N) + v0 - 1;
  }
  const int r_step = s.xfast ? W * nc : nc, b_step = s.xfast ? W : 1;
  auto r_at = [&](int l, int j) {
    return rl ? rl[static_cast<long long>(l) * kd + j] : r[op_r[j] + static_cast<long long>(l) * r_step];
  };
  auto b_at = [&](int l, int j) { return coef[op_b[j] + static_cast<long long>(l) * b_step]; };
  // the operands and contribution slots start at zero (no NaN pattern of an earlier kernel's
  // shared memory can meet a zero operand; the tile loads themselves are masked by selection)
  for (int j = tid; j < 2 * kdp_max; j += kTileThreads) wv[j] = 0.0;
  for (int j = tid; j < n_own * (nt + 1) * 32; j += kTileThreads) slots[j] = 0.0;
  cl_sync();  // barriers and op_r / op_b initialised (cluster-wide: before any remote arrival)

  // my tile of line step t -> stage t & 1 (one bulk copy per warp: the warp rewrites only its
  // own region, after its own reads of line t - 2), line step t + 1 into L2; lane 0 only
  auto issue_tile = [&](int t) {
    if (!has_tile || t >= nl || (dbg & 4)) return;
    const double* Fl = F + static_cast<long long>(chain_line(phase, chain, s, t)) * s.line_sz;
    fence_proxy_async();
    bulk_g2s(stage + static_cast<size_t>(t & 1) * stage_doubles + my_off, Fl + my_src,
             static_cast<uint32_t>(my_sz) * 8u, &full[t & 1]);
    if (t + 1 < nl)
      bulk_prefetch_l2(F + static_cast<long long>(chain_line(phase, chain, s, t + 1)) * s.line_sz + my_src,
                       static_cast<uint32_t>(my_sz) * 8u);
  };
  if (tid == 0 && !(dbg & 4)) {
    mbar_expect_tx(&full[0], static_cast<uint32_t>(cta_doubles) * 8u);
    if (nl > 1) mbar_expect_tx(&full[1], static_cast<uint32_t>(cta_doubles) * 8u);
  }
  if (lane == 0) issue_tile(0), issue_tile(1);
  // operand of line step 0, computed locally; later operands come from the owners, who form
  // w of line t + 1 from their x of line t:
  //   forward   w = r_l - b o x_prev,  backward  w = b_next o x_next
  // (the backward sweep starts at the middle line: w = r_m - b_m y_{m-1} - b_{m+1} y_{m+1})
  if (tid < kdp) {
    double w = 0.0;
    if (tid < kd) {
      const int l = chain_line(phase, chain, s, 0);
      w = r_at(l, tid);
      if (phase == 1) {
        if (m > 0) w -= b_at(m, tid) * yl[static_cast<long long>(m - 1) * kd + tid];
        if (m < L - 1) w -= b_at(m + 1, tid) * yl[static_cast<long long>(m + 1) * kd + tid];
      }
    }
    wv[tid] = w;
  }
  // owners, in registers: coupling and rhs of line step t + 1 (its operand) and, backward, y of
  // line step t (the subtraction)
  double pb0 = 0.0, pr0 = 0.0, py0 = 0.0, pb1 = 0.0, pr1 = 0.0, py1 = 0.0;
  auto owner_prefetch = [&](int tw, int ty) {  // operand terms of step tw, y of step ty
    pb0 = pr0 = py0 = pb1 = pr1 = py1 = 0.0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = q == 0 ? io0 : io1;
      if ((q == 0 ? ob0 : ob1) < 0 || i >= kd) continue;
      double b = 0.0, rr = 0.0, y = 0.0;
      if (tw < nl) {
        const int l = chain_line(phase, chain, s, tw);
        b = b_at(phase == 0 ? (chain == 0 ? l : l + 1) : (chain == 0 ? l + 1 : l), i);
        if (phase == 0) rr = r_at(l, i);
      }
      if (phase == 1 && ty >= 1 && ty < nl)
        y = yl[static_cast<long long>(chain_line(phase, chain, s, ty)) * kd + i];
      if (q == 0) pb0 = b, pr0 = rr, py0 = y; else pb1 = b, pr1 = rr, py1 = y;
    }
  };
  if (owner) owner_prefetch(1, 0);
  __syncthreads();  // operand of line 0
  PROF_DECL

  for (int t = 0; t < nl; ++t) {
    const int l = chain_line(phase, chain, s, t);
    const uint32_t par = t & 1;
    if (t > 0) mbar_wait_g(&w_bar[par], ((t - 1) >> 1) & 1);  // operand of line t, all owners
    const double* wt = wv + par * kdp_max;
    PROF_MARK(0); TL_MARK(0);
    if (tid == 0 && t + 1 < nl) {
      mbar_arrive_expect(&w_bar[par ^ 1], w_tx);
      // stage (t + 1) & 1: the phase of line t - 1 has completed (its contributions are in
      // the operand of line t); the copies of line t + 1 may already be landing
      if (t >= 1 && !(dbg & 4)) mbar_expect_tx(&full[(t + 1) & 1], static_cast<uint32_t>(cta_doubles) * 8u);
    }
    if (lane == 0) {
      if (ob0 >= 0) mbar_arrive_expect(&blk_bar[ob0], blk_tx0);
      if (ob1 >= 0) mbar_arrive_expect(&blk_bar[ob1], blk_tx1);
    }
    if (has_tile) {
      // my tile from its stage into registers. The diagonal tile's entries right of the
      // diagonal read as zero (pads) and its diagonal is stored halved (pack_line): the row
      // and the column partial take the same FMA loop and add up to the full term.
      double a[8][4];
      if (!(dbg & 4)) mbar_wait_g(&full[par], (t >> 1) & 1);
      const double* Ts = stage + static_cast<size_t>(par) * stage_doubles + my_off;
      if (!diag && th == 32) {
        const double* p = Ts + 256 * rg + 2 * cg;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double2 v0 = *reinterpret_cast<const double2*>(p + 32 * k);
          const double2 v1 = *reinterpret_cast<const double2*>(p + 32 * k + 16);
          a[k][0] = v0.x, a[k][1] = v0.y, a[k][2] = v1.x, a[k][3] = v1.y;
        }
      } else if (!diag) {  // last tile row: th < 32 rows
        const double* p = Ts + 256 * rg + 2 * cg;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const bool live = 8 * rg + k < th;
          const double2 v0 = live ? *reinterpret_cast<const double2*>(p + 32 * k) : make_double2(0.0, 0.0);
          const double2 v1 = live ? *reinterpret_cast<const double2*>(p + 32 * k + 16) : make_double2(0.0, 0.0);
          a[k][0] = v0.x, a[k][1] = v0.y, a[k][2] = v1.x, a[k][3] = v1.y;
        }
      } else {  // packed lower rows: row rr at prow_off(rr), rr + 1 entries padded to even
        // (pads are zero and the diagonal is stored halved, so a loaded pair needs no masking)
        int ro = prow_off32(8 * rg);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int rr = 8 * rg + k;
          const bool live = rr < th;
          const double2 v0 = live && 2 * cg <= rr ? *reinterpret_cast<const double2*>(Ts + ro + 2 * cg)
                                                 : make_double2(0.0, 0.0);
          const double2 v1 = live && 16 + 2 * cg <= rr
                                 ? *reinterpret_cast<const double2*>(Ts + ro + 16 + 2 * cg)
                                 : make_double2(0.0, 0.0);
          a[k][0] = v0.x, a[k][1] = v0.y, a[k][2] = v1.x, a[k][3] = v1.y;
          ro += (rr + 2) & ~1;
        }
      }
      double racc[8], cacc[4];
      double wc[4];
      {
        const double2 u0 = *reinterpret_cast<const double2*>(wt + jc0);
        const double2 u1 = *reinterpret_cast<const double2*>(wt + jc0 + 16);
        wc[0] = u0.x, wc[1] = u0.y, wc[2] = u1.x, wc[3] = u1.y;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) cacc[c] = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double wr = wt[i0 + k];
        racc[k] = a[k][0] * wc[0];
#pragma unroll
        for (int c = 1; c < 4; ++c) racc[k] = fma(a[k][c], wc[c], racc[k]);
#pragma unroll
        for (int c = 0; c < 4; ++c) cacc[c] = fma(a[k][c], wr, cacc[c]);
      }
      PROF_MARK(2); TL_MARK(2);
      // rows: sum over the 8 lanes of the row group (lane bits 0-2); lane ends with row
      // i0 + cg. Columns: sum over the 4 row groups (lane bits 3-4); lane ends with column
      // c = rg of its four.
      {
        const bool b2 = lane & 4, b1 = lane & 2, b0 = lane & 1;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double send = b2 ? racc[k] : racc[k + 4];
          racc[k] = (b2 ? racc[k + 4] : racc[k]) + __shfl_xor_sync(~0u, send, 4);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double send = b1 ? racc[k] : racc[k + 2];
          racc[k] = (b1 ? racc[k + 2] : racc[k]) + __shfl_xor_sync(~0u, send, 2);
        }
        {
          const double send = b0 ? racc[0] : racc[1];
          racc[0] = (b0 ? racc[1] : racc[0]) + __shfl_xor_sync(~0u, send, 1);
        }
        const bool b4 = lane & 16, b3 = lane & 8;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const double send = b4 ? cacc[c] : cacc[c + 2];
          cacc[c] = (b4 ? cacc[c + 2] : cacc[c]) + __shfl_xor_sync(~0u, send, 16);
        }
        {
          const double send = b3 ? cacc[0] : cacc[1];
          cacc[0] = (b3 ? cacc[1] : cacc[0]) + __shfl_xor_sync(~0u, send, 8);
        }
      }
      if (orow == crank) slots[er] = racc[0]; else st_async_to(er_remote, racc[0], er_bar);
      if (ocol == crank) slots[ec] = cacc[0]; else st_async_to(ec_remote, cacc[0], ec_bar);
      if (orow == crank || ocol == crank) {
        __syncwarp();
        if (lane == 0) {
          if (orow == crank) mbar_arrive(&blk_bar[TI / C]);
          if (ocol == crank) mbar_arrive(&blk_bar[TJ / C]);
        }
      }
      PROF_MARK(3); TL_MARK(3);
      // the tile is in registers (consumed): its stage region takes line step t + 2
      if (lane == 0) issue_tile(t + 2);
    }
    if (owner) {
      // my blocks' contributions, summed in a fixed order (contribution k into acc[k & 3])
      mbar_wait_g(&blk_bar[ob0], par);
      if (ob1 >= 0) mbar_wait_g(&blk_bar[ob1], par);
      PROF_MARK(5); TL_MARK(5);
      const double* s0 = slots + static_cast<size_t>(ob0) * (nt + 1) * 32 + lane;
      const double* s1 = slots + static_cast<size_t>(ob1 < 0 ? ob0 : ob1) * (nt + 1) * 32 + lane;
      // unrolled to the table maximum and predicated, so every slot load is issued before the
      // first add (a runtime-bounded loop serialised load -> add per group of four)
      double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k <= kTileMaxNt; ++k)
        if (k <= nt) a0[k & 3] += s0[k * 32], a1[k & 3] += s1[k * 32];
      const double tv0 = (a0[0] + a0[1]) + (a0[2] + a0[3]);
      const double tv1 = (a1[0] + a1[1]) + (a1[2] + a1[3]);
      // x of my rows, the outputs, and the operand of the next line
      const bool more = t + 1 < nl;
      double wn0 = 0.0, wn1 = 0.0, vo0 = 0.0, vo1 = 0.0;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int i = q == 0 ? io0 : io1;
        if ((q == 0 ? ob0 : ob1) < 0 || i >= kd) continue;
        const double tv = q == 0 ? tv0 : tv1;
        const double v = (phase == 1 && t > 0) ? (q == 0 ? py0 : py1) - tv : tv;
        const double b = q == 0 ? pb0 : pb1, rr = q == 0 ? pr0 : pr1;
        const double w = phase == 0 ? rr - b * v : b * v;
        if (q == 0) wn0 = w, vo0 = v; else wn1 = w, vo1 = v;
      }
      TL_MARK(1);  // owners: sums done
      if (more) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if ((q == 0 ? ob0 : ob1) < 0) continue;
          const int i = q == 0 ? io0 : io1;
          const double w = q == 0 ? wn0 : wn1;
          double* wn = wv + (par ^ 1) * kdp_max + i;
          const uint32_t wl = smem_u32(wn), bl = smem_u32(&w_bar[par ^ 1]);
          for (int c = 0; c < C; ++c)
            if (c != crank) st_async_to(mapa_u32(wl, c), w, mapa_u32(bl, c));
          *wn = w;
        }
        TL_MARK(4);  // owners: operand broadcast issued
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&w_bar[par ^ 1]);
          if (ob1 >= 0) mbar_arrive(&w_bar[par ^ 1]);
        }
      }
      // the outputs after the broadcast: they are off the chain to the next line, and global
      // stores issued before it would queue in the memory pipeline ahead of the broadcast
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int i = q == 0 ? io0 : io1;
        if ((q == 0 ? ob0 : ob1) < 0 || i >= kd) continue;
        const long long e = static_cast<long long>(l) * kd + i;
        const double v = q == 0 ? vo0 : vo1;
        if (phase == 0) {
          yl[e] = v;
          if (L == 1) zl[e] = v;
        } else if (t > 0 || chain == mid_writer(s)) {
          zl[e] = v;  // (t == 0: the middle line, written once)
        }
      }
      owner_prefetch(t + 2, t + 1);
      PROF_MARK(6); TL_MARK(6);
    }
  }
  PROF_FLUSH(48);
}

}  // namespace

long long packed_line_size(int kd) { return prow_off(kd); }

void debug_prof(unsigned long long* out, int reset) {
#ifdef FFB_PROFILE
  FFB_CUDA(cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * 64));
  if (reset == 2 || reset == 3) {  // the solve (2) or factor (3) kernel's event timeline
    if (reset == 2) FFB_CUDA(cudaMemcpyFromSymbol(out, g_tl, sizeof(g_tl)));
    else FFB_CUDA(cudaMemcpyFromSymbol(out, g_ftl, sizeof(g_ftl)));
    return;
  }
  if (reset) {
    static const unsigned long long z[64] = {0};
    FFB_CUDA(cudaMemcpyToSymbol(g_prof, z, sizeof(z)));
  }
#else
  for (int i = 0; i < 64; ++i) out[i] = 0;
  (void)reset;
#endif
}

template <class K, class... Args>
static void launch_cluster(K kernel, int nblocks, int threads, size_t smem, int C,
                           cudaStream_t st, Args... args) {
  FFB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FFB_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
}

size_t factor_scratch_doubles(int /*nsub*/, int /*kd_max*/) {
  return 1;  // lines are factored in place in the packed factor storage
}

// changed[sub] = (first, last) local line touched by a triangle whose alpha differs from
// alpha_fact (a triangle touches the lines of its three vertices); (INT_MAX, -1) if none
__global__ void k_changed_lines(const SubInfo* __restrict__ subs, const double* __restrict__ alpha,
                                const double* __restrict__ alpha_fact, int W, int H,
                                int2* __restrict__ changed) {
  const SubInfo s = subs[blockIdx.x];
  int lo = 0x7fffffff, hi = -1;
  const int cx0 = max(s.fx0 - 1, 0), cx1 = min(s.fx0 + s.fw, W - 1);
  const int cy0 = max(s.fy0 - 1, 0), cy1 = min(s.fy0 + s.fh, H - 1);
  const int ncx = cx1 - cx0, ncy = cy1 - cy0;
  for (int e = threadIdx.x; e < ncx * ncy; e += blockDim.x) {
    const int cx = cx0 + e % ncx, cy = cy0 + e / ncx;
    const long long t = 2LL * (static_cast<long long>(cy) * (W - 1) + cx);
    if (alpha[t] == alpha_fact[t] && alpha[t + 1] == alpha_fact[t + 1]) continue;
    // the cell's vertices (cx..cx+1, cy..cy+1) inside the free rectangle -> their lines
    for (int dy = 0; dy <= 1; ++dy)
      for (int dx = 0; dx <= 1; ++dx) {
        const int lx = cx + dx - s.fx0, ly = cy + dy - s.fy0;
        if (lx < 0 || ly < 0 || lx >= s.fw || ly >= s.fh) continue;
        const int l = s.xfast ? ly : lx;
        lo = min(lo, l);
        hi = max(hi, l);
      }
  }
  __shared__ int slo[32], shi[32];
  for (int off = 16; off; off >>= 1) {
    lo = min(lo, __shfl_xor_sync(~0u, lo, off));
    hi = max(hi, __shfl_xor_sync(~0u, hi, off));
  }
  if ((threadIdx.x & 31) == 0) slo[threadIdx.x >> 5] = lo, shi[threadIdx.x >> 5] = hi;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (blockDim.x >> 5); ++w) lo = min(lo, slo[w]), hi = max(hi, shi[w]);
    changed[blockIdx.x] = make_int2(lo, hi);
  }
}

void changed_lines(const SubInfo* d_subs, int nsub, const double* alpha, const double* alpha_fact,
                   int W, int H, int2* changed, cudaStream_t st) {
  if (nsub <= 0) return;  // a rank without subdomains (world > parts)
  k_changed_lines<<<nsub, 256, 0, st>>>(d_subs, alpha, alpha_fact, W, H, changed);
  FFB_LAUNCHED();
}

// Single-precision copy of the packed line inverses for the opt-in f32 solve stream: lines
// [lo, hi] of every subdomain (the ones the last factorisation rewrote; all without `changed`),
// a line of the copy at fac32_off + l * ((line_sz + 3) & ~3). blockIdx.y strides the lines.
__global__ void __launch_bounds__(256)
    k_fac_to_f32(const SubInfo* __restrict__ subs, const double* __restrict__ fac,
                 float* __restrict__ fac32, const int2* __restrict__ changed) {
  const SubInfo s = subs[blockIdx.x];
  int2 chg = changed ? changed[blockIdx.x] : make_int2(0, s.L - 1);
  if (chg.x > chg.y) return;  // nothing changed in this subdomain
  // chain 0 restarts at the first changed line and runs to the middle, chain 1 at the last
  // one, and the middle line is redone (k_line_factor)
  chg.x = min(chg.x, s.m), chg.y = max(chg.y, s.m);
  const long long lstride = (s.line_sz + 3) & ~3LL;
  for (int l = chg.x + static_cast<int>(blockIdx.y); l <= chg.y; l += gridDim.y) {
    const double2* src = reinterpret_cast<const double2*>(fac + s.fac_off + static_cast<long long>(l) * s.line_sz);
    float2* dst = reinterpret_cast<float2*>(fac32 + s.fac32_off + static_cast<long long>(l) * lstride);
    const long long n2 = s.line_sz >> 1;  // line_sz is even
    for (long long i = threadIdx.x; i < n2; i += blockDim.x) {
      const double2 v = src[i];
      dst[i] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
    }
    if (threadIdx.x < 2 && (s.line_sz & 3))  // the stride's padding: read by the chunk tails
      fac32[s.fac32_off + static_cast<long long>(l) * lstride + s.line_sz + threadIdx.x] = 0.0f;
  }
}

void factor_to_f32(const SubInfo* d_subs, int nsub, const double* fac, float* fac32,
                   const int2* changed, cudaStream_t st) {
  if (nsub <= 0) return;
  k_fac_to_f32<<<dim3(nsub, 64), 256, 0, st>>>(d_subs, fac, fac32, changed);
  FFB_LAUNCHED();
}

void line_factor(const SubInfo* d_subs, int nsub, int C, int nb, int kd_max,
                 const double* coef, size_t N, int W, int nc, double* fac, double* scratch,
                 long long scratch_stride, int* d_bad, cudaStream_t st, const int2* changed,
                 double* fac_t) {
  if (nsub <= 0) return;  // a rank without subdomains (world > parts)
  const int kdp = (kd_max + 31) / 32 * 32;
  // schedule switches are read per call (tests switch them within one process)
  const int la = [] {
    const char* e = std::getenv("FFB_LOOKAHEAD");
    return e ? std::atoi(e) : 1;
  }();
  const int ldl = nb == 32 ? li_stride<32>() : li_stride<16>();
  const size_t smem = (nb * (nb + 1) + 2 * nb * ldl + 2 * nb + static_cast<size_t>(nb) * (kdp + 8)) *
                      sizeof(double);
  if (smem > 227 * 1024) fail("linsolve.cholesky: subdomain line too wide for shared memory");
  // Factor clusters of 4 CTAs regardless of how many SMs that asks for: the hardware runs the
  // clusters in waves, so only ~37 chains' lines are being rewritten at a time and stay in L2
  // (measured: c3 1.56 -> 0.78 s, c4 2.1 -> 1.5 s per adaptive chain vs one CTA per chain)
  C = nb == 16 ? 8 : 4;  // wide lines (c5): 8 (4.2 -> 3.4 s)
  if (const char* e = std::getenv("FFB_FCLUSTER")) {
    const int v = std::atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8) C = v;
  }
  // the look-ahead through D is a single-CTA schedule; the NB = 32 one works in clusters
  int lac = (C > 1 && nb != 32) ? 0 : la;
  // DMMA tile updates (measured c2 -9%, c3 -13% of the factorisation time; NB = 16, c5: -14%
  // once the tiles' read-modify-writes went to 16-byte pairs). FFB_FACTOR_MMA=0 forces FFMA.
  const int mma = [] {
    const char* e = std::getenv("FFB_FACTOR_MMA");
    return e ? std::atoi(e) : -1;
  }();
  if (mma != 0) lac |= 2;
  // subdomains per launch (FFB_FGROUP): the lines being inverted stay L2-resident only while
  // the chains in flight are few enough (every sweep step rewrites each line once)
  int G = nsub;
  if (const char* e = std::getenv("FFB_FGROUP")) G = std::max(1, std::min(nsub, std::atoi(e)));
  for (int g0 = 0; g0 < nsub; g0 += G) {
    const int ng = std::min(G, nsub - g0);
    const int2* chg = changed ? changed + g0 : nullptr;
    for (int mid = 0; mid <= 1; ++mid) {
      const int grid = (mid ? ng : 2 * ng) * C;
      if (nb == 32) {
        launch_cluster(k_line_factor<32>, grid, kFT, smem, C, st, d_subs + g0, coef, N, W, nc,
                       fac, fac_t, scratch, scratch_stride, kdp, mid, d_bad + g0, chg, lac);
      } else if (nb == 16) {
        launch_cluster(k_line_factor<16>, grid, kFT, smem, C, st, d_subs + g0, coef, N, W, nc,
                       fac, fac_t, scratch, scratch_stride, kdp, mid, d_bad + g0, chg, lac);
      } else {
        fail("internal: unsupported pivot block size");
      }
      FFB_LAUNCHED();
    }
  }
}

// placement tables of the register-tiled solve kernel (see c_tile_of), once per device.
// Tiles are weighed by their bytes with full tile rows (the last row of a line is shorter,
// so a CTA's share of any line fits the stage sized by tile_stage_doubles).
static void build_tile_tables(unsigned char (*tile_of)[kTileMaxNt + 1][8][kTileWarps],
                              unsigned char (*nloc)[kTileMaxNt + 1][kTileMaxNt],
                              unsigned char (*owner)[kTileMaxNt + 1][kTileMaxNt],
                              int (*stage)[kTileMaxNt + 1]) {
  std::memset(tile_of, 255, sizeof(unsigned char) * 4 * (kTileMaxNt + 1) * 8 * kTileWarps);
  std::memset(nloc, 0, sizeof(unsigned char) * 4 * (kTileMaxNt + 1) * kTileMaxNt);
  std::memset(owner, 0, sizeof(unsigned char) * 4 * (kTileMaxNt + 1) * kTileMaxNt);
  for (int ci = 0; ci < 4; ++ci) {
    const int C = 1 << ci;
    for (int nt = 1; nt <= kTileMaxNt; ++nt) {
      stage[ci][nt] = 0;
      const int T = nt * (nt + 1) / 2;
      if (T > kTileWarps * C) continue;
      const int total = 1024 * (T - nt) + 544 * nt;
      const int cap = (total + C - 1) / C + 1024;  // bytes/8 per CTA, one tile of slack
      int cnt[8] = {0}, load[8] = {0};
      // leave each CTA one warp per block it reduces; when the warps run out, the CTA of the
      // last block (short when kd is just past a multiple of 32) takes the extra tile and
      // its owner warp reduces that block too
      int wcap[8];
      const int c_last = (nt - 1) % C;
      for (int c = 0; c < C; ++c)
        wcap[c] = kTileWarps - (nt - c + C - 1) / C + (c == c_last && nt > C ? 1 : 0);
      int tau = 0;
      for (int I = 0; I < nt; ++I)
        for (int J = 0; J <= I; ++J, ++tau) {
          const int wgt = I == J ? 544 : 1024;
          const int a = I % C, b = J % C;
          auto fits = [&](int c) { return cnt[c] < wcap[c] && load[c] + wgt <= cap; };
          int c = load[a] <= load[b] ? a : b;
          if (!fits(c)) c = c == a ? b : a;
          if (!fits(c)) {  // both owners full: the least loaded CTA with a free slot
            c = -1;
            for (int q = 0; q < C; ++q)
              if (cnt[q] < wcap[q] && (c < 0 || load[q] < load[c])) c = q;
          }
          if (c < 0) {  // every CTA at its reserve: any warp left
            for (int q = 0; q < C; ++q)
              if (cnt[q] < kTileWarps && (c < 0 || load[q] < load[c])) c = q;
          }
          tile_of[ci][nt][c][cnt[c]++] = static_cast<unsigned char>(tau);
          load[c] += wgt;
          if (c == a) ++nloc[ci][nt][I];  // row partial stays local
          if (c == b) ++nloc[ci][nt][J];  // column partial stays local
        }
      for (int c = 0; c < C; ++c) {
        if (stage[ci][nt] >= 0) stage[ci][nt] = std::max(stage[ci][nt], load[c]);
        const int n_own = (nt - c + C - 1) / C, nfree = kTileWarps - cnt[c];
        const bool dedicated = nfree > 0 && (n_own + nfree - 1) / nfree <= kTileMaxOwn;
        for (int q = 0; q < n_own; ++q) {
          int w = dedicated ? kTileWarps - 1 - q % nfree : q;
          // exactly one warp short in the CTA of the last block: that (short) block shares
          // the first owner's warp, every other block has its own
          if (dedicated && c == c_last && nfree == n_own - 1)
            w = q == n_own - 1 ? kTileWarps - 1 : kTileWarps - 1 - q;
          owner[ci][nt][q * C + c] = static_cast<unsigned char>(w);
        }
        // the kernel reduces at most kTileMaxOwn blocks per warp: a table that asks for more
        // is not used (stage 0 -> solve_plan keeps the ring kernel)
        int per_warp[kTileWarps] = {0};
        for (int q = 0; q < n_own; ++q)
          if (++per_warp[owner[ci][nt][q * C + c]] > kTileMaxOwn) stage[ci][nt] = -1;
      }
      if (stage[ci][nt] < 0) stage[ci][nt] = 0;
    }
  }
}
static unsigned char h_tile_of[4][kTileMaxNt + 1][8][kTileWarps];
static unsigned char h_nloc[4][kTileMaxNt + 1][kTileMaxNt];
static unsigned char h_owner[4][kTileMaxNt + 1][kTileMaxNt];
static int h_stage[4][kTileMaxNt + 1];
static void ensure_tile_tables_host() {
  static std::once_flag once;
  std::call_once(once, [] { build_tile_tables(h_tile_of, h_nloc, h_owner, h_stage); });
}
// Uploaded once per device, under a lock (contexts may live on several host threads), and
// followed by a device synchronisation: the solve kernels run on non-blocking streams, which
// are not ordered after the legacy-stream symbol copies.
static void set_tile_tables() {
  static std::mutex mu;
  static unsigned long long done_mask = 0;
  int dev = 0;
  FFB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && (done_mask >> dev) & 1ull) return;
  ensure_tile_tables_host();
  FFB_CUDA(cudaMemcpyToSymbol(c_tile_of, h_tile_of, sizeof(h_tile_of)));
  FFB_CUDA(cudaMemcpyToSymbol(c_nloc, h_nloc, sizeof(h_nloc)));
  FFB_CUDA(cudaMemcpyToSymbol(c_owner, h_owner, sizeof(h_owner)));
  FFB_CUDA(cudaDeviceSynchronize());
  if (dev < 64) done_mask |= 1ull << dev;
}

void set_solve_dbg(int v) { FFB_CUDA(cudaMemcpyToSymbol(g_solve_dbg, &v, sizeof(int))); }

SolvePlan solve_plan(int kd_max, int C) {
  kd_max = (kd_max + 1) & ~1;  // even: the per-line shared arrays stay 16-byte aligned
  SolvePlan pl{};
  // measured (tools/solve_probe.py): 16 for lines up to 512 unknowns (c2: -12%), 0 beyond
  pl.row_cost = kd_max <= 512 ? 16 : 0;
  if (const char* e = std::getenv("FFB_ROW_COST")) pl.row_cost = std::atoi(e);
  pl.C = C;
  // column-partial slots: one per compute warp, or 8 (two-round reduction) for wide lines
  // where the 7 kd doubles buy ring capacity (measured: c5 -32%, c2 +5%)
  pl.ncs = (kd_max + 31) / 32 > 14 ? kCS : kCW;  // the kernels' MAXM >= 20 instantiations
  const size_t fixed = kSolveHdr + (static_cast<size_t>(pl.ncs) * kd_max + 5 * kd_max +
                                    2 * static_cast<size_t>(C) * kd_max) * sizeof(double);
  size_t budget = 227 * 1024 - 1024;
  if (const char* e = std::getenv("FFB_SOLVE_SMEM_KB")) budget = static_cast<size_t>(std::atoi(e)) * 1024;
  if (kd_max > 2 * kCT || fixed + 2 * 1024 * sizeof(double) > budget)
    fail("linsolve.cholesky: subdomain line too wide for the solve kernel");
  const size_t avail = budget - fixed;
  // as many ring stages (<= 8) as keep each stage >= 2 rows of the widest line and >= 16 KB
  int max_stages = 2;  // measured: two large stages beat 3-8 smaller ones (bulk-copy size)
  if (const char* e = std::getenv("FFB_STAGES")) max_stages = std::max(2, std::min(8, std::atoi(e)));
  int stages = max_stages;
  long long cap = 0;
  for (; stages >= 2; --stages) {
    cap = static_cast<long long>(avail / (stages * sizeof(double))) & ~1LL;
    if (cap >= 2LL * (kd_max + 2) && cap * 8 >= 16384) break;
  }
  if (stages < 2) {
    stages = 2;
    cap = static_cast<long long>(avail / (stages * sizeof(double))) & ~1LL;
  }
  if (cap < kd_max + 2) fail("linsolve.cholesky: subdomain line too wide for the solve ring");
  pl.stages = stages;
  pl.cap = static_cast<int>(cap);
  pl.smem = fixed + static_cast<size_t>(stages) * cap * sizeof(double);
  pl.maxm = (kd_max + 31) / 32;
  pl.kd_max = kd_max;
  // register-tiled kernel when the line's 32x32 tiles fit one per warp over the cluster and
  // two lines of a CTA's share fit shared memory (the latency regime: c1, c2); FFB_SOLVE=ring
  // forces the shared-memory ring kernel
  const int nt = (kd_max + 31) / 32;
  pl.tile = 0;
  const char* force = std::getenv("FFB_SOLVE");
  const bool ring_forced = force && std::string(force) == "ring";
  const bool rt_forced = force && std::string(force) == "rt" && C <= 4 && kd_max <= kRtMaxKd;
  if (!ring_forced && !rt_forced && nt <= kTileMaxNt && nt * (nt + 1) / 2 <= kTileWarps * C) {
    ensure_tile_tables_host();
    const int ci = C == 1 ? 0 : (C == 2 ? 1 : (C == 4 ? 2 : 3));
    // a stage holds a CTA's tiles of one line: the most over the CTAs and every line width
    // up to kd_max (each width uses the table of its own tile count)
    int stage = 0;
    for (int kd = 1; kd <= kd_max; ++kd) {
      const int n = (kd + 31) / 32;
      for (int c = 0; c < C; ++c) {
        int sz = 0;
        for (int q = 0; q < kTileWarps; ++q) {
          const int tq = h_tile_of[ci][n][c][q];
          if (tq == 255) break;
          int I = 0;
          while ((I + 1) * (I + 2) / 2 <= tq) ++I;
          sz += tile_size(I, tq - I * (I + 1) / 2, kd);
        }
        stage = std::max(stage, sz);
      }
    }
    pl.stage_doubles = (stage + 1) & ~1;
    const int nown = (nt + C - 1) / C;
    const size_t smem = 256 + (2 * static_cast<size_t>(pl.stage_doubles) + 4 * static_cast<size_t>(nt) * 32 +
                               static_cast<size_t>(nown) * (nt + 1) * 32) * sizeof(double);
    bool tables_ok = true;  // every tile count a subdomain of this plan can have
    for (int n = 1; n <= nt; ++n) tables_ok = tables_ok && h_stage[ci][n] > 0;
    if (tables_ok && smem <= 227 * 1024) pl.tile = 1, pl.smem = smem;
  }
  // row-group tiles (k_line_solve_rt) for one CTA per chain or clusters of 2 / 4 (each CTA a
  // run of row groups, partial sums exchanged per line): two ring stages, each holding at
  // least one 16-row group of the widest line; FFB_SOLVE=ring keeps the row-batch ring,
  // FFB_SOLVE=rt takes the row-group tiles also where the register-tiled kernel fits
  pl.rt = 0;
  if (!pl.tile && !ring_forced && C <= 4 && kd_max <= kRtMaxKd) {
    const size_t fx = kSolveHdr + (static_cast<size_t>(kCW + 3) + (C > 1 ? 2 * C : 0)) * kd_max * sizeof(double);
    const long long cap_rt = static_cast<long long>((budget - fx) / (2 * sizeof(double))) & ~1LL;
    if (cap_rt >= 16LL * (kd_max + 2)) {
      pl.rt = 1;
      pl.stages = 2;
      pl.cap = static_cast<int>(cap_rt);
      pl.smem = fx + 2 * static_cast<size_t>(cap_rt) * sizeof(double);
    }
  }
  return pl;
}

template <int M>
static void launch_solve_m(const SubInfo* d_subs, int nsub, const SolvePlan& pl,
                           const double* fac, const double* coef, size_t N, const double* r,
                           double* ylocal, double* zlocal, int W, int nc, const int* flags,
                           const double* rlocal, cudaStream_t st, int* qsync, int n_cta,
                           const float* fac32) {
  for (int phase = 0; phase <= 1; ++phase) {
    if (pl.tile) {
      set_tile_tables();
      launch_cluster(k_line_solve_tile, 2 * nsub * pl.C, kTileThreads, pl.smem, pl.C, st, d_subs,
                     fac, coef, N, r, ylocal, zlocal, W, nc, (pl.maxm) * 32, pl.stage_doubles,
                     phase, flags, rlocal);
    } else {
      // one CTA per chain: n_cta persistent CTAs pull the chains of both sweeps from a queue;
      // else one cluster per (subdomain, chain), one launch per sweep
      if (pl.rt && fac32) {  // the single-precision factor copy: a stage holds 2 cap floats
        if (qsync) {
          if (phase == 1) break;
          FFB_CUDA(cudaMemsetAsync(qsync, 0, (nsub + 1) * sizeof(int), st));
          launch_cluster(k_line_solve_rt<true, float>, n_cta, kST, pl.smem, 1, st, d_subs, fac32,
                         coef, N, r, ylocal, zlocal, W, nc, 2 * pl.cap, pl.kd_max, 0, flags, rlocal,
                         qsync, nsub);
        } else {
          launch_cluster(k_line_solve_rt<false, float>, 2 * nsub * pl.C, kST, pl.smem, pl.C, st,
                         d_subs, fac32, coef, N, r, ylocal, zlocal, W, nc, 2 * pl.cap, pl.kd_max,
                         phase, flags, rlocal, nullptr, nsub);
        }
      } else if (pl.rt) {
        if (qsync) {
          if (phase == 1) break;
          FFB_CUDA(cudaMemsetAsync(qsync, 0, (nsub + 1) * sizeof(int), st));
          launch_cluster(k_line_solve_rt<true, double>, n_cta, kST, pl.smem, 1, st, d_subs, fac,
                         coef, N, r, ylocal, zlocal, W, nc, pl.cap, pl.kd_max, 0, flags, rlocal,
                         qsync, nsub);
        } else {
          launch_cluster(k_line_solve_rt<false, double>, 2 * nsub * pl.C, kST, pl.smem, pl.C, st,
                         d_subs, fac, coef, N, r, ylocal, zlocal, W, nc, pl.cap, pl.kd_max, phase,
                         flags, rlocal, nullptr, nsub);
        }
      } else if (qsync) {  // one launch for both sweeps (the dynamic queue holds them in order)
        if (phase == 1) break;
        FFB_CUDA(cudaMemsetAsync(qsync, 0, (nsub + 1) * sizeof(int), st));
        launch_cluster(k_line_solve<M, true>, n_cta, kST, pl.smem, 1, st, d_subs, fac, coef, N, r,
                       ylocal, zlocal, W, nc, pl.stages, pl.cap, pl.kd_max, pl.row_cost, 0,
                       flags, rlocal, qsync, nsub);
      } else {
        launch_cluster(k_line_solve<M, false>, 2 * nsub * pl.C, kST, pl.smem, pl.C, st, d_subs,
                       fac, coef, N, r, ylocal, zlocal, W, nc, pl.stages, pl.cap, pl.kd_max,
                       pl.row_cost, phase, flags, rlocal, nullptr, nsub);
      }
    }
    FFB_LAUNCHED();
  }
}

void line_solve(const SubInfo* d_subs, int nsub, const SolvePlan& pl, const double* fac,
                const double* coef, size_t N, const double* r, double* ylocal, double* zlocal,
                int W, int nc, const int* flags, cudaStream_t st, const double* rlocal,
                int* qsync, int n_cta, const float* fac32) {
  if (pl.tile || pl.C != 1) qsync = nullptr;  // the task queue: ring kernel, one CTA per chain
  if (nsub <= 0) return;  // a rank without subdomains (world > parts)
  if (pl.maxm <= 4)
    launch_solve_m<4>(d_subs, nsub, pl, fac, coef, N, r, ylocal, zlocal, W, nc, flags, rlocal, st,
                      qsync, n_cta, fac32);
  else if (pl.maxm <= 8)
    launch_solve_m<8>(d_subs, nsub, pl, fac, coef, N, r, ylocal, zlocal, W, nc, flags, rlocal, st,
                      qsync, n_cta, fac32);
  else if (pl.maxm <= 14)
    launch_solve_m<14>(d_subs, nsub, pl, fac, coef, N, r, ylocal, zlocal, W, nc, flags, rlocal, st,
                      qsync, n_cta, fac32);
  else if (pl.maxm <= 20)
    launch_solve_m<20>(d_subs, nsub, pl, fac, coef, N, r, ylocal, zlocal, W, nc, flags, rlocal, st,
                      qsync, n_cta, fac32);
  else if (pl.maxm <= 26)
    launch_solve_m<26>(d_subs, nsub, pl, fac, coef, N, r, ylocal, zlocal, W, nc, flags, rlocal, st,
                      qsync, n_cta, fac32);
  else
    fail("linsolve.cholesky: subdomain line too wide (kd > 832)");
}

}  // namespace ffb
