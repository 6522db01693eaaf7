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
// Factor (K5, one CTA per subdomain): per line, build D_l in an L2-resident kd x kd scratch
// and invert it in place with a blocked symmetric sweep (Gauss-Jordan for SPD):
//     pivot block K: Lc = chol(A_KK), Li = Lc^-1, Z = A_RK Li^T,
//     A_RR -= Z Z^T (8x8 register tiles, FP64 FMA), A_RK <- Z Li, A_KK <- -Li^T Li,
// which leaves -D^{-1}; the flops equal a banded Cholesky's (n kd^2 / 2 FMAs).
// Solve (K6, one CTA per subdomain): the packed rows of each line are streamed through a
// shared-memory ring with cp.async.bulk + mbarrier (TMA bulk copies); each warp takes whole
// rows, producing the row dot products and, for the symmetric half, per-lane column partial
// sums in registers, combined in a fixed order (deterministic).
#include "ffb_internal.cuh"

#include <algorithm>

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
#else
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
// address of `p` (a shared-memory variable of this CTA) in CTA `rank` of the cluster
template <class T>
__device__ __forceinline__ T* cl_map(T* p, unsigned rank) {
  size_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(p), "r"(rank));
  return reinterpret_cast<T*>(out);
}

// rows [row_lo(c), row_lo(c+1)) of a packed lower triangle of size kd: equal shares of the
// kd(kd+1)/2 entries (cumulative work ~ i^2/2)
__device__ __forceinline__ int row_lo(int c, int C, int kd) {
  if (c <= 0) return 0;
  if (c >= C) return kd;
  int r = static_cast<int>(kd * sqrt(static_cast<double>(c) / C) + 0.5);
  return min(max(r, c), kd - (C - c));
}

// ----------------------------------------------------------------- K5 factor
constexpr int kFT = 256;  // factor threads per CTA
constexpr int kFW = kFT / 32;

template <int NB, int ZR>
__global__ void __launch_bounds__(kFT, 1)
    k_line_factor(const SubInfo* __restrict__ subs, const double* __restrict__ coef, size_t N,
                  int W, int nc, double* __restrict__ fac, double* __restrict__ scratch,
                  long long scratch_stride, int kdp, int* __restrict__ bad) {
  const int C = static_cast<int>(cl_size()), crank = static_cast<int>(cl_rank());
  const int sub = blockIdx.x / C;
  const SubInfo s = subs[sub];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gtid = crank * kFT + tid, GT = C * kFT;       // cluster-wide thread id
  const int gwarp = crank * kFW + warp, GW = C * kFW;     // cluster-wide warp id
  const int kd = s.kd;
  double* D = scratch + sub * scratch_stride;  // kd x kd row-major, lower triangle used
  double* F = fac + s.fac_off;
  extern __shared__ __align__(16) double fsm[];
  double* P = fsm;                    // NB x (NB+1): Cholesky factor of the pivot block
  double* Li = P + NB * (NB + 1);     // NB x (NB+1): its inverse
  double* rcp = Li + NB * (NB + 1);   // NB: 1 / diag
  double* Z = rcp + NB;               // NB x kdp: Z[c*kdp + i]
  for (int e = tid; e < NB * kdp; e += kFT) Z[e] = 0.0;
  int first_bad = 0x7fffffff;
  PROF_DECL

  for (int l = 0; l < s.L; ++l) {
    // ---- D_l = A_ll - B_l Dinv_{l-1} B_l  (lower triangle), rows shared by the cluster
    const double* Fp = F + static_cast<long long>(l - 1) * s.line_sz;
    for (int i = gwarp; i < kd; i += GW) {
      const double bi = l > 0 ? bcoef(s, coef, N, W, nc, l, i) : 0.0;
      for (int j = lane; j <= i; j += 32) {
        double v = aline(s, coef, N, W, nc, l, i, j);
        if (l > 0) v -= bi * bcoef(s, coef, N, W, nc, l, j) * Fp[prow_off(i) + j];
        D[static_cast<long long>(i) * kd + j] = v;
      }
    }
    cl_sync();
    PROF_MARK(0);
    // ---- blocked symmetric sweep: D -> -D^{-1}
    for (int k0 = 0; k0 < kd; k0 += NB) {
      const int nbk = min(NB, kd - k0);
      const int k1 = k0 + nbk;
      // ---- prefetch this thread's rows of the column block A_RK into L1: their latency
      // overlaps the pivot factorization below
#pragma unroll
      for (int q = 0; q < ZR; ++q) {
        const int i = tid + kFT * q;
        if (i >= kd || (i >= k0 && i < k1)) continue;
        if (i > k0) {
          const double* p = D + static_cast<long long>(i) * kd + k0;
          asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(p + NB - 1));
        } else if ((i & 15) == 0) {
          for (int c = 0; c < nbk; ++c)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(D + static_cast<long long>(k0 + c) * kd + i));
        }
      }
      // ---- pivot block (warp 0, redundantly in every CTA): Cholesky with lane r holding
      // row r in registers (breakdown semantics of linsolve.cpp:235-249), then Li = inv(L)
      // with lane c producing column c from broadcast shared-memory reads
      if (warp == 0) {
        const int r = lane;
        double row[NB];
#pragma unroll
        for (int c = 0; c < NB; ++c)
          row[c] = (r < nbk && c <= r) ? D[static_cast<long long>(k0 + r) * kd + k0 + c]
                                       : (r == c ? 1.0 : 0.0);
        double my_rcp = 1.0;
#pragma unroll NB
        for (int k = 0; k < NB; ++k) {
          double dkk = __shfl_sync(0xffffffffu, row[k], k);
          if (!(dkk > 0.0) || !isfinite(dkk)) {
            if (lane == 0 && k < nbk) first_bad = min(first_bad, l * kd + k0 + k);
            dkk = 1.0;
          }
          const double piv = sqrt(dkk), ip = 1.0 / piv;
          const double lk = r > k ? row[k] * ip : (r == k ? piv : 0.0);
          row[k] = lk;
          if (r == k) my_rcp = ip;
#pragma unroll NB
          for (int c = k + 1; c < NB; ++c) {
            const double lck = __shfl_sync(0xffffffffu, lk, c);
            if (r >= c) row[c] -= lk * lck;
          }
        }
#pragma unroll
        for (int c = 0; c < NB; ++c) P[r * (NB + 1) + c] = c <= r ? row[c] : 0.0;
        rcp[r] = my_rcp;
        __syncwarp();
        // Li = inv(L): lane c builds column c directly in shared memory
        const int c = lane;
#pragma unroll
        for (int rr = 0; rr < NB; ++rr) {
          double a0 = rr == c ? 1.0 : 0.0, a1 = 0.0;
          for (int k = c; k + 1 < rr; k += 2) {
            a0 -= P[rr * (NB + 1) + k] * Li[k * (NB + 1) + c];
            a1 -= P[rr * (NB + 1) + k + 1] * Li[(k + 1) * (NB + 1) + c];
          }
          if (((rr - c) & 1) && rr > c) a0 -= P[rr * (NB + 1) + rr - 1] * Li[(rr - 1) * (NB + 1) + c];
          Li[rr * (NB + 1) + c] = (rr < nbk && c < nbk && rr >= c) ? (a0 + a1) * rcp[rr] : 0.0;
        }
      }
      __syncthreads();
      PROF_MARK(1);
      double a[ZR][NB];
#pragma unroll
      for (int q = 0; q < ZR; ++q) {
        const int i = tid + kFT * q;
        const bool live = i < kd && (i < k0 || i >= k1);
#pragma unroll
        for (int c = 0; c < NB; ++c)
          a[q][c] = (live && c < nbk) ? (i > k0 ? D[static_cast<long long>(i) * kd + k0 + c]
                                                : D[static_cast<long long>(k0 + c) * kd + i])
                                      : 0.0;
      }
      PROF_MARK(2);
      // ---- Z = A_RK Li^T for every row outside K (each CTA keeps the whole Z); each Li
      // element read from shared memory feeds ZR rows
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        double acc[ZR];
#pragma unroll
        for (int q = 0; q < ZR; ++q) acc[q] = 0.0;
#pragma unroll
        for (int c2 = 0; c2 <= c; ++c2) {
          const double li = Li[c * (NB + 1) + c2];
#pragma unroll
          for (int q = 0; q < ZR; ++q) acc[q] = fma(a[q][c2], li, acc[q]);
        }
#pragma unroll
        for (int q = 0; q < ZR; ++q) {
          const int i = tid + kFT * q;
          if (i < kdp) Z[c * kdp + i] = acc[q];
        }
      }
      PROF_MARK(3);
      cl_sync();  // Z complete everywhere; all reads of A_RK done before it is overwritten
      PROF_MARK(4);
      // ---- A_RR -= Z Z^T over the lower triangle (K excluded): 64x32 warp tiles spread
      // over the cluster's warps; thread tile 8x8 with rows ub0+16q+2ui+{0,1} and columns
      // vb0+8q+2vi+{0,1} so that shared-memory reads are conflict-free double2 loads
      {
        const int ui = lane & 7, vi = lane >> 3;
        const int nmu = (kd + 63) / 64, nmv_all = (kd + 31) / 32;
        int MU = 0, MV = 0, m = 0;  // walk the (MU, MV) list, taking every GW-th entry
        auto advance = [&](int steps) {
          while (steps-- > 0) {
            if (++MV >= min(nmv_all, 2 * MU + 2)) MV = 0, ++MU;
          }
        };
        advance(gwarp);
        m = gwarp;
        for (; MU < nmu; advance(GW), m += GW) {
          {
            const int ub0 = 64 * MU + 2 * ui, vb0 = 32 * MV + 2 * vi;
            double acc[8][8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
#pragma unroll 2
            for (int c = 0; c < nbk; ++c) {
              const double* zc = Z + c * kdp;
              double a[8], b[8];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const double2 x = *reinterpret_cast<const double2*>(zc + ub0 + 16 * q);
                const double2 y = *reinterpret_cast<const double2*>(zc + vb0 + 8 * q);
                a[2 * q] = x.x, a[2 * q + 1] = x.y;
                b[2 * q] = y.x, b[2 * q + 1] = y.y;
              }
#pragma unroll
              for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int u = ub0 + 16 * (i >> 1) + (i & 1);
              if (u >= kd || (u >= k0 && u < k1)) continue;
              double* rowp = D + static_cast<long long>(u) * kd;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int v = vb0 + 8 * (j >> 1) + (j & 1);
                if (v <= u && (v < k0 || v >= k1)) rowp[v] -= acc[i][j];
              }
            }
          }
        }
      }
      PROF_MARK(5);
      // ---- A_RK <- Z Li ; A_KK <- -Li^T Li   (entries disjoint from the update above)
      for (int i = gtid; i < kd; i += GT) {
        if (i >= k0 && i < k1) continue;
        double z[NB];
#pragma unroll
        for (int c = 0; c < NB; ++c) z[c] = Z[c * kdp + i];
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          if (c < nbk) {
            double acc = 0.0;
#pragma unroll
            for (int c2 = c; c2 < NB; ++c2) acc = fma(z[c2], Li[c2 * (NB + 1) + c], acc);
            if (i > k0)
              D[static_cast<long long>(i) * kd + k0 + c] = acc;
            else
              D[static_cast<long long>(k0 + c) * kd + i] = acc;
          }
        }
      }
      for (int e = gtid; e < nbk * nbk; e += GT) {
        const int a = e / nbk, b = e - a * nbk;
        if (b > a) continue;
        double acc = 0.0;
        for (int mm = a; mm < nbk; ++mm) acc += Li[mm * (NB + 1) + a] * Li[mm * (NB + 1) + b];
        D[static_cast<long long>(k0 + a) * kd + k0 + b] = -acc;
      }
      PROF_MARK(6);
      cl_sync();
      PROF_MARK(7);
    }
    // ---- Dinv_l = -D, packed rows
    double* Fl = F + static_cast<long long>(l) * s.line_sz;
    for (int i = gwarp; i < kd; i += GW) {
      const long long o = prow_off(i);
      for (int j = lane; j <= i; j += 32) Fl[o + j] = -D[static_cast<long long>(i) * kd + j];
      if ((i & 1) == 0 && lane == 0) Fl[o + i + 1] = 0.0;  // pad of even rows
    }
    cl_sync();
    PROF_MARK(8);
  }
  PROF_FLUSH(0);
  if (crank == 0 && tid == 0 && first_bad != 0x7fffffff) atomicMin(bad + sub, first_bad);
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

constexpr int kSW = 16;  // solve warps per CTA
constexpr int kST = kSW * 32;

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

template <int MAXM>
__global__ void __launch_bounds__(kST, 1)
    k_line_solve(const SubInfo* __restrict__ subs, const double* __restrict__ fac,
                 const double* __restrict__ coef, size_t N, const double* __restrict__ r,
                 double* __restrict__ ylocal, double* __restrict__ zlocal, int W, int nc,
                 int stages, int cap, int kd_max, const int* __restrict__ flags) {
  if (flags && (flags[0] | flags[1])) return;  // PCG converged or failed (cluster-uniform)
  const int C = static_cast<int>(cl_size()), crank = static_cast<int>(cl_rank());
  const int sub = blockIdx.x / C;
  const SubInfo s = subs[sub];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kd = s.kd, L = s.L;
  const int rlo = row_lo(crank, C, kd), rhi = row_lo(crank + 1, C, kd);
  const int share = (kd + C - 1) / C + kd;  // upper bound on any CTA's row count
  const double* F = fac + s.fac_off;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double* stage0 = reinterpret_cast<double*>(smem_raw + 128);
  double* colpart = stage0 + static_cast<size_t>(stages) * cap;  // kSW x kd_max
  double* wv = colpart + static_cast<size_t>(kSW) * kd_max;      // kd_max
  double* yrow = wv + kd_max;                                    // kd_max (own rows)
  double* xprev = yrow + kd_max;                                 // kd_max
  double* red = xprev + kd_max;                                  // 8 x kd_max reduce slots
  double* yl = ylocal + s.vec_off;
  double* zl = zlocal + s.vec_off;
  (void)share;

  if (tid == 0) {
    for (int q = 0; q < stages; ++q) mbar_init(&bar[q], 1);
    fence_barrier_init();
  }
  for (int j = tid; j < kd_max; j += kST) xprev[j] = 0.0;
  __syncthreads();

  const int nlines_total = L + (L - 1);  // forward lines 0..L-1, backward L-2..0
  auto line_of = [&](int li) { return li < L ? li : (L - 2) - (li - L); };
  int p_seq = 0, p_li = 0, p_r0 = rlo;  // producer (thread 0)
  auto produce = [&]() {
    if (p_li >= nlines_total || rlo >= rhi) return;
    const int l = line_of(p_li);
    const int r1 = chunk_end(p_r0, rhi, cap);
    const long long o0 = prow_off(p_r0), o1 = prow_off(r1);
    const int st = p_seq % stages;
    fence_proxy_async();
    mbar_expect_tx(&bar[st], static_cast<uint32_t>((o1 - o0) * sizeof(double)));
    bulk_g2s(stage0 + static_cast<size_t>(st) * cap, F + static_cast<long long>(l) * s.line_sz + o0,
             static_cast<uint32_t>((o1 - o0) * sizeof(double)), &bar[st]);
    ++p_seq;
    p_r0 = r1;
    if (p_r0 >= rhi) {
      p_r0 = rlo;
      ++p_li;
    }
  };
  if (tid == 0)
    for (int q = 0; q < stages; ++q) produce();

  // operands of the next line are prefetched into registers one line ahead: r_l and B_l
  // (forward), B_{l+1} and y_l of the owned rows (backward); only x_{l-1} / x_{l+1} (from
  // the previous line, in shared memory) is on the line-to-line critical path
  constexpr int PS = 2;  // j = tid + kST*q, kd <= 2*kST
  double pf_r[PS], pf_b[PS], pf_y[PS];
  auto prefetch = [&](int li) {
#pragma unroll
    for (int q = 0; q < PS; ++q) {
      pf_r[q] = pf_b[q] = pf_y[q] = 0.0;
      if (li >= nlines_total) continue;
      const bool fw = li < L;
      const int l = line_of(li);
      const int j = tid + kST * q;
      if (j < kd) {
        if (fw) {
          pf_r[q] = r[gidx(s, l, j, W, nc)];
          if (l > 0) pf_b[q] = bcoef(s, coef, N, W, nc, l, j);
        } else {
          pf_b[q] = bcoef(s, coef, N, W, nc, l + 1, j);
        }
      }
      const int jo = rlo + tid + kST * q;  // owned row
      if (!fw && jo < rhi) pf_y[q] = yl[static_cast<long long>(l) * kd + jo];
    }
  };
  prefetch(0);
  PROF_DECL

  int c_seq = 0;
  for (int li = 0; li < nlines_total; ++li) {
    const bool fwd = li < L;
    const int l = line_of(li);
    double cur_y[PS];
#pragma unroll
    for (int q = 0; q < PS; ++q) {
      const int j = tid + kST * q;
      if (j < kd) wv[j] = fwd ? pf_r[q] - pf_b[q] * xprev[j] : pf_b[q] * xprev[j];
      cur_y[q] = pf_y[q];
    }
    prefetch(li + 1);
    __syncthreads();
    PROF_MARK(0);
    double colacc[MAXM];
#pragma unroll
    for (int m = 0; m < MAXM; ++m) colacc[m] = 0.0;
    int r0 = rlo;
    while (r0 < rhi) {
      const int r1 = chunk_end(r0, rhi, cap);
      const int st = c_seq % stages;
      PROF_MARK(1);
      mbar_wait(&bar[st], (c_seq / stages) & 1);
      PROF_MARK(2);
      const double* Sb = stage0 + static_cast<size_t>(st) * cap - prow_off(r0);
      for (int i = r0 + warp; i < r1; i += kSW) {
        const double* Si = Sb + prow_off(i);
        const double wi = wv[i];
        double racc = 0.0;
#pragma unroll
        for (int m = 0; m < MAXM; ++m) {
          const int j = lane + 32 * m;
          if (32 * m > i) break;
          if (j <= i) {
            const double sij = Si[j];
            racc = fma(sij, wv[j], racc);
            if (j < i) colacc[m] = fma(sij, wi, colacc[m]);
          }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) racc += __shfl_xor_sync(0xffffffffu, racc, off);
        if (lane == 0) yrow[i] = racc;
      }
      PROF_MARK(3);
      __syncthreads();
      PROF_MARK(4);
      if (tid == 0) produce();
      ++c_seq;
      r0 = r1;
    }
#pragma unroll
    for (int m = 0; m < MAXM; ++m) {
      const int j = lane + 32 * m;
      if (j < rhi) colpart[warp * kd_max + j] = colacc[m];
    }
    __syncthreads();
    PROF_MARK(5);
    // column partials of this CTA (+ its own row dots), reduced in a fixed warp order and
    // scattered to the CTA that owns each row
    int owner = 0;
    for (int j = tid; j < rhi; j += kST) {
      double t = (j >= rlo) ? yrow[j] : 0.0;
#pragma unroll 4
      for (int w = 0; w < kSW; ++w) t += colpart[w * kd_max + j];
      while (owner + 1 < C && row_lo(owner + 1, C, kd) <= j) ++owner;
      if (C == 1)
        red[j] = t;
      else
        cl_map(red, static_cast<unsigned>(owner))[crank * kd_max + j] = t;
    }
    PROF_MARK(6);
    if (C == 1) __syncthreads(); else cl_sync();
    PROF_MARK(7);
    // owners finish their rows (contributions from CTAs crank..C-1, ascending) and
    // broadcast the line's result to every CTA
#pragma unroll
    for (int q = 0; q < PS; ++q) {
      const int j = rlo + tid + kST * q;
      if (j >= rhi) continue;
      double t = 0.0;
      if (C == 1) {
        t = red[j];
      } else {
        for (int c = crank; c < C; ++c) t += red[c * kd_max + j];
      }
      const long long k = static_cast<long long>(l) * kd + j;
      double v;
      if (fwd) {
        yl[k] = t;
        if (l == L - 1) zl[k] = t;  // x_{L-1} = y_{L-1}
        v = t;
      } else {
        v = cur_y[q] - t;
        zl[k] = v;
      }
      if (C == 1) {
        xprev[j] = v;
      } else {
        for (int c = 0; c < C; ++c) cl_map(xprev, static_cast<unsigned>(c))[j] = v;
      }
    }
    PROF_MARK(8);
    if (C == 1) __syncthreads(); else cl_sync();
    PROF_MARK(9);
  }
  PROF_FLUSH(16);
}

}  // namespace

long long packed_line_size(int kd) { return prow_off(kd); }

void debug_prof(unsigned long long* out, bool reset) {
#ifdef FFB_PROFILE
  FFB_CUDA(cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * 64));
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

void line_factor(const SubInfo* d_subs, int nsub, int C, int nb, int kd_max, const double* coef,
                 size_t N, int W, int nc, double* fac, double* scratch, long long scratch_stride,
                 int* d_bad, cudaStream_t st) {
  const int kdp = (kd_max + 63) / 64 * 64;
  const size_t smem =
      (2 * nb * (nb + 1) + nb + static_cast<size_t>(nb) * kdp) * sizeof(double);
  if (smem > 227 * 1024) fail("linsolve.cholesky: subdomain line too wide for shared memory");
  const int zr = (kdp + kFT - 1) / kFT;
#define FFB_FACTOR(NBV, ZRV)                                                                 \
  launch_cluster(k_line_factor<NBV, ZRV>, nsub * C, kFT, smem, C, st, d_subs, coef, N, W, nc, \
                 fac, scratch, scratch_stride, kdp, d_bad)
  if (nb == 32 && zr <= 1) FFB_FACTOR(32, 1);
  else if (nb == 32 && zr <= 2) FFB_FACTOR(32, 2);
  else if (nb == 16 && zr <= 2) FFB_FACTOR(16, 2);
  else if (nb == 16 && zr <= 4) FFB_FACTOR(16, 4);
  else fail("internal: unsupported pivot block / line width combination");
#undef FFB_FACTOR
  FFB_LAUNCHED();
}

SolvePlan solve_plan(int kd_max, int C) {
  SolvePlan pl{};
  pl.C = C;
  const size_t fixed =
      128 + (static_cast<size_t>(kSW) * kd_max + 3 * kd_max + 8 * kd_max) * sizeof(double);
  const size_t budget = 227 * 1024 - 1024;
  if (fixed + 2 * 1024 * sizeof(double) > budget)
    fail("linsolve.cholesky: subdomain line too wide for the solve kernel");
  const size_t avail = budget - fixed;
  int stages = 3;
  long long cap = static_cast<long long>(avail / (stages * sizeof(double))) & ~1LL;
  if (cap < 4LL * (kd_max + 2)) {
    stages = 2;
    cap = static_cast<long long>(avail / (stages * sizeof(double))) & ~1LL;
  }
  if (cap < kd_max + 2) fail("linsolve.cholesky: subdomain line too wide for the solve ring");
  pl.stages = stages;
  pl.cap = static_cast<int>(cap);
  pl.smem = fixed + static_cast<size_t>(stages) * cap * sizeof(double);
  pl.maxm = (kd_max + 31) / 32;
  pl.kd_max = kd_max;
  return pl;
}

template <int M>
static void launch_solve_m(const SubInfo* d_subs, int nsub, const SolvePlan& pl,
                           const double* fac, const double* coef, size_t N, const double* r,
                           double* ylocal, double* zlocal, int W, int nc, const int* flags,
                           cudaStream_t st) {
  launch_cluster(k_line_solve<M>, nsub * pl.C, kST, pl.smem, pl.C, st, d_subs, fac, coef, N, r,
                 ylocal, zlocal, W, nc, pl.stages, pl.cap, pl.kd_max, flags);
}

void line_solve(const SubInfo* d_subs, int nsub, const SolvePlan& pl, const double* fac,
                const double* coef, size_t N, const double* r, double* ylocal, double* zlocal,
                int W, int nc, const int* flags, cudaStream_t st) {
  if (pl.maxm <= 4)
    launch_solve_m<4>(d_subs, nsub, pl, fac, coef, N, r, ylocal, zlocal, W, nc, flags, st);
  else if (pl.maxm <= 8)
    launch_solve_m<8>(d_subs, nsub, pl, fac, coef, N, r, ylocal, zlocal, W, nc, flags, st);
  else if (pl.maxm <= 14)
    launch_solve_m<14>(d_subs, nsub, pl, fac, coef, N, r, ylocal, zlocal, W, nc, flags, st);
  else if (pl.maxm <= 20)
    launch_solve_m<20>(d_subs, nsub, pl, fac, coef, N, r, ylocal, zlocal, W, nc, flags, st);
  else if (pl.maxm <= 26)
    launch_solve_m<26>(d_subs, nsub, pl, fac, coef, N, r, ylocal, zlocal, W, nc, flags, st);
  else
    fail("linsolve.cholesky: subdomain line too wide (kd > 832)");
  FFB_LAUNCHED();
}

}  // namespace ffb
