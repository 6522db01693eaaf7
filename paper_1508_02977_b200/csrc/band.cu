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
    const int mi[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
    return coef[mi[ci][cj] * N + v];
  }
  if (aj == ai - 1 && ci == cj) {
    const int k = ci < 2 ? 0 : 1;
    return s.xfast ? coef[(6 + k) * N + v - 1] : coef[(8 + k) * N + v - W];
  }
  return 0.0;
}

// ----------------------------------------------------------------- K5 factor
constexpr int kFT = 256;  // factor threads

template <int NB>
__global__ void __launch_bounds__(kFT, 1)
    k_line_factor(const SubInfo* __restrict__ subs, const double* __restrict__ coef, size_t N,
                  int W, int nc, double* __restrict__ fac, double* __restrict__ scratch,
                  long long scratch_stride, int kdp, int* __restrict__ bad) {
  const SubInfo s = subs[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kd = s.kd;
  double* D = scratch + blockIdx.x * scratch_stride;  // kd x kd row-major, lower used
  double* F = fac + s.fac_off;
  extern __shared__ __align__(16) double fsm[];
  double* P = fsm;                // NB x (NB+1): pivot block, then Lc
  double* Li = P + NB * (NB + 1); // NB x (NB+1): inv(Lc)
  double* rcp = Li + NB * (NB + 1);  // NB
  double* Z = rcp + NB;           // NB x kdp: Z[c*kdp + i]
  for (int e = tid; e < NB * kdp; e += kFT) Z[e] = 0.0;
  int first_bad = 0x7fffffff;

  for (int l = 0; l < s.L; ++l) {
    // ---- D_l = A_ll - B_l Dinv_{l-1} B_l  (lower triangle)
    const double* Fp = F + static_cast<long long>(l - 1) * s.line_sz;
    for (int i = warp; i < kd; i += kFT / 32) {
      const double bi = l > 0 ? bcoef(s, coef, N, W, nc, l, i) : 0.0;
      for (int j = lane; j <= i; j += 32) {
        double v = aline(s, coef, N, W, nc, l, i, j);
        if (l > 0) v -= bi * bcoef(s, coef, N, W, nc, l, j) * Fp[prow_off(i) + j];
        D[static_cast<long long>(i) * kd + j] = v;
      }
    }
    __syncthreads();
    // ---- blocked symmetric sweep: D -> -D^{-1}
    for (int k0 = 0; k0 < kd; k0 += NB) {
      const int nbk = min(NB, kd - k0);
      const int k1 = k0 + nbk;
      for (int e = tid; e < NB * NB; e += kFT) {
        const int a = e / NB, b = e - a * NB;
        P[a * (NB + 1) + b] =
            (a < nbk && b <= a) ? D[static_cast<long long>(k0 + a) * kd + k0 + b] : 0.0;
        Li[a * (NB + 1) + b] = 0.0;
      }
      __syncthreads();
      if (warp == 0) {
        // Cholesky of the pivot block (linsolve.cpp:235-249 breakdown semantics)
        for (int k = 0; k < nbk; ++k) {
          double d = P[k * (NB + 1) + k];
          if (!(d > 0.0) || !isfinite(d)) {
            if (lane == 0) first_bad = min(first_bad, l * kd + k0 + k);
            d = 1.0;
          }
          const double piv = sqrt(d), ip = 1.0 / piv;
          __syncwarp();
          for (int r = k + 1 + lane; r < nbk; r += 32) P[r * (NB + 1) + k] *= ip;
          if (lane == 0) {
            P[k * (NB + 1) + k] = piv;
            rcp[k] = ip;
          }
          __syncwarp();
          if (lane > k && lane < nbk) {
            const double lrk = P[lane * (NB + 1) + k];
            for (int c = k + 1; c <= lane; ++c) P[lane * (NB + 1) + c] -= lrk * P[c * (NB + 1) + k];
          }
          __syncwarp();
        }
        // Li = inv(Lc), lane c computes column c
        if (lane < nbk) {
          const int c = lane;
          for (int r = 0; r < c; ++r) Li[r * (NB + 1) + c] = 0.0;
          Li[c * (NB + 1) + c] = rcp[c];
          for (int r = c + 1; r < nbk; ++r) {
            double a0 = 0.0, a1 = 0.0;
            int k = c;
            for (; k + 1 < r; k += 2) {
              a0 += P[r * (NB + 1) + k] * Li[k * (NB + 1) + c];
              a1 += P[r * (NB + 1) + k + 1] * Li[(k + 1) * (NB + 1) + c];
            }
            if (k < r) a0 += P[r * (NB + 1) + k] * Li[k * (NB + 1) + c];
            Li[r * (NB + 1) + c] = -(a0 + a1) * rcp[r];
          }
        }
      }
      __syncthreads();
      // ---- Z = A_RK Li^T for all rows outside K (rows inside K stay zero)
      for (int i = tid; i < kd; i += kFT) {
        if (i >= k0 && i < k1) {
          for (int c = 0; c < NB; ++c) Z[c * kdp + i] = 0.0;
          continue;
        }
        double a[NB];
#pragma unroll
        for (int c = 0; c < NB; ++c)
          a[c] = c < nbk ? (i > k0 ? D[static_cast<long long>(i) * kd + k0 + c]
                                   : D[static_cast<long long>(k0 + c) * kd + i])
                         : 0.0;
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int c2 = 0; c2 <= c; ++c2) acc = fma(a[c2], Li[c * (NB + 1) + c2], acc);
          Z[c * kdp + i] = acc;
        }
      }
      __syncthreads();
      // ---- A_RR -= Z Z^T over the lower triangle, K rows/columns excluded
      {
        const int ui = lane & 7, vi = lane >> 3;
        const int nmu = (kd + 63) / 64;
        int m = 0;
        for (int MU = 0; MU < nmu; ++MU) {
          const int nmv = min((kd + 31) / 32, 2 * MU + 2);
          for (int MV = 0; MV < nmv; ++MV, ++m) {
            if ((m & 7) != warp) continue;
            const int ub = 64 * MU + 8 * ui, vb = 32 * MV + 8 * vi;
            if (vb > ub + 7 || ub >= kd) continue;
            double acc[8][8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
#pragma unroll 2
            for (int c = 0; c < nbk; ++c) {
              const double2* pu = reinterpret_cast<const double2*>(Z + c * kdp + ub);
              const double2* pv = reinterpret_cast<const double2*>(Z + c * kdp + vb);
              double a[8], b[8];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const double2 x = pu[q], y = pv[q];
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
              const int u = ub + i;
              if (u >= kd) break;
              if (u >= k0 && u < k1) continue;
              double* rowp = D + static_cast<long long>(u) * kd;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int v = vb + j;
                if (v <= u && (v < k0 || v >= k1)) rowp[v] -= acc[i][j];
              }
            }
          }
        }
      }
      // ---- A_RK <- Z Li ; A_KK <- -Li^T Li   (entries disjoint from the update above)
      for (int i = tid; i < kd; i += kFT) {
        if (i >= k0 && i < k1) continue;
        double z[NB];
#pragma unroll
        for (int c = 0; c < NB; ++c) z[c] = Z[c * kdp + i];
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          if (c >= nbk) break;
          double acc = 0.0;
#pragma unroll
          for (int c2 = c; c2 < NB; ++c2) acc = fma(z[c2], Li[c2 * (NB + 1) + c], acc);
          if (i > k0)
            D[static_cast<long long>(i) * kd + k0 + c] = acc;
          else
            D[static_cast<long long>(k0 + c) * kd + i] = acc;
        }
      }
      for (int e = tid; e < nbk * nbk; e += kFT) {
        const int a = e / nbk, b = e - a * nbk;
        if (b > a) continue;
        double acc = 0.0;
        for (int mm = a; mm < nbk; ++mm) acc += Li[mm * (NB + 1) + a] * Li[mm * (NB + 1) + b];
        D[static_cast<long long>(k0 + a) * kd + k0 + b] = -acc;
      }
      __syncthreads();
    }
    // ---- Dinv_l = -D, packed rows
    double* Fl = F + static_cast<long long>(l) * s.line_sz;
    for (int i = warp; i < kd; i += kFT / 32) {
      const long long o = prow_off(i);
      for (int j = lane; j <= i; j += 32) Fl[o + j] = -D[static_cast<long long>(i) * kd + j];
      if ((i & 1) == 0 && lane == 0) Fl[o + i + 1] = 0.0;  // pad of even rows
    }
    __syncthreads();
  }
  if (tid == 0 && first_bad != 0x7fffffff) atomicMin(bad + blockIdx.x, first_bad);
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

constexpr int kSW = 16;  // solve warps
constexpr int kST = kSW * 32;

// Row chunking of one line's packed triangle: a chunk is the longest run of rows starting at
// r0 whose packed size fits `cap` doubles (at least one row). Identical on every thread.
__device__ __forceinline__ int chunk_end(int r0, int kd, long long cap) {
  const long long base = prow_off(r0);
  int r1 = r0 + 1;
  // jump close with the closed form of prow_off, then fix up
  {
    const double t = static_cast<double>(base + cap);
    int m = static_cast<int>((sqrt(1.0 + 2.0 * t) - 1.0) * 0.5);  // 2m(m+1) <= t
    int guess = 2 * m;
    if (guess > r1) r1 = guess;
  }
  if (r1 > kd) r1 = kd;
  while (r1 > r0 + 1 && prow_off(r1) - base > cap) --r1;
  while (r1 < kd && prow_off(r1 + 1) - base <= cap) ++r1;
  return r1;
}

template <int MAXM>
__global__ void __launch_bounds__(kST, 1)
    k_line_solve(const SubInfo* __restrict__ subs, const double* __restrict__ fac,
                 const double* __restrict__ coef, size_t N, const double* __restrict__ r,
                 double* __restrict__ ylocal, double* __restrict__ zlocal, int W, int nc,
                 int stages, int cap, const int* __restrict__ flags) {
  if (flags && (flags[0] | flags[1])) return;  // PCG converged or failed
  const SubInfo s = subs[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kd = s.kd, L = s.L;
  const double* F = fac + s.fac_off;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double* stage0 = reinterpret_cast<double*>(smem_raw + 128);
  double* colpart = stage0 + static_cast<size_t>(stages) * cap;  // kSW x kd
  double* wv = colpart + static_cast<size_t>(kSW) * kd;            // kd
  double* yrow = wv + kd;                                          // kd
  double* xprev = yrow + kd;                                       // kd
  double* yl = ylocal + s.vec_off;
  double* zl = zlocal + s.vec_off;

  if (tid == 0) {
    for (int q = 0; q < stages; ++q) mbar_init(&bar[q], 1);
    fence_barrier_init();
  }
  __syncthreads();

  // producer state (thread 0): sequence of chunks over forward lines 0..L-1 then backward
  // lines L-2..0; every thread tracks the consumer side identically
  const int nlines_total = L + (L - 1);
  int p_seq = 0, p_li = 0, p_r0 = 0;  // producer: next chunk
  auto line_of = [&](int li) { return li < L ? li : (L - 2) - (li - L); };
  auto produce = [&]() {  // issue one chunk if any remain (thread 0 only)
    if (p_li >= nlines_total) return;
    const int l = line_of(p_li);
    const int r1 = chunk_end(p_r0, kd, cap);
    const long long o0 = prow_off(p_r0), o1 = prow_off(r1);
    const int st = p_seq % stages;
    fence_proxy_async();
    mbar_expect_tx(&bar[st], static_cast<uint32_t>((o1 - o0) * sizeof(double)));
    bulk_g2s(stage0 + static_cast<size_t>(st) * cap, F + static_cast<long long>(l) * s.line_sz + o0,
             static_cast<uint32_t>((o1 - o0) * sizeof(double)), &bar[st]);
    ++p_seq;
    p_r0 = r1;
    if (p_r0 >= kd) {
      p_r0 = 0;
      ++p_li;
    }
  };
  if (tid == 0)
    for (int q = 0; q < stages; ++q) produce();

  int c_seq = 0;  // consumer chunk counter
  for (int li = 0; li < nlines_total; ++li) {
    const bool fwd = li < L;
    const int l = line_of(li);
    // operand of this line's GEMV
    for (int j = tid; j < kd; j += kST) {
      double w;
      if (fwd) {
        w = r[gidx(s, l, j, W, nc)];
        if (l > 0) w -= bcoef(s, coef, N, W, nc, l, j) * xprev[j];
      } else {
        w = bcoef(s, coef, N, W, nc, l + 1, j) * xprev[j];
      }
      wv[j] = w;
    }
    __syncthreads();
    double colacc[MAXM];
#pragma unroll
    for (int m = 0; m < MAXM; ++m) colacc[m] = 0.0;
    int r0 = 0;
    while (r0 < kd) {
      const int r1 = chunk_end(r0, kd, cap);
      const int st = c_seq % stages;
      mbar_wait(&bar[st], (c_seq / stages) & 1);
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
      __syncthreads();
      if (tid == 0) produce();
      ++c_seq;
      r0 = r1;
    }
#pragma unroll
    for (int m = 0; m < MAXM; ++m) {
      const int j = lane + 32 * m;
      if (j < kd) colpart[warp * kd + j] = colacc[m];
    }
    __syncthreads();
    for (int j = tid; j < kd; j += kST) {
      double t = yrow[j];
#pragma unroll 4
      for (int w = 0; w < kSW; ++w) t += colpart[w * kd + j];
      const long long k = static_cast<long long>(l) * kd + j;
      if (fwd) {
        yl[k] = t;
        xprev[j] = t;
        if (l == L - 1) zl[k] = t;  // x_{L-1} = y_{L-1}
      } else {
        const double x = yl[k] - t;
        zl[k] = x;
        xprev[j] = x;
      }
    }
    __syncthreads();
  }
}

}  // namespace

long long packed_line_size(int kd) { return prow_off(kd); }

void line_factor(const SubInfo* d_subs, int nsub, int nb, int kd_max, const double* coef,
                 size_t N, int W, int nc, double* fac, double* scratch, long long scratch_stride,
                 int* d_bad, cudaStream_t st) {
  const int kdp = (kd_max + 63) / 64 * 64;
  const size_t smem = (2 * nb * (nb + 1) + nb + static_cast<size_t>(nb) * kdp) * sizeof(double);
  if (smem > 227 * 1024) fail("linsolve.cholesky: subdomain line too wide for shared memory");
  if (nb == 32) {
    FFB_CUDA(cudaFuncSetAttribute(k_line_factor<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    k_line_factor<32><<<nsub, kFT, smem, st>>>(d_subs, coef, N, W, nc, fac, scratch,
                                               scratch_stride, kdp, d_bad);
  } else if (nb == 16) {
    FFB_CUDA(cudaFuncSetAttribute(k_line_factor<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    k_line_factor<16><<<nsub, kFT, smem, st>>>(d_subs, coef, N, W, nc, fac, scratch,
                                               scratch_stride, kdp, d_bad);
  } else {
    fail("internal: unsupported pivot block size");
  }
  FFB_LAUNCHED();
}

SolvePlan solve_plan(int kd_max) {
  SolvePlan pl{};
  const size_t fixed = 128 + (static_cast<size_t>(kSW) * kd_max + 3 * kd_max) * sizeof(double);
  const size_t budget = 227 * 1024 - 1024;
  if (fixed + 2 * 1024 * sizeof(double) > budget)
    fail("linsolve.cholesky: subdomain line too wide for the solve kernel");
  const size_t avail = budget - fixed;
  // 3 stages when each still holds >= 4 rows of the widest line, else 2
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
  return pl;
}

template <int M>
static void launch_solve_m(const SubInfo* d_subs, int nsub, const SolvePlan& pl,
                           const double* fac, const double* coef, size_t N, const double* r,
                           double* ylocal, double* zlocal, int W, int nc, const int* flags,
                           cudaStream_t st) {
  auto k = k_line_solve<M>;
  FFB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(pl.smem)));
  k<<<nsub, kST, pl.smem, st>>>(d_subs, fac, coef, N, r, ylocal, zlocal, W, nc, pl.stages,
                                pl.cap, flags);
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
