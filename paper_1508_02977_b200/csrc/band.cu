// K4/K5/K6: batched banded Cholesky of the Schwarz subdomain operators and the
// forward/backward band solves of the additive-Schwarz preconditioner.
//
// Replaces the reference's per-part SparseCholesky (src/linsolve.cpp:107-273: RCM,
// elimination tree, up-looking level-scheduled factorization, two triangular sweeps) that
// schwarz_solve drives per subdomain (src/schwarz.cpp:236-248). On the pixel grid a
// lexicographic ordering with the short side fast already gives the RCM-sized band, so the
// symbolic phase disappears: A_i is stored as a dense row-major band (row i holds columns
// i-kd .. i, kd = nc*S), factored in place.
//
// Storage of the factor: the band holds L, except that each NB x NB diagonal block holds
// inv(L_BB) (lower triangular). The solves then never divide and the only sequential
// dependency left between NB-row blocks is one NB-wide matrix-vector product.
//
// Factor (one CTA per subdomain, right-looking, NB-column steps):
//   D = chol(A_BB) in shared memory, I = inv(D), panel L_TB = A_TB I^T (kd rows),
//   trailing update A_TT -= L_TB L_TB^T over the kd x kd lower triangle (8x8 register
//   tiles, 64x32 warp tiles; FP64 FMA pipe).
// Solve (one CTA per subdomain, HBM-streaming): NB-row blocks of the band are streamed
//   through a shared-memory ring with cp.async.bulk + mbarrier (TMA bulk copies); forward
//   x_B = I (b_B - L_B,old x_old), backward x_B = I^T (y_B - acc_B) then
//   acc_old += L_B,old^T x_B. The factor is read exactly twice per application.
#include "ffb_internal.cuh"

#include <algorithm>

namespace ffb {

namespace {

// ---------------------------------------------------------------- index helpers
__device__ __forceinline__ long long glob_index(const SubInfo& s, int k, int W, int nc) {
  const int vloc = k / nc, c = k - vloc * nc;
  const int a = vloc % s.S, b = vloc / s.S;
  const int lx = s.xfast ? a : b, ly = s.xfast ? b : a;
  return (static_cast<long long>(s.fy0 + ly) * W + (s.fx0 + lx)) * nc + c;
}

// ---------------------------------------------------------------- K4 band assembly
// One warp per band row: A_i = R_i A R_i^T in the local ordering. Couplings to vertices
// outside the free rectangle are dropped (Dirichlet restriction, assembly.cpp:155-160
// moves them to the rhs, which the preconditioner does not need).
__global__ void k_band_assemble(const SubInfo* __restrict__ subs, const double* __restrict__ coef,
                                int W, int nc, size_t N, double* __restrict__ band) {
  const SubInfo s = subs[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int kd = s.kd, kd1 = kd + 1;
  for (int row = warp; row < s.npad; row += nwarps) {
    double* out = band + s.band_off + static_cast<long long>(row) * kd1;
    double vdiag = 1.0, vb1 = 0.0, vb2 = 0.0, vfast = 0.0, vslow = 0.0;
    int c = 0;
    bool has_fast = false, has_slow = false;
    if (row < s.n) {
      const int vloc = row / nc;
      c = row - vloc * nc;
      const int a = vloc % s.S, b = vloc / s.S;
      const int lx = s.xfast ? a : b, ly = s.xfast ? b : a;
      const int gx = s.fx0 + lx, gy = s.fy0 + ly;
      const size_t v = static_cast<size_t>(gy) * W + gx;
      // m planes: 0 m11, 1 m12, 2 m13, 3 m22, 4 m23, 5 m33
      const int mi[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
      vdiag = coef[mi[c][c] * N + v];
      if (c >= 1) vb1 = coef[mi[c][c - 1] * N + v];
      if (c >= 2) vb2 = coef[mi[c][c - 2] * N + v];
      const int k = c < 2 ? 0 : 1;
      if (a > 0) {  // fast-axis predecessor
        has_fast = true;
        vfast = s.xfast ? coef[(6 + k) * N + v - 1] : coef[(8 + k) * N + v - W];
      }
      if (b > 0) {  // slow-axis predecessor
        has_slow = true;
        vslow = s.xfast ? coef[(8 + k) * N + v - W] : coef[(6 + k) * N + v - 1];
      }
    }
    const int off_slow = nc * s.S;
    for (int kk = lane; kk < kd1; kk += 32) {
      const int off = kd - kk;  // column = row - off
      double val = 0.0;
      if (off == 0) val = vdiag;
      else if (off == 1 && c >= 1) val = vb1;
      else if (off == 2 && c >= 2) val = vb2;
      else if (off == off_slow && has_slow) val = vslow;
      else if (off == nc && has_fast) val = vfast;
      out[kk] = val;
    }
  }
}

// ---------------------------------------------------------------- K5 band factor
constexpr int kFactorThreads = 256;

template <int NB>
__global__ void __launch_bounds__(kFactorThreads, 1)
    k_band_factor(const SubInfo* __restrict__ subs, double* __restrict__ band, int kdp,
                  int* __restrict__ bad) {
  const SubInfo s = subs[blockIdx.x];
  const int tid = threadIdx.x;
  const int kd = s.kd, kd1 = kd + 1;
  double* Lb = band + s.band_off;
  extern __shared__ __align__(16) double fsm[];
  double* D = fsm;                  // NB x (NB+1)
  double* I = D + NB * (NB + 1);    // NB x (NB+1)
  double* P = I + NB * (NB + 1);    // NB x kdp, P[c*kdp + u]
  // zero the panel once (its padding beyond kd stays zero)
  for (int e = tid; e < NB * kdp; e += kFactorThreads) P[e] = 0.0;
  int first_bad = 0x7fffffff;

  for (int blk = 0; blk < s.nblk; ++blk) {
    const long long i0 = static_cast<long long>(blk) * NB;
    // (1) diagonal block, lower triangle
    for (int e = tid; e < NB * NB; e += kFactorThreads) {
      const int r = e / NB, c = e - r * NB;
      D[r * (NB + 1) + c] = c <= r ? Lb[(i0 + r) * kd1 + kd - r + c] : 0.0;
    }
    __syncthreads();
    // (2) Cholesky of D: LDL^T-style elimination on unscaled columns, one barrier per step
    for (int k = 0; k < NB; ++k) {
      double dkk = D[k * (NB + 1) + k];
      if (!(dkk > 0.0) || !isfinite(dkk)) {  // linsolve.cpp:235-240
        if (tid == 0) first_bad = min(first_bad, static_cast<int>(i0) + k);
        dkk = 1.0;
      }
      const double inv = 1.0 / dkk;
      const int m = NB - 1 - k;  // trailing size
      for (int e = tid; e < m * (m + 1) / 2; e += kFactorThreads) {
        // e -> (r, c) with k < c <= r
        int rr = static_cast<int>((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
        while ((rr + 1) * (rr + 2) / 2 <= e) ++rr;
        while (rr * (rr + 1) / 2 > e) --rr;
        const int cc = e - rr * (rr + 1) / 2;
        const int r = k + 1 + rr, c = k + 1 + cc;
        D[r * (NB + 1) + c] -= D[r * (NB + 1) + k] * D[c * (NB + 1) + k] * inv;
      }
      __syncthreads();
    }
    // scale columns: L[r][k] = D[r][k] / sqrt(D[k][k]); diagonal -> sqrt
    for (int e = tid; e < NB * NB; e += kFactorThreads) {
      const int r = e / NB, c = e - r * NB;
      if (c < r) {
        double dcc = D[c * (NB + 1) + c];
        if (!(dcc > 0.0) || !isfinite(dcc)) dcc = 1.0;
        I[r * (NB + 1) + c] = D[r * (NB + 1) + c] / sqrt(dcc);
      }
    }
    __syncthreads();
    for (int r = tid; r < NB; r += kFactorThreads) {
      double d = D[r * (NB + 1) + r];
      if (!(d > 0.0) || !isfinite(d)) d = 1.0;
      I[r * (NB + 1) + r] = sqrt(d);
    }
    __syncthreads();
    for (int e = tid; e < NB * NB; e += kFactorThreads) {
      const int r = e / NB, c = e - r * NB;
      if (c <= r) D[r * (NB + 1) + c] = I[r * (NB + 1) + c];
    }
    __syncthreads();
    // (3) I = inv(D): thread c solves D y = e_c by forward substitution
    if (tid < NB) {
      const int c = tid;
      for (int r = 0; r < NB; ++r) {
        if (r < c) {
          I[r * (NB + 1) + c] = 0.0;
          continue;
        }
        double acc = r == c ? 1.0 : 0.0;
        for (int k = c; k < r; ++k) acc -= D[r * (NB + 1) + k] * I[k * (NB + 1) + c];
        I[r * (NB + 1) + c] = acc / D[r * (NB + 1) + r];
      }
    }
    __syncthreads();
    // (4) store inv(L_BB) in the band's diagonal block
    for (int e = tid; e < NB * NB; e += kFactorThreads) {
      const int r = e / NB, c = e - r * NB;
      if (c <= r) Lb[(i0 + r) * kd1 + kd - r + c] = I[r * (NB + 1) + c];
    }
    // (5) panel: rows t = i0+NB+u, u < kd; A(u,c) at band column kd-NB-u+c when >= 0
    const long long t0 = i0 + NB;
    const int nrows = static_cast<int>(min(static_cast<long long>(kd), s.npad - t0));
    for (int e = tid; e < kd * NB; e += kFactorThreads) {
      const int u = e / NB, c = e - u * NB;
      const int col = kd - NB - u + c;
      P[c * kdp + u] = (u < nrows && col >= 0) ? Lb[(t0 + u) * kd1 + col] : 0.0;
    }
    __syncthreads();
    for (int u = tid; u < nrows; u += kFactorThreads) {
      // L(u,c) = sum_{c'<=c} A(u,c') I[c][c'], descending c keeps A(u, c'<=c) intact
      for (int c = NB - 1; c >= 0; --c) {
        double acc = 0.0;
        for (int c2 = 0; c2 <= c; ++c2) acc += P[c2 * kdp + u] * I[c * (NB + 1) + c2];
        P[c * kdp + u] = acc;
      }
    }
    __syncthreads();
    for (int e = tid; e < nrows * NB; e += kFactorThreads) {
      const int u = e / NB, c = e - u * NB;
      const int col = kd - NB - u + c;
      if (col >= 0) Lb[(t0 + u) * kd1 + col] = P[c * kdp + u];
    }
    // (6) trailing update over the lower triangle of the kd x kd window
    {
      const int warp = tid >> 5, lane = tid & 31;
      const int ui = lane & 7, vi = lane >> 3;
      const int nmu = (nrows + 63) / 64;
      int m = 0;
      for (int MU = 0; MU < nmu; ++MU) {
        const int nmv = min((nrows + 31) / 32, 2 * MU + 2);
        for (int MV = 0; MV < nmv; ++MV, ++m) {
          if ((m & 7) != warp) continue;
          const int ub = 64 * MU + 8 * ui, vb = 32 * MV + 8 * vi;
          if (vb > ub + 7 || ub >= nrows) continue;  // tile entirely above the diagonal
          double acc[8][8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
#pragma unroll 4
          for (int c = 0; c < NB; ++c) {
            const double2* pu = reinterpret_cast<const double2*>(P + c * kdp + ub);
            const double2* pv = reinterpret_cast<const double2*>(P + c * kdp + vb);
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
            if (u >= nrows) break;
            double* rowp = Lb + (t0 + u) * kd1 + kd - u;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int v = vb + j;
              if (v <= u) rowp[v] -= acc[i][j];
            }
          }
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0 && first_bad != 0x7fffffff) atomicMin(bad + blockIdx.x, first_bad);
}

// ---------------------------------------------------------------- K6 band solves
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

template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

template <int NB, int THREADS>
__global__ void __launch_bounds__(THREADS, 1)
    k_asm(const SubInfo* __restrict__ subs, const double* __restrict__ band,
          const double* __restrict__ r, double* __restrict__ ylocal, double* __restrict__ zlocal,
          int W, int nc, int stages, int stage_stride, int win, const int* __restrict__ flags) {
  if (flags && (flags[0] | flags[1])) return;  // PCG converged or failed
  constexpr int G = THREADS / NB;
  static_assert(G >= 1 && G <= 32 && (G & (G - 1)) == 0, "group size");
  const SubInfo s = subs[blockIdx.x];
  const int tid = threadIdx.x;
  const int row = tid / G, g = tid % G;
  const int kd = s.kd, kd1 = kd + 1, nblk = s.nblk;
  const uint32_t bytes = static_cast<uint32_t>(NB) * kd1 * sizeof(double);
  const double* Lb = band + s.band_off;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double* stage0 = reinterpret_cast<double*>(smem_raw + 128);
  double* ring = stage0 + static_cast<size_t>(stages) * stage_stride;
  double* rhs = ring + win;
  double* xb = rhs + NB;
  const int wmask = win - 1;

  if (tid == 0) {
    for (int q = 0; q < stages; ++q) mbar_init(&bar[q], 1);
    fence_barrier_init();
  }
  for (int i = tid; i < win; i += THREADS) ring[i] = 0.0;
  __syncthreads();

  const int nq = 2 * nblk;  // forward blocks 0..nblk-1, then backward nblk-1..0
  auto issue = [&](int q) {
    const int blk = q < nblk ? q : nq - 1 - q;
    const int st = q % stages;
    fence_proxy_async();
    mbar_expect_tx(&bar[st], bytes);
    bulk_g2s(stage0 + static_cast<size_t>(st) * stage_stride,
             Lb + static_cast<long long>(blk) * NB * kd1, bytes, &bar[st]);
  };
  if (tid == 0)
    for (int q = 0; q < min(stages, nq); ++q) issue(q);

  double* yl = ylocal + s.vec_off;
  double* zl = zlocal + s.vec_off;

  // ---- forward: L y = R_i r
  for (int blk = 0; blk < nblk; ++blk) {
    const int q = blk, st = q % stages;
    const int i0 = blk * NB;
    double bval = 0.0;
    if (g == 0 && i0 + row < s.n) bval = r[glob_index(s, i0 + row, W, nc)];
    mbar_wait(&bar[st], (q / stages) & 1);
    const double* Ls = stage0 + static_cast<size_t>(st) * stage_stride;
    const double* Lr = Ls + row * kd1;
    double acc = 0.0;
    const int kmax = kd - row;  // columns i0+row-kd+k < i0
    const int jb = i0 + row - kd;
    for (int k = g; k < kmax; k += G) acc = fma(Lr[k], ring[(jb + k) & wmask], acc);
    acc = group_sum<G>(acc);
    if (g == 0) rhs[row] = bval - acc;
    __syncthreads();
    double xv = 0.0;
    for (int c = g; c <= row; c += G) xv = fma(Lr[kd - row + c], rhs[c], xv);
    xv = group_sum<G>(xv);
    if (g == 0) {
      ring[(i0 + row) & wmask] = xv;
      yl[i0 + row] = xv;
    }
    __syncthreads();
    if (tid == 0 && q + stages < nq) issue(q + stages);
  }
  // ---- backward: L^T z = y ; ring now accumulates acc_j = sum_{i>blk(j)} L_ij z_i
  for (int i = tid; i < win; i += THREADS) ring[i] = 0.0;
  __syncthreads();
  for (int bb = nblk - 1; bb >= 0; --bb) {
    const int q = nq - 1 - bb, st = q % stages;
    const int i0 = bb * NB;
    double yval = 0.0;
    if (g == 0) yval = yl[i0 + row];  // written by this same thread in the forward sweep
    mbar_wait(&bar[st], (q / stages) & 1);
    const double* Ls = stage0 + static_cast<size_t>(st) * stage_stride;
    if (g == 0) {
      const int slot = (i0 + row) & wmask;
      rhs[row] = yval - ring[slot];
      ring[slot] = 0.0;  // consumed: keep dead slots zero
    }
    __syncthreads();
    // z_B[c] = sum_{r>=c} I[r][c] rhs[r]  (c = row)
    double xv = 0.0;
    for (int rr = row + g; rr < NB; rr += G) xv = fma(Ls[rr * kd1 + kd - rr + row], rhs[rr], xv);
    xv = group_sum<G>(xv);
    if (g == 0) {
      xb[row] = xv;
      zl[i0 + row] = xv;
    }
    __syncthreads();
    // acc[j] += sum_r L[i0+r][j] z[r] for j in [i0-kd, i0): jj = j - i0 + kd
    for (int jj = tid; jj < kd; jj += THREADS) {
      const int j = i0 - kd + jj;
      if (j < 0) continue;
      const int rmax = min(NB - 1, jj);
      double sacc = 0.0;
      for (int rr = 0; rr <= rmax; ++rr) sacc = fma(Ls[rr * kd1 + jj - rr], xb[rr], sacc);
      ring[j & wmask] += sacc;
    }
    __syncthreads();
    if (tid == 0 && q + stages < nq) issue(q + stages);
  }
}

constexpr int kAsmThreads = 256;

int pow2_at_least(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace

void band_assemble(const SubInfo* d_subs, int nsub, const double* coef, int W, size_t N,
                     int nc, double* band, cudaStream_t st) {
  dim3 grid(128, nsub);
  k_band_assemble<<<grid, 256, 0, st>>>(d_subs, coef, W, nc, N, band);
  FFB_LAUNCHED();
}

void band_factor(const SubInfo* d_subs, int nsub, int nb, int kd_max, double* band, int* d_bad,
                 cudaStream_t st) {
  const int kdp = (kd_max + 63) / 64 * 64;
  const size_t smem = (2 * nb * (nb + 1) + static_cast<size_t>(nb) * kdp) * sizeof(double);
  if (nb == 32) {
    FFB_CUDA(cudaFuncSetAttribute(k_band_factor<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    k_band_factor<32><<<nsub, kFactorThreads, smem, st>>>(d_subs, band, kdp, d_bad);
  } else if (nb == 16) {
    FFB_CUDA(cudaFuncSetAttribute(k_band_factor<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    k_band_factor<16><<<nsub, kFactorThreads, smem, st>>>(d_subs, band, kdp, d_bad);
  } else {
    fail("internal: unsupported block size");
  }
  FFB_LAUNCHED();
}

AsmLaunch asm_plan(int nb, int kd_max) {
  AsmLaunch pl{};
  pl.nb = nb;
  pl.threads = kAsmThreads;
  const int win = pow2_at_least(std::max(2 * kd_max, kd_max + nb) + nb);
  const size_t stage_doubles = (static_cast<size_t>(nb) * (kd_max + 1) + 15) / 16 * 16;
  const size_t fixed = 128 + static_cast<size_t>(win + 2 * nb) * sizeof(double);
  const size_t budget = 227 * 1024;
  int stages = static_cast<int>((budget - fixed) / (stage_doubles * sizeof(double)));
  stages = std::min(stages, 4);
  if (stages < 2) fail("linsolve.cholesky: subdomain band too wide for the shared-memory ring");
  pl.stages = stages;
  pl.smem = fixed + stages * stage_doubles * sizeof(double);
  return pl;
}

void asm_solve(const SubInfo* d_subs, int nsub, int kd_max, const AsmLaunch& pl,
                 const double* band, const double* r, double* ylocal, double* zlocal, int W,
                 int nc, const int* d_ctl_flags, cudaStream_t st) {
  const int nb = pl.nb;
  const int win = pow2_at_least(std::max(2 * kd_max, kd_max + nb) + nb);
  const int stage_stride = static_cast<int>((static_cast<size_t>(nb) * (kd_max + 1) + 15) / 16 * 16);
  if (nb == 32) {
    auto k = k_asm<32, kAsmThreads>;
    FFB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(pl.smem)));
    k<<<nsub, kAsmThreads, pl.smem, st>>>(d_subs, band, r, ylocal, zlocal, W, nc, pl.stages,
                                          stage_stride, win, d_ctl_flags);
  } else if (nb == 16) {
    auto k = k_asm<16, kAsmThreads>;
    FFB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(pl.smem)));
    k<<<nsub, kAsmThreads, pl.smem, st>>>(d_subs, band, r, ylocal, zlocal, W, nc, pl.stages,
                                          stage_stride, win, d_ctl_flags);
  } else {
    fail("internal: unsupported block size");
  }
  FFB_LAUNCHED();
}

}  // namespace ffb
