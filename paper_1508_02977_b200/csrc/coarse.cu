// Two-level additive Schwarz: a coarse space added to the one-level preconditioner of pcg.cu.
//
//   M^-1 = sum_i R_i^T A_i^-1 R_i  +  Z A0^-1 Z^T,     A0 = Z^T A Z,
//
// Z has one column per (core, component): the indicator of the non-overlapping core i of the
// partition (build_partition's cores tile the image, schwarz.cpp:74-91) for component c — a
// piecewise-constant (Nicolaides-type) coarse space with nc * px * py unknowns (c4: 768).
// M^-1 stays symmetric positive definite, so CG converges to the same solution as with the
// one-level operator; what changes is the iteration count, which for the one-level method
// grows with the number of subdomains across the image (global information crosses one
// subdomain per iteration) — c3 (8x8) needs 36 iterations for its first solve, c4 (16x16,
// same subdomain size) 57. SURVEY §7 allows a coarse space that keeps M SPD.
//
// Per refactorisation (alpha or terms changed): k_coarse_assemble (one CTA per core: its
// rows of A summed per coarse column, fixed-order block reductions) -> A0 in band storage
// (coarse unknowns ordered with the shorter subdomain axis fastest: bandwidth nc * min(px,py))
// -> band Cholesky (linsolve.cu) -> k_coarse_inverse (one warp per column of A0^-1). Per CG
// iteration: k_coarse_restrict (g = Z^T r, one CTA per core) and k_coarse_apply (y = A0^-1 g,
// one warp per row); k_combine adds y[core(p)] to z. Both per-iteration kernels read only r
// (24 B/px) and A0^-1 (n0^2 doubles, 4.7 MB at c4), ~0.3% of an iteration's bytes.
// All reductions run in a fixed order: results are bitwise reproducible.
#include "ffb_internal.cuh"

namespace ffb {

namespace {

constexpr int kCT = 256;

__device__ __forceinline__ double block_sum_c(double v, double* sm) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_down_sync(~0u, v, off);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (kCT >> 5); ++i) s += sm[i];
  return s;  // valid in thread 0
}

struct CoreBox {
  int x0, y0, x1, y1;
};

__device__ __forceinline__ CoreBox core_box(const int* __restrict__ xs, const int* __restrict__ ys,
                                            int ix, int iy) {
  return CoreBox{xs[ix], ys[iy], xs[ix + 1], ys[iy + 1]};
}

// A0 rows of core I = (ix, iy): sum over p in core I of A[p][q] per coarse column (core(q), d).
// Neighbour order of the sums: 0 down (iy-1), 1 left (ix-1), 2 right (ix+1), 3 up (iy+1).
template <int NC>
__global__ void __launch_bounds__(kCT)
    k_coarse_assemble(const double* __restrict__ coef, int W, int H, const int* __restrict__ xs,
                      const int* __restrict__ ys, int px, int py, const int* __restrict__ ccol,
                      const int* __restrict__ crow, int bw, double* __restrict__ AB) {
  __shared__ double sm[32];
  const int I = blockIdx.x, ix = I % px, iy = I / px;
  const CoreBox b = core_box(xs, ys, ix, iy);
  const size_t n = static_cast<size_t>(W) * H;
  const int cw = b.x1 - b.x0, npx = cw * (b.y1 - b.y0);
  double d[NC][NC], nb[4][NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
#pragma unroll
    for (int e = 0; e < NC; ++e) d[c][e] = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) nb[k][c] = 0.0;
  }
  for (int k = threadIdx.x; k < npx; k += kCT) {
    const int x = b.x0 + k % cw, y = b.y0 + k / cw;
    const long long v = static_cast<long long>(y) * W + x;
    // the nodal block (coef planes m11 m12 m13 m22 m23 m33: data block + stiffness diagonal)
    const int plane[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int e = 0; e < NC; ++e) d[c][e] += coef[plane[c][e] * n + v];
    // the four couplings (eh at v: (x,y)-(x+1,y); ev at v: (x,y)-(x,y+1)); alpha weight for
    // u1, u2, lambda weight for mt
    double kk[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    if (y > 0) kk[0][0] = coef[8 * n + v - W], kk[0][1] = coef[9 * n + v - W];
    if (x > 0) kk[1][0] = coef[6 * n + v - 1], kk[1][1] = coef[7 * n + v - 1];
    if (x < W - 1) kk[2][0] = coef[6 * n + v], kk[2][1] = coef[7 * n + v];
    if (y < H - 1) kk[3][0] = coef[8 * n + v], kk[3][1] = coef[9 * n + v];
    const bool out[4] = {y == b.y0 && y > 0, x == b.x0 && x > 0, x == b.x1 - 1 && x < W - 1,
                         y == b.y1 - 1 && y < H - 1};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double w = kk[q][c < 2 ? 0 : 1];
        if (out[q])
          nb[q][c] += w;  // coupling into the neighbouring core
        else
          d[c][c] += w;  // coupling inside the core (or an absent neighbour: w = 0)
      }
  }
  // fixed-order block reductions, thread 0 writes the lower band of the rows of core I
  const int rowI = ccol[b.x0] + crow[b.y0];  // coarse node of core I
  const int ld = bw + 1;
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int e = 0; e < NC; ++e) {
      const double s = block_sum_c(d[c][e], sm);
      if (threadIdx.x == 0 && e <= c) {
        const long long i = static_cast<long long>(rowI) * NC + c, j = static_cast<long long>(rowI) * NC + e;
        AB[i * ld + (j - i + bw)] = s;
      }
    }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double s = block_sum_c(nb[q][c], sm);
      if (threadIdx.x != 0) continue;
      const bool exists = (q == 0 && iy > 0) || (q == 1 && ix > 0) || (q == 2 && ix < px - 1) ||
                          (q == 3 && iy < py - 1);
      if (!exists) continue;
      const int jx = ix + (q == 1 ? -1 : (q == 2 ? 1 : 0));
      const int jy = iy + (q == 0 ? -1 : (q == 3 ? 1 : 0));
      const int rowJ = ccol[xs[jx]] + crow[ys[jy]];
      const long long i = static_cast<long long>(rowI) * NC + c, j = static_cast<long long>(rowJ) * NC + c;
      if (j <= i) AB[i * ld + (j - i + bw)] = s;  // lower band only (A0 symmetric)
    }
}

// column j of A0^-1 = L^-T L^-1 e_j, one warp per column, written to Ainv[j * n0 + :]
__global__ void k_coarse_inverse(int n0, int bw, const double* __restrict__ AB,
                                 double* __restrict__ Ainv) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= n0) return;
  double* x = Ainv + static_cast<long long>(j) * n0;
  const int ld = bw + 1;
  for (int i = lane; i < n0; i += 32) x[i] = 0.0;
  __syncwarp();
  for (int i = j; i < n0; ++i) {  // L y = e_j (y_i = 0 for i < j)
    double s = 0.0;
    for (int k = max(j, i - bw) + lane; k < i; k += 32) s += AB[static_cast<long long>(i) * ld + (k - i + bw)] * x[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(~0u, s, off);
    if (lane == 0) x[i] = ((i == j ? 1.0 : 0.0) - s) / AB[static_cast<long long>(i) * ld + bw];
    __syncwarp();
  }
  for (int i = n0 - 1; i >= 0; --i) {  // L^T x = y
    double s = 0.0;
    for (int k = i + 1 + lane; k <= min(n0 - 1, i + bw); k += 32)
      s += AB[static_cast<long long>(k) * ld + (i - k + bw)] * x[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(~0u, s, off);
    if (lane == 0) x[i] = (x[i] - s) / AB[static_cast<long long>(i) * ld + bw];
    __syncwarp();
  }
}

// g[core I, c] = sum over the core's pixels of r (fixed order per CTA)
template <int NC>
__global__ void __launch_bounds__(kCT)
    k_coarse_restrict(const double* __restrict__ r, int W, const int* __restrict__ xs,
                      const int* __restrict__ ys, int px, const int* __restrict__ ccol,
                      const int* __restrict__ crow, double* __restrict__ g,
                      const PcgCtl* __restrict__ ctl) {
  if (ctl && (ctl->done | ctl->err)) return;
  __shared__ double sm[32];
  const int I = blockIdx.x, ix = I % px, iy = I / px;
  const CoreBox b = core_box(xs, ys, ix, iy);
  const int cw = b.x1 - b.x0, npx = cw * (b.y1 - b.y0);
  double s[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) s[c] = 0.0;
  for (int k = threadIdx.x; k < npx; k += kCT) {
    const long long v = static_cast<long long>(b.y0 + k / cw) * W + b.x0 + k % cw;
#pragma unroll
    for (int c = 0; c < NC; ++c) s[c] += r[v * NC + c];
  }
  const int node = ccol[b.x0] + crow[b.y0];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double t = block_sum_c(s[c], sm);
    if (threadIdx.x == 0) g[node * NC + c] = t;
  }
}

// y = A0^-1 g, one warp per row (A0^-1 symmetric: row i = column i, contiguous)
__global__ void k_coarse_apply(int n0, const double* __restrict__ Ainv, const double* __restrict__ g,
                               double* __restrict__ y, const PcgCtl* __restrict__ ctl) {
  if (ctl && (ctl->done | ctl->err)) return;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n0) return;
  const double* a = Ainv + static_cast<long long>(i) * n0;
  double s = 0.0;
  for (int k = lane; k < n0; k += 32) s += a[k] * g[k];
#pragma unroll
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(~0u, s, off);
  if (lane == 0) y[i] = s;
}

}  // namespace

void coarse_build(const double* coef, int W, int H, int nc, const int* xs, const int* ys, int px,
                  int py, const int* ccol, const int* crow, int bw, double* AB, double* Ainv,
                  int* bad, cudaStream_t st) {
  const int n0 = nc * px * py;
  FFB_CUDA(cudaMemsetAsync(AB, 0, static_cast<size_t>(n0) * (bw + 1) * sizeof(double), st));
  if (nc == 3)
    k_coarse_assemble<3><<<px * py, kCT, 0, st>>>(coef, W, H, xs, ys, px, py, ccol, crow, bw, AB);
  else
    k_coarse_assemble<2><<<px * py, kCT, 0, st>>>(coef, W, H, xs, ys, px, py, ccol, crow, bw, AB);
  FFB_LAUNCHED();
  band_cholesky(n0, bw, AB, bad, st);
  k_coarse_inverse<<<(n0 + 7) / 8, 256, 0, st>>>(n0, bw, AB, Ainv);
  FFB_LAUNCHED();
}

void coarse_apply(const double* r, int W, int nc, const int* xs, const int* ys, int px, int py,
                  const int* ccol, const int* crow, const double* Ainv, double* g, double* y,
                  const PcgCtl* ctl, cudaStream_t st) {
  const int n0 = nc * px * py;
  if (nc == 3)
    k_coarse_restrict<3><<<px * py, kCT, 0, st>>>(r, W, xs, ys, px, ccol, crow, g, ctl);
  else
    k_coarse_restrict<2><<<px * py, kCT, 0, st>>>(r, W, xs, ys, px, ccol, crow, g, ctl);
  FFB_LAUNCHED();
  k_coarse_apply<<<(n0 + 7) / 8, 256, 0, st>>>(n0, Ainv, g, y, ctl);
  FFB_LAUNCHED();
}

}  // namespace ffb
