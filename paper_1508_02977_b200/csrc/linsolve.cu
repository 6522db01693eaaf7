// The linsolve boundary on the device for an explicit CSR SparseSystem (
// proj/include/flowfem/linsolve.hpp:26-62): spmv, the reference's Jacobi-PCG cg_solve and the
// direct solve() (band Cholesky under the reference's RCM ordering + one refinement step).
//
// Compiled with --fmad=false. cg_solve reproduces the reference's arithmetic bit for bit:
//   * spmv (assembly.cpp:240-249): one thread per row, the row's products summed in CSR order;
//   * det_dot (linsolve.cpp:279-294): fixed 8192-entry chunks, each summed sequentially, the
//     chunk partials summed in chunk order — the products are formed in parallel and staged
//     in shared memory, one thread keeps the sequential sum;
//   * the vector updates and the scalar recurrences in the reference's operation order.
// The CG control flow stays on the device (CgCtl flags, every kernel returns early once the
// iteration has stopped), so the host checks the state once per batch of iterations.
#include "ffb_internal.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>

namespace ffb {

namespace {

constexpr int kDotChunk = 8192;  // linsolve.cpp:282
constexpr int kDotThreads = 256;
constexpr int kDotTile = 2048;

__global__ void k_csr_diag(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ v, double* __restrict__ diag,
                           int* __restrict__ bad_row) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double d = 0.0;
    for (int q = rp[r]; q < rp[r + 1]; ++q)
      if (ci[q] == r) d = v[q];
    diag[r] = d;
    if (!(d > 0.0)) atomicMin(bad_row, r);
  }
}

__global__ void k_csr_spmv(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ v, const double* __restrict__ x,
                           double* __restrict__ y, const CgCtl* __restrict__ ctl) {
  if (ctl && ctl->done) return;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = rp[r]; q < rp[r + 1]; ++q) s += v[q] * x[ci[q]];
    y[r] = s;
  }
}

// partial[c] = sum_{i in chunk c} a[i] b[i], sequentially (one block per chunk)
__global__ void __launch_bounds__(kDotThreads)
    k_dot_chunks(const double* __restrict__ a, const double* __restrict__ b, long long n,
                 double* __restrict__ partial, const CgCtl* __restrict__ ctl) {
  if (ctl && ctl->done) return;
  __shared__ double prod[kDotTile];
  const long long lo = static_cast<long long>(blockIdx.x) * kDotChunk;
  const long long hi = min(n, lo + kDotChunk);
  double s = 0.0;
  for (long long t0 = lo; t0 < hi; t0 += kDotTile) {
    const int m = static_cast<int>(min(static_cast<long long>(kDotTile), hi - t0));
    for (int i = threadIdx.x; i < m; i += kDotThreads) prod[i] = a[t0 + i] * b[t0 + i];
    __syncthreads();
    if (threadIdx.x == 0) {
      int i = 0;
      for (; i + 4 <= m; i += 4) {
        s += prod[i];
        s += prod[i + 1];
        s += prod[i + 2];
        s += prod[i + 3];
      }
      for (; i < m; ++i) s += prod[i];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

enum CgStage { kNormB = 0, kInitRz, kInitRes, kPap, kRes, kRz };

// the scalar part of cg_solve (linsolve.cpp:323-357) after a det_dot
__global__ void k_cg_scalar(const double* __restrict__ partial, int nchunks, int stage,
                            CgCtl* __restrict__ c) {
  if (c->done) return;
  double s = 0.0;
  for (int q = 0; q < nchunks; ++q) s += partial[q];
  switch (stage) {
    case kNormB:
      c->normb = sqrt(s);
      if (c->normb == 0.0) c->done = 1, c->zero = 1;
      break;
    case kInitRz:
      c->rz = s;
      break;
    case kInitRes:
      c->res = sqrt(s) / c->normb;
      if (!(c->res > c->tol && c->it < c->max_iters)) c->done = 1;
      break;
    case kPap:
      ++c->it;
      if (s <= 0.0) {
        c->done = 1, c->err = 2;
        break;
      }
      c->alpha = c->rz / s;
      break;
    case kRes:
      c->res = sqrt(s) / c->normb;
      if (c->res <= c->tol) c->done = 1;
      break;
    case kRz: {
      const double beta = s / c->rz;
      c->beta = beta;
      c->rz = s;
      if (!(c->it < c->max_iters)) c->done = 1;  // res > tol here
      break;
    }
  }
}

__global__ void k_cg_init(int n, const double* __restrict__ b, const double* __restrict__ Ap,
                          const double* __restrict__ diag, double* __restrict__ r,
                          double* __restrict__ z, double* __restrict__ p,
                          const CgCtl* __restrict__ c) {
  if (c->done) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    r[i] = b[i] - Ap[i];
    z[i] = r[i] / diag[i];
    p[i] = z[i];
  }
}

__global__ void k_cg_xr(int n, double* __restrict__ x, double* __restrict__ r,
                        const double* __restrict__ p, const double* __restrict__ Ap,
                        const CgCtl* __restrict__ c) {
  if (c->done) return;
  const double alpha = c->alpha;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    r[i] -= alpha * Ap[i];
  }
}

__global__ void k_cg_z(int n, const double* __restrict__ r, const double* __restrict__ diag,
                       double* __restrict__ z, const CgCtl* __restrict__ c) {
  if (c->done) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    z[i] = r[i] / diag[i];
}

__global__ void k_cg_p(int n, const double* __restrict__ z, double* __restrict__ p,
                       const CgCtl* __restrict__ c) {
  if (c->done) return;
  const double beta = c->beta;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

// ------------------------------------------------------------------ band Cholesky
// Lower band of the RCM-permuted matrix, row-major: AB[i * (bw + 1) + (j - i + bw)], j <= i.
__global__ void k_band_scatter(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                               const double* __restrict__ v, const int* __restrict__ iperm,
                               int bw, double* __restrict__ AB) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int i = iperm[r];
    for (int q = rp[r]; q < rp[r + 1]; ++q) {
      const int j = iperm[ci[q]];
      if (j <= i) AB[static_cast<long long>(i) * (bw + 1) + (j - i + bw)] = v[q];
    }
  }
}

constexpr int kBandThreads = 1024;

// right-looking band Cholesky A = L L^T in place (one CTA; column k scales its band and
// updates the (bw x bw) trailing window). Records the first non-positive pivot.
__global__ void __launch_bounds__(kBandThreads)
    k_band_chol(int n, int bw, double* __restrict__ AB, int* __restrict__ bad) {
  const int ld = bw + 1;
  __shared__ double lcol[1024];
  for (int k = 0; k < n; ++k) {
    __syncthreads();
    const double d = AB[static_cast<long long>(k) * ld + bw];
    if (!(d > 0.0)) {
      if (threadIdx.x == 0) *bad = k;
      return;  // uniform: every thread read the same d
    }
    const double lkk = sqrt(d);
    const int m = min(bw, n - 1 - k);  // rows k+1 .. k+m
    for (int t = threadIdx.x; t < m; t += kBandThreads) {
      const int i = k + 1 + t;
      double* e = AB + static_cast<long long>(i) * ld + (k - i + bw);
      const double l = *e / lkk;
      *e = l;
      lcol[t] = l;
    }
    __syncthreads();
    if (threadIdx.x == 0) AB[static_cast<long long>(k) * ld + bw] = lkk;
    // trailing update: rows i = k+1+a, columns j = k+1+b, b <= a
    const int pairs = m * (m + 1) / 2;
    for (int e = threadIdx.x; e < pairs; e += kBandThreads) {
      int a = static_cast<int>((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (a * (a + 1) / 2 > e) --a;
      while ((a + 1) * (a + 2) / 2 <= e) ++a;
      const int b = e - a * (a + 1) / 2;
      const int i = k + 1 + a, j = k + 1 + b;
      AB[static_cast<long long>(i) * ld + (j - i + bw)] -= lcol[a] * lcol[b];
    }
  }
}

// x <- L^-T L^-1 x in place (one CTA): forward and backward substitution, one row at a time
// with a block reduction of its band
__global__ void __launch_bounds__(256)
    k_band_solve(int n, int bw, const double* __restrict__ AB, double* __restrict__ x) {
  const int ld = bw + 1;
  __shared__ double red[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = 0; i < n; ++i) {  // L y = b
    double s = 0.0;
    for (int j = max(0, i - bw) + threadIdx.x; j < i; j += 256)
      s += AB[static_cast<long long>(i) * ld + (j - i + bw)] * x[j];
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(~0u, s, off);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      x[i] = (x[i] - t) / AB[static_cast<long long>(i) * ld + bw];
    }
    __syncthreads();
  }
  for (int i = n - 1; i >= 0; --i) {  // L^T x = y
    double s = 0.0;
    for (int j = i + 1 + threadIdx.x; j <= min(n - 1, i + bw); j += 256)
      s += AB[static_cast<long long>(j) * ld + (i - j + bw)] * x[j];
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(~0u, s, off);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      x[i] = (x[i] - t) / AB[static_cast<long long>(i) * ld + bw];
    }
    __syncthreads();
  }
}

__global__ void k_gather(int n, const int* __restrict__ idx, const double* __restrict__ src,
                         double* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}
__global__ void k_scatter_add(int n, const int* __restrict__ idx, const double* __restrict__ src,
                              double* __restrict__ dst, int add) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[idx[i]] = add ? dst[idx[i]] + src[i] : src[i];
}
__global__ void k_sub(int n, const double* __restrict__ b, const double* __restrict__ y,
                      double* __restrict__ r) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    r[i] = b[i] - y[i];
}
// solve()'s report (linsolve.cpp:389-397): sqrt(rn / bn), both sums in row order
__global__ void k_residual_report(int n, const double* __restrict__ b,
                                  const double* __restrict__ Ax, double* __restrict__ out) {
  double rn = 0.0, bn = 0.0;
  for (int i = 0; i < n; ++i) {
    const double d = b[i] - Ax[i];
    rn += d * d;
    bn += b[i] * b[i];
  }
  *out = bn > 0 ? sqrt(rn / bn) : 0.0;
}

int grid_for(long long n, int threads) {
  return static_cast<int>(std::min<long long>(std::max<long long>((n + threads - 1) / threads, 1),
                                              4LL * 148 * 8));
}

}  // namespace

// ---------------------------------------------------------------------------- host side
void csr_spmv(const CsrDev& A, const double* x, double* y, const CgCtl* ctl, cudaStream_t st) {
  k_csr_spmv<<<grid_for(A.n, 256), 256, 0, st>>>(A.n, A.rp, A.ci, A.v, x, y, ctl);
  FFB_LAUNCHED();
}

void csr_diag(const CsrDev& A, double* diag, int* bad_row, cudaStream_t st) {
  k_csr_diag<<<grid_for(A.n, 256), 256, 0, st>>>(A.n, A.rp, A.ci, A.v, diag, bad_row);
  FFB_LAUNCHED();
}

int dot_chunks(long long n) { return static_cast<int>(std::max<long long>((n + kDotChunk - 1) / kDotChunk, 1)); }

void det_dot(const double* a, const double* b, long long n, double* partial, const CgCtl* ctl,
             cudaStream_t st) {
  k_dot_chunks<<<dot_chunks(n), kDotThreads, 0, st>>>(a, b, n, partial, ctl);
  FFB_LAUNCHED();
}

void cg_scalar(const double* partial, long long n, int stage, CgCtl* ctl, cudaStream_t st) {
  k_cg_scalar<<<1, 1, 0, st>>>(partial, n > 0 ? dot_chunks(n) : 0, stage, ctl);
  FFB_LAUNCHED();
}

void cg_init(int n, const double* b, const double* Ap, const double* diag, double* r, double* z,
             double* p, const CgCtl* c, cudaStream_t st) {
  k_cg_init<<<grid_for(n, 256), 256, 0, st>>>(n, b, Ap, diag, r, z, p, c);
  FFB_LAUNCHED();
}

// one CG iteration (linsolve.cpp:330-357), every kernel a no-op once the iteration stopped
void cg_iteration(const CsrDev& A, double* x, double* r, double* z, double* p, double* Ap,
                  const double* diag, double* partial, CgCtl* c, cudaStream_t st) {
  const int n = A.n;
  csr_spmv(A, p, Ap, c, st);
  det_dot(p, Ap, n, partial, c, st);
  cg_scalar(partial, n, kPap, c, st);
  k_cg_xr<<<grid_for(n, 256), 256, 0, st>>>(n, x, r, p, Ap, c);
  FFB_LAUNCHED();
  det_dot(r, r, n, partial, c, st);
  cg_scalar(partial, n, kRes, c, st);
  k_cg_z<<<grid_for(n, 256), 256, 0, st>>>(n, r, diag, z, c);
  FFB_LAUNCHED();
  det_dot(r, z, n, partial, c, st);
  cg_scalar(partial, n, kRz, c, st);
  k_cg_p<<<grid_for(n, 256), 256, 0, st>>>(n, z, p, c);
  FFB_LAUNCHED();
}

int cg_stage_normb() { return kNormB; }
int cg_stage_init_rz() { return kInitRz; }
int cg_stage_init_res() { return kInitRes; }

void band_scatter(const CsrDev& A, const int* iperm, int bw, double* AB, cudaStream_t st) {
  k_band_scatter<<<grid_for(A.n, 256), 256, 0, st>>>(A.n, A.rp, A.ci, A.v, iperm, bw, AB);
  FFB_LAUNCHED();
}

void band_cholesky(int n, int bw, double* AB, int* bad, cudaStream_t st) {
  if (bw > 1024) fail("linsolve.cholesky: band width " + std::to_string(bw) + " exceeds 1024");
  k_band_chol<<<1, kBandThreads, 0, st>>>(n, bw, AB, bad);
  FFB_LAUNCHED();
}

void band_solve(int n, int bw, const double* AB, double* x, cudaStream_t st) {
  k_band_solve<<<1, 256, 0, st>>>(n, bw, AB, x);
  FFB_LAUNCHED();
}

void gather(int n, const int* idx, const double* src, double* dst, cudaStream_t st) {
  k_gather<<<grid_for(n, 256), 256, 0, st>>>(n, idx, src, dst);
  FFB_LAUNCHED();
}

void scatter(int n, const int* idx, const double* src, double* dst, bool add, cudaStream_t st) {
  k_scatter_add<<<grid_for(n, 256), 256, 0, st>>>(n, idx, src, dst, add ? 1 : 0);
  FFB_LAUNCHED();
}

void vec_sub(int n, const double* b, const double* y, double* r, cudaStream_t st) {
  k_sub<<<grid_for(n, 256), 256, 0, st>>>(n, b, y, r);
  FFB_LAUNCHED();
}

void residual_report(int n, const double* b, const double* Ax, double* out, cudaStream_t st) {
  k_residual_report<<<1, 1, 0, st>>>(n, b, Ax, out);
  FFB_LAUNCHED();
}

}  // namespace ffb
