// The reference's own Schwarz loop on the device: the synchronous
// restricted-additive-Schwarz iteration of schwarz_solve (src/schwarz.cpp:162-319),
//   G_{k+1}[core_i] = ( A_i^-1 (R_i b - A_{i,ring} G_k[ring_i]) )[core_i],
// with the subdomain factors of band.cu, one step of iterative refinement as the
// reference's Cholesky path does (schwarz.cpp:242-247), the max-norm increment
// (schwarz.cpp:294-300) and the interleaved alpha update (schwarz.cpp:303-311, host side).
//
// Compiled with --fmad=false: the right-hand side and the refinement residual are formed in
// the reference's assembly/spmv operation order.
#include "ffb_internal.cuh"

namespace ffb {

namespace {

__device__ __forceinline__ void local_coords(const SubInfo& s, int k, int nc, int& lx, int& ly,
                                             int& c) {
  const int l = k / s.kd, j = k - l * s.kd;
  const int a = j / nc;
  c = j - a * nc;
  lx = s.xfast ? a : l;
  ly = s.xfast ? l : a;
}

__device__ __forceinline__ long long local_index(const SubInfo& s, int lx, int ly, int c,
                                                 int nc) {
  const long long vloc = s.xfast ? static_cast<long long>(ly) * s.fw + lx
                                 : static_cast<long long>(lx) * s.fh + ly;
  return vloc * nc + c;
}

// rhs_i = R_i b - A_{i, ring} G: the Dirichlet elimination of assemble() (assembly.cpp:
// 150-160) — couplings to ring vertices in ascending vertex order (down, left, right, up)
__global__ void k_ras_rhs(const SubInfo* __restrict__ subs, const double* __restrict__ coef,
                          const double* __restrict__ b, const double* __restrict__ G, size_t N,
                          int W, int H, int nc, double* __restrict__ rl) {
  const SubInfo s = subs[blockIdx.y];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < s.n; k += gridDim.x * blockDim.x) {
    int lx, ly, c;
    local_coords(s, k, nc, lx, ly, c);
    const int gx = s.fx0 + lx, gy = s.fy0 + ly;
    const long long v = static_cast<long long>(gy) * W + gx;
    const int kk = c < 2 ? 0 : 1;
    double val = b[v * nc + c];
    if (gy > 0 && ly == 0) val -= coef[(8 + kk) * N + v - W] * G[(v - W) * nc + c];
    if (gx > 0 && lx == 0) val -= coef[(6 + kk) * N + v - 1] * G[(v - 1) * nc + c];
    if (gx < W - 1 && lx == s.fw - 1) val -= coef[(6 + kk) * N + v] * G[(v + 1) * nc + c];
    if (gy < H - 1 && ly == s.fh - 1) val -= coef[(8 + kk) * N + v] * G[(v + W) * nc + c];
    rl[s.vec_off + k] = val;
  }
}

// res = rhs - A_i x in the reference CSR order (spmv, assembly.cpp:240-249)
__global__ void k_ras_residual(const SubInfo* __restrict__ subs, const double* __restrict__ coef,
                               size_t N, int W, int nc, const double* __restrict__ rl,
                               const double* __restrict__ xl, double* __restrict__ res) {
  const SubInfo s = subs[blockIdx.y];
  const double* x = xl + s.vec_off;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < s.n; k += gridDim.x * blockDim.x) {
    int lx, ly, c;
    local_coords(s, k, nc, lx, ly, c);
    const int gx = s.fx0 + lx, gy = s.fy0 + ly;
    const long long v = static_cast<long long>(gy) * W + gx;
    const int kk = c < 2 ? 0 : 1;
    double acc = 0.0;
    if (ly > 0) acc += coef[(8 + kk) * N + v - W] * x[local_index(s, lx, ly - 1, c, nc)];
    if (lx > 0) acc += coef[(6 + kk) * N + v - 1] * x[local_index(s, lx - 1, ly, c, nc)];
    const int base = static_cast<int>(local_index(s, lx, ly, 0, nc));
    for (int c2 = 0; c2 < nc; ++c2) {
      const int lo = c < c2 ? c : c2, hi = c < c2 ? c2 : c;
      const int plane = lo == hi ? (lo == 0 ? 0 : (lo == 1 ? 3 : 5))
                                 : (lo + hi == 1 ? 1 : (lo + hi == 2 ? 2 : 4));
      acc += coef[plane * N + v] * x[base + c2];
    }
    if (lx < s.fw - 1) acc += coef[(6 + kk) * N + v] * x[local_index(s, lx + 1, ly, c, nc)];
    if (ly < s.fh - 1) acc += coef[(8 + kk) * N + v] * x[local_index(s, lx, ly + 1, c, nc)];
    res[s.vec_off + k] = rl[s.vec_off + k] - acc;
  }
}

__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }

// G_new[core_i] = (x_i + dx_i)[core_i]; increment = max |G_new - G| (schwarz.cpp:255-300)
__global__ void k_ras_compose(const int* __restrict__ own_col, const int* __restrict__ own_row,
                              const SubInfo* __restrict__ subs, int px,
                              const double* __restrict__ xl, const double* __restrict__ dl,
                              const double* __restrict__ G, double* __restrict__ Gnew, int W,
                              int H, int nc, double* __restrict__ blockmax,
                              double* __restrict__ inc_out, unsigned* __restrict__ counter) {
  const long long N = static_cast<long long>(W) * H;
  double m = 0.0;
  for (long long v = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; v < N;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int x = static_cast<int>(v % W), y = static_cast<int>(v / W);
    const SubInfo& s = subs[own_row[y] * px + own_col[x]];
    for (int c = 0; c < nc; ++c) {
      const long long idx = s.vec_off + local_index(s, x - s.fx0, y - s.fy0, c, nc);
      double g = xl[idx];
      if (dl) g += dl[idx];
      Gnew[v * nc + c] = g;
      m = dmax(m, fabs(g - G[v * nc + c]));
    }
  }
  __shared__ double sm[32];
  for (int off = 16; off; off >>= 1) m = dmax(m, __shfl_xor_sync(~0u, m, off));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) mm = dmax(mm, sm[w]);
    blockmax[blockIdx.x] = mm;
    __threadfence();
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      double t = 0.0;
      for (unsigned b2 = 0; b2 < gridDim.x; ++b2) t = dmax(t, __ldcg(blockmax + b2));
      *inc_out = t;
      *counter = 0;
    }
  }
}

__global__ void k_copy(double* __restrict__ d, const double* __restrict__ s, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    d[i] = s[i];
}

// ---- CG subdomain solves (SolveMethod::ConjugateGradient, schwarz.cpp:248-252) -------------
// Every subdomain runs the reference's Jacobi-PCG cg_solve (linsolve.cpp:298-361) on its
// Dirichlet system, all subdomains in lockstep (blockIdx.y = subdomain), each with its own
// control block; a subdomain that has stopped skips the remaining kernels. The vectors are
// kept in the reference's unknown order (free vertices row-major over the free rectangle,
// component minor — assemble()'s numbering of the subdomain mesh, assembly.cpp:44-60), so
// det_dot's 8192-entry chunks (linsolve.cpp:279-294) and the CSR row order of spmv
// (assembly.cpp:240-249) are reproduced exactly: bitwise equal to the reference.
constexpr int kBChunk = 8192;
constexpr int kBTile = 2048;
constexpr int kBThreads = 256;

__device__ __forceinline__ int diag_plane(int c) { return c == 0 ? 0 : (c == 1 ? 3 : 5); }

// line-major (solve layout) <-> reference order
__global__ void k_bperm(const SubInfo* __restrict__ subs, int nc, const double* __restrict__ src,
                        double* __restrict__ dst, int to_ref) {
  const SubInfo s = subs[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const int f = i / nc, c = i - f * nc;
    const int ly = f / s.fw, lx = f - ly * s.fw;
    const long long li = s.vec_off + local_index(s, lx, ly, c, nc);
    if (to_ref)
      dst[s.vec_off + i] = src[li];
    else
      dst[li] = src[s.vec_off + i];
  }
}

// y = A_i x, rows in CSR column order (down, left, own components, right, up)
__global__ void k_bspmv(const SubInfo* __restrict__ subs, const double* __restrict__ coef,
                        size_t N, int W, int nc, const double* __restrict__ xr,
                        double* __restrict__ yr, const CgCtl* __restrict__ ctl) {
  if (ctl[blockIdx.y].done) return;
  const SubInfo s = subs[blockIdx.y];
  const double* x = xr + s.vec_off;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const int f = i / nc, c = i - f * nc;
    const int ly = f / s.fw, lx = f - ly * s.fw;
    const long long v = static_cast<long long>(s.fy0 + ly) * W + (s.fx0 + lx);
    const int kk = c < 2 ? 0 : 1;
    double acc = 0.0;
    if (ly > 0) acc += coef[(8 + kk) * N + v - W] * x[(f - s.fw) * nc + c];
    if (lx > 0) acc += coef[(6 + kk) * N + v - 1] * x[(f - 1) * nc + c];
    for (int c2 = 0; c2 < nc; ++c2) {
      const int lo = c < c2 ? c : c2, hi = c < c2 ? c2 : c;
      const int plane = lo == hi ? diag_plane(lo) : (lo + hi == 1 ? 1 : (lo + hi == 2 ? 2 : 4));
      acc += coef[plane * N + v] * x[f * nc + c2];
    }
    if (lx < s.fw - 1) acc += coef[(6 + kk) * N + v] * x[(f + 1) * nc + c];
    if (ly < s.fh - 1) acc += coef[(8 + kk) * N + v] * x[(f + s.fw) * nc + c];
    yr[s.vec_off + i] = acc;
  }
}

// partial[sub * maxch + chunk] = sequential sum of a*b over the chunk (det_dot)
__global__ void __launch_bounds__(kBThreads)
    k_bdot(const SubInfo* __restrict__ subs, const double* __restrict__ a,
           const double* __restrict__ b, int maxch, double* __restrict__ partial,
           const CgCtl* __restrict__ ctl) {
  if (ctl[blockIdx.y].done) return;
  const SubInfo s = subs[blockIdx.y];
  const int lo = blockIdx.x * kBChunk;
  if (lo >= s.n) return;
  const int hi = min(s.n, lo + kBChunk);
  __shared__ double prod[kBTile];
  double acc = 0.0;
  for (int t0 = lo; t0 < hi; t0 += kBTile) {
    const int m = min(kBTile, hi - t0);
    for (int i = threadIdx.x; i < m; i += kBThreads)
      prod[i] = a[s.vec_off + t0 + i] * b[s.vec_off + t0 + i];
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < m; ++i) acc += prod[i];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[static_cast<long long>(blockIdx.y) * maxch + blockIdx.x] = acc;
}

enum BStage { kBNormB = 0, kBInitRz, kBInitRes, kBPap, kBRes, kBRz };

__global__ void k_bscalar(const SubInfo* __restrict__ subs, int nsub, const double* __restrict__ partial,
                          int maxch, int stage, CgCtl* __restrict__ ctl) {
  const int sub = blockIdx.x * blockDim.x + threadIdx.x;
  if (sub >= nsub) return;
  CgCtl* c = ctl + sub;
  if (c->done) return;
  const int nch = (subs[sub].n + kBChunk - 1) / kBChunk;
  double s = 0.0;
  for (int q = 0; q < nch; ++q) s += partial[static_cast<long long>(sub) * maxch + q];
  switch (stage) {
    case kBNormB:
      c->normb = sqrt(s);
      if (c->normb == 0.0) c->done = 1, c->zero = 1;
      break;
    case kBInitRz:
      c->rz = s;
      break;
    case kBInitRes:
      c->res = sqrt(s) / c->normb;
      if (!(c->res > c->tol && c->it < c->max_iters)) c->done = 1;
      break;
    case kBPap:
      ++c->it;
      if (s <= 0.0) {
        c->done = 1, c->err = 2;
        break;
      }
      c->alpha = c->rz / s;
      break;
    case kBRes:
      c->res = sqrt(s) / c->normb;
      if (c->res <= c->tol) c->done = 1;
      break;
    case kBRz:
      c->beta = s / c->rz;
      c->rz = s;
      if (!(c->it < c->max_iters)) c->done = 1;
      break;
  }
}

// r = b - Ap, z = r / diag, p = z (linsolve.cpp:323-328)
__global__ void k_binit(const SubInfo* __restrict__ subs, const double* __restrict__ coef, size_t N,
                        int W, int nc, const double* __restrict__ b, const double* __restrict__ Ap,
                        double* __restrict__ r, double* __restrict__ z, double* __restrict__ p,
                        const CgCtl* __restrict__ ctl) {
  if (ctl[blockIdx.y].done) return;
  const SubInfo s = subs[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const int f = i / nc, c = i - f * nc;
    const int ly = f / s.fw, lx = f - ly * s.fw;
    const long long v = static_cast<long long>(s.fy0 + ly) * W + (s.fx0 + lx);
    const long long k = s.vec_off + i;
    r[k] = b[k] - Ap[k];
    z[k] = r[k] / coef[diag_plane(c) * N + v];
    p[k] = z[k];
  }
}

// stage 0: x += alpha p, r -= alpha Ap; stage 1: z = r / diag; stage 2: p = z + beta p
__global__ void k_bvec(const SubInfo* __restrict__ subs, const double* __restrict__ coef, size_t N,
                       int W, int nc, int stage, double* __restrict__ x, double* __restrict__ r,
                       double* __restrict__ z, double* __restrict__ p,
                       const double* __restrict__ Ap, const CgCtl* __restrict__ ctl) {
  const CgCtl& c = ctl[blockIdx.y];
  if (c.done) return;
  const SubInfo s = subs[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x) {
    const long long k = s.vec_off + i;
    if (stage == 0) {
      x[k] += c.alpha * p[k];
      r[k] -= c.alpha * Ap[k];
    } else if (stage == 1) {
      const int f = i / nc, cc = i - f * nc;
      const int ly = f / s.fw, lx = f - ly * s.fw;
      const long long v = static_cast<long long>(s.fy0 + ly) * W + (s.fx0 + lx);
      z[k] = r[k] / coef[diag_plane(cc) * N + v];
    } else {
      p[k] = z[k] + c.beta * p[k];
    }
  }
}

// a zero right-hand side returns the zero vector (linsolve.cpp:318-321)
__global__ void k_bzero(const SubInfo* __restrict__ subs, double* __restrict__ x,
                        const CgCtl* __restrict__ ctl) {
  if (!ctl[blockIdx.y].zero) return;
  const SubInfo s = subs[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += gridDim.x * blockDim.x)
    x[s.vec_off + i] = 0.0;
}

__global__ void k_bctl_init(CgCtl* ctl, const SubInfo* __restrict__ subs, int nsub, double tol,
                            long long max_iters) {
  const int sub = blockIdx.x * blockDim.x + threadIdx.x;
  if (sub >= nsub) return;
  CgCtl c{};
  c.tol = tol;
  c.max_iters = max_iters > 0 ? max_iters : 10LL * subs[sub].n;
  ctl[sub] = c;
}

}  // namespace

void ras_rhs(const SubInfo* d_subs, int nsub, const double* coef, const double* b,
             const double* G, size_t N, int W, int H, int nc, double* rl, cudaStream_t st) {
  k_ras_rhs<<<dim3(64, nsub), 256, 0, st>>>(d_subs, coef, b, G, N, W, H, nc, rl);
  FFB_LAUNCHED();
}

void ras_residual(const SubInfo* d_subs, int nsub, const double* coef, size_t N, int W, int nc,
                  const double* rl, const double* xl, double* res, cudaStream_t st) {
  k_ras_residual<<<dim3(64, nsub), 256, 0, st>>>(d_subs, coef, N, W, nc, rl, xl, res);
  FFB_LAUNCHED();
}

void ras_compose(const int* own_col, const int* own_row, const SubInfo* d_subs, int px,
                 const double* xl, const double* dl, const double* G, double* Gnew, int W, int H,
                 int nc, double* blockmax, double* inc_out, unsigned* counter, cudaStream_t st) {
  k_ras_compose<<<kRedBlocks, kRedThreads, 0, st>>>(own_col, own_row, d_subs, px, xl, dl, G, Gnew,
                                                     W, H, nc, blockmax, inc_out, counter);
  FFB_LAUNCHED();
}

void vec_copy(double* dst, const double* src, long long n, cudaStream_t st) {
  k_copy<<<kRedBlocks, 256, 0, st>>>(dst, src, n);
  FFB_LAUNCHED();
}

void ras_perm(const SubInfo* d_subs, int nsub, int nc, const double* src, double* dst, int to_ref,
              cudaStream_t st) {
  k_bperm<<<dim3(64, nsub), 256, 0, st>>>(d_subs, nc, src, dst, to_ref);
  FFB_LAUNCHED();
}

int ras_cg_chunks(int max_n) { return (max_n + kBChunk - 1) / kBChunk; }

void ras_cg_begin(const SubInfo* d_subs, int nsub, int maxch, const double* coef, size_t N, int W,
                  int nc, double tol, long long max_iters, const double* b, double* x, double* r,
                  double* z, double* p, double* Ap, double* partial, CgCtl* ctl, cudaStream_t st) {
  const dim3 g(64, nsub), gd(maxch, nsub);
  const int sb = (nsub + 127) / 128;
  k_bctl_init<<<sb, 128, 0, st>>>(ctl, d_subs, nsub, tol, max_iters);
  k_bdot<<<gd, kBThreads, 0, st>>>(d_subs, b, b, maxch, partial, ctl);
  k_bscalar<<<sb, 128, 0, st>>>(d_subs, nsub, partial, maxch, kBNormB, ctl);
  k_bspmv<<<g, 256, 0, st>>>(d_subs, coef, N, W, nc, x, Ap, ctl);
  k_binit<<<g, 256, 0, st>>>(d_subs, coef, N, W, nc, b, Ap, r, z, p, ctl);
  k_bdot<<<gd, kBThreads, 0, st>>>(d_subs, r, z, maxch, partial, ctl);
  k_bscalar<<<sb, 128, 0, st>>>(d_subs, nsub, partial, maxch, kBInitRz, ctl);
  k_bdot<<<gd, kBThreads, 0, st>>>(d_subs, r, r, maxch, partial, ctl);
  k_bscalar<<<sb, 128, 0, st>>>(d_subs, nsub, partial, maxch, kBInitRes, ctl);
  ffb::note_launch(8);
  FFB_CUDA(cudaPeekAtLastError());
}

void ras_cg_iterations(const SubInfo* d_subs, int nsub, int maxch, const double* coef, size_t N,
                       int W, int nc, int k, double* x, double* r, double* z, double* p,
                       double* Ap, double* partial, CgCtl* ctl, cudaStream_t st) {
  const dim3 g(64, nsub), gd(maxch, nsub);
  const int sb = (nsub + 127) / 128;
  for (int it = 0; it < k; ++it) {
    k_bspmv<<<g, 256, 0, st>>>(d_subs, coef, N, W, nc, p, Ap, ctl);
    k_bdot<<<gd, kBThreads, 0, st>>>(d_subs, p, Ap, maxch, partial, ctl);
    k_bscalar<<<sb, 128, 0, st>>>(d_subs, nsub, partial, maxch, kBPap, ctl);
    k_bvec<<<g, 256, 0, st>>>(d_subs, coef, N, W, nc, 0, x, r, z, p, Ap, ctl);
    k_bdot<<<gd, kBThreads, 0, st>>>(d_subs, r, r, maxch, partial, ctl);
    k_bscalar<<<sb, 128, 0, st>>>(d_subs, nsub, partial, maxch, kBRes, ctl);
    k_bvec<<<g, 256, 0, st>>>(d_subs, coef, N, W, nc, 1, x, r, z, p, Ap, ctl);
    k_bdot<<<gd, kBThreads, 0, st>>>(d_subs, r, z, maxch, partial, ctl);
    k_bscalar<<<sb, 128, 0, st>>>(d_subs, nsub, partial, maxch, kBRz, ctl);
    k_bvec<<<g, 256, 0, st>>>(d_subs, coef, N, W, nc, 2, x, r, z, p, Ap, ctl);
  }
  ffb::note_launch(10LL * k);
  FFB_CUDA(cudaPeekAtLastError());
}

void ras_cg_zero(const SubInfo* d_subs, int nsub, double* x, const CgCtl* ctl, cudaStream_t st) {
  k_bzero<<<dim3(64, nsub), 256, 0, st>>>(d_subs, x, ctl);
  FFB_LAUNCHED();
}

}  // namespace ffb
