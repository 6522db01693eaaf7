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

}  // namespace ffb
