// K3/K7: the coupled P1 operator of the flow equations, matrix-free on the pixel grid.
//
// assemble() (src/assembly.cpp:32-166) gathers, per free vertex, the P1 stiffness over the
// incident triangles weighted by alpha (u1, u2) or lambda (mt), plus the lumped 3x3 data
// block and load. On the half-pixel triangulation (src/mesh.cpp:30-35) the diagonal-edge
// couplings are exactly zero and each h/v edge couples with -1/2 of the two adjacent
// triangles' weights, so the operator is a weighted 5-point stencil per component plus a
// nodal block. We precompute 10 coefficient planes per vertex (80 B/px) once per alpha and
// apply the operator without a matrix.
//
// Compiled with --fmad=false: coefficients are accumulated in the reference's triangle
// order and the apply sums in its CSR column order (ascending vertex id, the vertex's own
// block in place), so ffb_assemble_apply is bitwise equal to reference spmv(assemble()).
#include "ffb_internal.cuh"

namespace ffb {

namespace {

__device__ __forceinline__ long long tri_lo(int x, int y, int W) {
  return 2LL * (static_cast<long long>(y) * (W - 1) + x);
}

// lumped vertex weight: sum of area/3 over the incident triangles (src/mesh.cpp:122-126)
__device__ __forceinline__ double lumped(int x, int y, int W, int H) {
  int cnt = 0;
  if (x > 0 && y > 0) cnt += 2;
  if (x < W - 1 && y > 0) cnt += 1;
  if (x > 0 && y < H - 1) cnt += 1;
  if (x < W - 1 && y < H - 1) cnt += 2;
  double s = 0.0;
  for (int k = 0; k < cnt; ++k) s += 0.5 / 3.0;
  return s;
}

struct Stencil {
  double diag, down, left, right, up;
};

// Stiffness row of vertex (x,y), triangles in ascending id as assemble() visits them
// (assembly.cpp:114-129): cell(x-1,y-1) lower, upper; cell(x,y-1) upper; cell(x-1,y)
// lower; cell(x,y) lower, upper. area*|grad phi_v|^2 is 1/2 at the two acute vertices of a
// half-pixel triangle and 1 at its right-angle vertex; h/v neighbour pairs give -1/2 and
// the diagonal pair exactly 0 (p1_gradients, src/mesh.cpp:172-186).
__device__ __forceinline__ Stencil stiffness(const double* __restrict__ w, int x, int y, int W,
                                             int H) {
  Stencil s{0.0, 0.0, 0.0, 0.0, 0.0};
  if (x > 0 && y > 0) {
    const double a = w[tri_lo(x - 1, y - 1, W)], b = w[tri_lo(x - 1, y - 1, W) + 1];
    s.diag += a * 0.5;
    s.down += a * -0.5;
    s.diag += b * 0.5;
    s.left += b * -0.5;
  }
  if (x < W - 1 && y > 0) {
    const double b = w[tri_lo(x, y - 1, W) + 1];
    s.diag += b * 1.0;
    s.down += b * -0.5;
    s.right += b * -0.5;
  }
  if (x > 0 && y < H - 1) {
    const double a = w[tri_lo(x - 1, y, W)];
    s.diag += a * 1.0;
    s.left += a * -0.5;
    s.up += a * -0.5;
  }
  if (x < W - 1 && y < H - 1) {
    const double a = w[tri_lo(x, y, W)], b = w[tri_lo(x, y, W) + 1];
    s.diag += a * 0.5;
    s.right += a * -0.5;
    s.diag += b * 0.5;
    s.up += b * -0.5;
  }
  return s;
}

__global__ void k_build_coef(const double* __restrict__ t10, const double* __restrict__ alpha,
                             const double* __restrict__ lambda, int W, int H, int nc,
                             double* __restrict__ coef, int* bad_diag) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= W) return;
  const size_t n = static_cast<size_t>(W) * H;
  const size_t v = static_cast<size_t>(y) * W + x;
  const double wv = lumped(x, y, W, H);
  const Stencil sa = stiffness(alpha, x, y, W, H);
  // nodal_terms (assembly.cpp:19-28) times the lumped weight, stiffness on the diagonal
  const double m11 = wv * t10[0 * n + v] + sa.diag;
  const double m12 = wv * t10[1 * n + v];
  const double m22 = wv * t10[3 * n + v] + sa.diag;
  double m13 = 0.0, m23 = 0.0, m33 = 1.0, ehl = 0.0, evl = 0.0;
  if (nc == 3) {
    const Stencil sl = stiffness(lambda, x, y, W, H);
    m13 = wv * t10[2 * n + v];
    m23 = wv * t10[4 * n + v];
    m33 = wv * t10[5 * n + v] + sl.diag;
    ehl = sl.right;
    evl = sl.up;
  }
  coef[0 * n + v] = m11;
  coef[1 * n + v] = m12;
  coef[2 * n + v] = m13;
  coef[3 * n + v] = m22;
  coef[4 * n + v] = m23;
  coef[5 * n + v] = m33;
  coef[6 * n + v] = sa.right;
  coef[7 * n + v] = ehl;
  coef[8 * n + v] = sa.up;
  coef[9 * n + v] = evl;
  // cg_solve's diagonal check (linsolve.cpp:311-312): first offending scalar row
  if (bad_diag) {
    long long row = -1;
    if (!(m11 > 0.0)) row = static_cast<long long>(v) * nc;
    else if (!(m22 > 0.0)) row = static_cast<long long>(v) * nc + 1;
    else if (nc == 3 && !(m33 > 0.0)) row = static_cast<long long>(v) * nc + 2;
    if (row >= 0) atomicMin(bad_diag, static_cast<int>(row));
  }
}

__global__ void k_build_rhs(const double* __restrict__ t10, int W, int H, int nc,
                            double* __restrict__ b) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= W) return;
  const size_t n = static_cast<size_t>(W) * H;
  const size_t v = static_cast<size_t>(y) * W + x;
  const double wv = lumped(x, y, W, H);
  for (int c = 0; c < nc; ++c) b[v * nc + c] = wv * t10[(6 + c) * n + v];  // assembly.cpp:140
}

// y = A x, one thread per vertex, reference CSR order per scalar row (assembly.cpp:240-249)
__global__ void k_apply(const double* __restrict__ coef, int W, int H, int nc,
                        const double* __restrict__ xs, double* __restrict__ ys) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= W) return;
  const size_t n = static_cast<size_t>(W) * H;
  const long long v = static_cast<long long>(y) * W + x;
  double m[3][3];
  m[0][0] = coef[0 * n + v];
  m[0][1] = m[1][0] = coef[1 * n + v];
  m[0][2] = m[2][0] = coef[2 * n + v];
  m[1][1] = coef[3 * n + v];
  m[1][2] = m[2][1] = coef[4 * n + v];
  m[2][2] = coef[5 * n + v];
  for (int c = 0; c < nc; ++c) {
    const int k = c < 2 ? 0 : 1;
    double s = 0.0;
    if (y > 0) s += coef[(8 + k) * n + v - W] * xs[(v - W) * nc + c];
    if (x > 0) s += coef[(6 + k) * n + v - 1] * xs[(v - 1) * nc + c];
    for (int c2 = 0; c2 < nc; ++c2) s += m[c][c2] * xs[v * nc + c2];
    if (x < W - 1) s += coef[(6 + k) * n + v] * xs[(v + 1) * nc + c];
    if (y < H - 1) s += coef[(8 + k) * n + v] * xs[(v + W) * nc + c];
    ys[v * nc + c] = s;
  }
}

__global__ void k_planes_to_inter(const double* __restrict__ p3, double* __restrict__ x,
                                  long long N, int nc) {
  const long long v = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= N) return;
  for (int c = 0; c < nc; ++c) x[v * nc + c] = p3[c * N + v];
}

__global__ void k_inter_to_planes(const double* __restrict__ x, double* __restrict__ p3,
                                  long long N, int nc) {
  const long long v = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= N) return;
  for (int c = 0; c < nc; ++c) p3[c * N + v] = x[v * nc + c];
  if (nc == 2) p3[2 * N + v] = 0.0;
}

__global__ void k_fill(double* __restrict__ p, double v, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[i] = v;
}

// assemble()'s CSR SparseSystem (assembly.cpp:32-166) from the coefficient planes: one thread
// per free vertex writes its nc rows in the reference's column order — the vertex's mesh
// neighbours ascending (v-W-1, v-W, v-1, own nc x nc block, v+1, v+W, v+W+1; the diagonal
// pair couples with exactly 0.0, mesh.cpp:172-186) — and eliminates constrained neighbours
// into the right-hand side in the same order (assembly.cpp:150-160). Bitwise equal to the
// reference (same values as the matrix-free operator, same subtraction order).
__global__ void k_csr_fill(const double* __restrict__ coef, const double* __restrict__ t10,
                           int W, int H, int nc, int n_free, const int* __restrict__ free_to_vert,
                           const int* __restrict__ vert_to_free, const int* __restrict__ row_ptr,
                           const double* __restrict__ g, int* __restrict__ cols,
                           double* __restrict__ vals, double* __restrict__ rhs) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n_free) return;
  const size_t n = static_cast<size_t>(W) * H;
  const int v = free_to_vert[f];
  const int x = v % W, y = v / W;
  const double wv = lumped(x, y, W, H);
  const int plane[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
  // neighbours ascending: 0 v-W-1, 1 v-W, 2 v-1, (self), 3 v+1, 4 v+W, 5 v+W+1
  const bool has[6] = {x > 0 && y > 0, y > 0, x > 0, x < W - 1, y < H - 1, x < W - 1 && y < H - 1};
  const int nbv[6] = {v - W - 1, v - W, v - 1, v + 1, v + W, v + W + 1};
  for (int c = 0; c < nc; ++c) {
    const int k = c < 2 ? 0 : 1;
    const double st[6] = {0.0, has[1] ? coef[(8 + k) * n + v - W] : 0.0,
                          has[2] ? coef[(6 + k) * n + v - 1] : 0.0,
                          has[3] ? coef[(6 + k) * n + v] : 0.0,
                          has[4] ? coef[(8 + k) * n + v] : 0.0, 0.0};
    const int row = f * nc + c;
    int q = row_ptr[row];
    double r = wv * t10[(6 + c) * n + v];
    for (int a = 0; a < 7; ++a) {
      if (a == 3) {  // the vertex's own block
        for (int c2 = 0; c2 < nc; ++c2) {
          cols[q] = f * nc + c2;
          vals[q] = coef[plane[c][c2] * n + v];
          ++q;
        }
        continue;
      }
      const int e = a < 3 ? a : a - 1;
      if (!has[e]) continue;
      const int w = nbv[e];
      const int fw = vert_to_free[w];
      if (fw >= 0) {
        cols[q] = fw * nc + c;
        vals[q] = st[e];
        ++q;
      } else {
        r -= st[e] * g[static_cast<size_t>(w) * nc + c];
      }
    }
    rhs[row] = r;
  }
}

constexpr int kT = 128;

}  // namespace

void fill(double* p, double v, long long n, cudaStream_t st) {
  k_fill<<<kRedBlocks, 256, 0, st>>>(p, v, n);
  FFB_LAUNCHED();
}

void build_coef(const double* t10, const double* alpha, const double* lambda, int W, int H,
                int nc, double* coef, int* bad_diag, cudaStream_t st) {
  dim3 grid((W + kT - 1) / kT, H);
  k_build_coef<<<grid, kT, 0, st>>>(t10, alpha, lambda, W, H, nc, coef, bad_diag);
  FFB_LAUNCHED();
}

void build_rhs(const double* t10, int W, int H, int nc, double* b, cudaStream_t st) {
  dim3 grid((W + kT - 1) / kT, H);
  k_build_rhs<<<grid, kT, 0, st>>>(t10, W, H, nc, b);
  FFB_LAUNCHED();
}

void apply_op(const double* coef, int W, int H, int nc, const double* x, double* y,
              cudaStream_t st) {
  dim3 grid((W + kT - 1) / kT, H);
  k_apply<<<grid, kT, 0, st>>>(coef, W, H, nc, x, y);
  FFB_LAUNCHED();
}

void planes_to_inter(const double* p3, double* x, long long N, int nc, cudaStream_t st) {
  k_planes_to_inter<<<(N + 255) / 256, 256, 0, st>>>(p3, x, N, nc);
  FFB_LAUNCHED();
}

void inter_to_planes(const double* x, double* p3, long long N, int nc, cudaStream_t st) {
  k_inter_to_planes<<<(N + 255) / 256, 256, 0, st>>>(x, p3, N, nc);
  FFB_LAUNCHED();
}

void csr_fill(const double* coef, const double* t10, int W, int H, int nc, int n_free,
              const int* free_to_vert, const int* vert_to_free, const int* row_ptr,
              const double* g, int* cols, double* vals, double* rhs, cudaStream_t st) {
  if (n_free <= 0) return;
  k_csr_fill<<<(n_free + 127) / 128, 128, 0, st>>>(coef, t10, W, H, nc, n_free, free_to_vert,
                                                   vert_to_free, row_ptr, g, cols, vals, rhs);
  FFB_LAUNCHED();
}

}  // namespace ffb
