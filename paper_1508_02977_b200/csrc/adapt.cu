// K9/K10: residual-based error indicator and the multiplicative alpha update of the
// adaptive loop (src/adapt.cpp:9-112).
//
// One thread per pixel cell computes eta for both of its triangles. Triangle gradients
// (adapt.cpp:17-36) are recomputed on the fly from the 8 vertices a cell and its four
// edge-neighbours touch, instead of being materialised (48 B per triangle saved); every
// edge term (adapt.cpp:38-64) is evaluated with the reference's t0/t1 orientation and
// expression order. Compiled with --fmad=false, so eta is bitwise equal to the reference.
// eta_max is a max-reduction (order-free) finished by the last CTA.
#include "ffb_internal.cuh"

namespace ffb {

namespace {

// P1 gradients of the two half-pixel triangle shapes, local vertex order of
// src/mesh.cpp:30-35 (p1_gradients, mesh.cpp:172-186)
__device__ const double GX_LO[3] = {-1.0, 1.0, -0.0}, GY_LO[3] = {0.0, -1.0, 1.0};
__device__ const double GX_UP[3] = {-0.0, 1.0, -1.0}, GY_UP[3] = {-1.0, 0.0, 1.0};

struct Grad {
  double g[6];  // d/dx u1, d/dy u1, d/dx u2, d/dy u2, d/dx mt, d/dy mt
};

// gradient of triangle `up` of cell (x,y) (adapt.cpp:18-36)
__device__ __forceinline__ Grad tri_grad(const double* __restrict__ u1,
                                         const double* __restrict__ u2,
                                         const double* __restrict__ mt, int W, int x, int y,
                                         int up, int nc) {
  const long long v00 = static_cast<long long>(y) * W + x;
  long long v[3];
  if (!up) {
    v[0] = v00, v[1] = v00 + 1, v[2] = v00 + W + 1;
  } else {
    v[0] = v00, v[1] = v00 + W + 1, v[2] = v00 + W;
  }
  const double* gx = up ? GX_UP : GX_LO;
  const double* gy = up ? GY_UP : GY_LO;
  Grad G;
#pragma unroll
  for (int i = 0; i < 6; ++i) G.g[i] = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double a = u1[v[k]], b = u2[v[k]];
    G.g[0] += gx[k] * a;
    G.g[1] += gy[k] * a;
    G.g[2] += gx[k] * b;
    G.g[3] += gy[k] * b;
    if (nc == 3) {
      const double m = mt[v[k]];
      G.g[4] += gx[k] * m;
      G.g[5] += gy[k] * m;
    }
  }
  return G;
}

// edge term (adapt.cpp:41-63): t1 < 0 marks a boundary edge
__device__ __forceinline__ double edge_term(const Grad& g0, double a0, double l0, const Grad* g1,
                                            double a1, double l1, double nx, double ny,
                                            double len, int nc) {
  double sum = 0.0;
  for (int c = 0; c < nc; ++c) {
    const double k0 = c < 2 ? a0 : l0;
    const double flux0 = k0 * (g0.g[2 * c] * nx + g0.g[2 * c + 1] * ny);
    double jump, coef_e;
    if (g1) {
      const double k1 = c < 2 ? a1 : l1;
      const double flux1 = k1 * (g1->g[2 * c] * nx + g1->g[2 * c + 1] * ny);
      jump = flux0 - flux1;
      coef_e = (k0 < k1) ? k1 : k0;  // std::max
    } else {
      jump = flux0;
      coef_e = k0;
    }
    sum += jump * jump / coef_e;
  }
  return len * sqrt(sum);
}

__device__ __forceinline__ double elem_part(const double* __restrict__ t10, size_t n,
                                            const double* __restrict__ u1,
                                            const double* __restrict__ u2,
                                            const double* __restrict__ mt, const long long v[3],
                                            double alpha, double lambda, int nc) {
  // adapt.cpp:71-90
  double R[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const long long q = v[k];
    const double U0 = u1[q], U1 = u2[q], U2 = nc == 3 ? mt[q] : 0.0;
    const double a13 = nc == 3 ? t10[2 * n + q] : 0.0;
    const double a23 = nc == 3 ? t10[4 * n + q] : 0.0;
    R[0][k] = t10[6 * n + q] - (t10[0 * n + q] * U0 + t10[1 * n + q] * U1 + a13 * U2);
    R[1][k] = t10[7 * n + q] - (t10[1 * n + q] * U0 + t10[3 * n + q] * U1 + a23 * U2);
    R[2][k] = nc == 3 ? t10[8 * n + q] - (t10[2 * n + q] * U0 + t10[4 * n + q] * U1 +
                                          t10[5 * n + q] * U2)
                      : 0.0;
  }
  double elem = 0.0;
  for (int c = 0; c < nc; ++c) {
    const double s = R[c][0] + R[c][1] + R[c][2];
    const double sq = R[c][0] * R[c][0] + R[c][1] * R[c][1] + R[c][2] * R[c][2];
    const double l2 = 0.5 / 12.0 * (s * s + sq);
    elem += l2 / (c < 2 ? alpha : lambda);
  }
  return elem;
}

__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }

__global__ void k_indicator(const double* __restrict__ t10, const double* __restrict__ alpha,
                            const double* __restrict__ lambda, const double* __restrict__ u3,
                            int W, int H, int nc, double* __restrict__ eta,
                            double* __restrict__ blockmax, double* __restrict__ eta_max_out,
                            unsigned* __restrict__ counter) {
  const int cw = W - 1, ch = H - 1;
  const size_t n = static_cast<size_t>(W) * H;
  const double* u1 = u3;
  const double* u2 = u3 + n;
  const double* mt = u3 + 2 * n;
  const double inv_sqrt2 = 1.0 / sqrt(2.0);
  const double hK = sqrt(2.0);
  double local_max = 0.0;
  const long long ncell = static_cast<long long>(cw) * ch;
  for (long long cell = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       cell < ncell; cell += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int x = static_cast<int>(cell % cw), y = static_cast<int>(cell / cw);
    const long long tlo = 2 * cell, tup = tlo + 1;
    const Grad gl = tri_grad(u1, u2, mt, W, x, y, 0, nc);
    const Grad gu = tri_grad(u1, u2, mt, W, x, y, 1, nc);
    const double al = alpha[tlo], ll = lambda[tlo], au = alpha[tup], lu = lambda[tup];
    // diagonal edge: t0 = lower, t1 = upper, n = (-1/sqrt2, 1/sqrt2), length sqrt2
    const double e_diag = edge_term(gl, al, ll, &gu, au, lu, -inv_sqrt2, inv_sqrt2, sqrt(2.0), nc);
    // bottom h-edge of the cell: below = upper of cell (x,y-1), above = lower (this cell)
    double e_bot;
    if (y > 0) {
      const long long tb = 2 * (cell - cw) + 1;
      const Grad gb = tri_grad(u1, u2, mt, W, x, y - 1, 1, nc);
      e_bot = edge_term(gb, alpha[tb], lambda[tb], &gl, al, ll, 0.0, 1.0, 1.0, nc);
    } else {
      e_bot = edge_term(gl, al, ll, nullptr, 0.0, 0.0, 0.0, -1.0, 1.0, nc);
    }
    // top h-edge: below = upper (this cell), above = lower of cell (x,y+1)
    double e_top;
    if (y + 1 < ch) {
      const long long ta = 2 * (cell + cw);
      const Grad ga = tri_grad(u1, u2, mt, W, x, y + 1, 0, nc);
      e_top = edge_term(gu, au, lu, &ga, alpha[ta], lambda[ta], 0.0, 1.0, 1.0, nc);
    } else {
      e_top = edge_term(gu, au, lu, nullptr, 0.0, 0.0, 0.0, 1.0, 1.0, nc);
    }
    // left v-edge: left = lower of cell (x-1,y), right = upper (this cell)
    double e_left;
    if (x > 0) {
      const long long tl = 2 * (cell - 1);
      const Grad gL = tri_grad(u1, u2, mt, W, x - 1, y, 0, nc);
      e_left = edge_term(gL, alpha[tl], lambda[tl], &gu, au, lu, 1.0, 0.0, 1.0, nc);
    } else {
      e_left = edge_term(gu, au, lu, nullptr, 0.0, 0.0, -1.0, 0.0, 1.0, nc);
    }
    // right v-edge: left = lower (this cell), right = upper of cell (x+1,y)
    double e_right;
    if (x + 1 < cw) {
      const long long tr = 2 * (cell + 1) + 1;
      const Grad gR = tri_grad(u1, u2, mt, W, x + 1, y, 1, nc);
      e_right = edge_term(gl, al, ll, &gR, alpha[tr], lambda[tr], 1.0, 0.0, 1.0, nc);
    } else {
      e_right = edge_term(gl, al, ll, nullptr, 0.0, 0.0, 1.0, 0.0, 1.0, nc);
    }
    const long long v00 = static_cast<long long>(y) * W + x;
    const long long vl[3] = {v00, v00 + 1, v00 + W + 1};
    const long long vu[3] = {v00, v00 + W + 1, v00 + W};
    // eta = hK sqrt(elem) + 1/2 sum over tri_edges (mesh.cpp:106-120 order)
    double el = hK * sqrt(elem_part(t10, n, u1, u2, mt, vl, al, ll, nc));
    el += 0.5 * e_bot;
    el += 0.5 * e_right;
    el += 0.5 * e_diag;
    double eu = hK * sqrt(elem_part(t10, n, u1, u2, mt, vu, au, lu, nc));
    eu += 0.5 * e_diag;
    eu += 0.5 * e_top;
    eu += 0.5 * e_left;
    if (eta) {
      eta[tlo] = el;
      eta[tup] = eu;
    }
    local_max = dmax(local_max, el);
    local_max = dmax(local_max, eu);
  }
  // block max, then the last block finishes the (order-free) max
  __shared__ double sm[32];
  for (int off = 16; off; off >>= 1) local_max = dmax(local_max, __shfl_xor_sync(~0u, local_max, off));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = local_max;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) m = dmax(m, sm[w]);
    blockmax[blockIdx.x] = m;
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    if (t == gridDim.x - 1) {
      double mm = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) mm = dmax(mm, __ldcg(blockmax + b));
      *eta_max_out = mm;
      *counter = 0;
    }
  }
}

// update_alpha (adapt.cpp:101-112)
__global__ void k_update_alpha(double* __restrict__ out, const double* __restrict__ alpha,
                               const double* __restrict__ eta, const double* __restrict__ eta_max_p,
                               long long ntri, double kappa, double thr, double alpha_th) {
  const double eta_max = *eta_max_p;
  for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < ntri;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (eta_max <= 0.0) {
      out[t] = alpha[t];
      continue;
    }
    const double excess = dmax(eta[t] / eta_max - thr, 0.0);
    out[t] = dmax(alpha[t] / (1.0 + kappa * excess), alpha_th);
  }
}

// a25: discrete energy (assembly.cpp:201-238), a device reduction. One thread takes the
// two triangles of a cell (gradient term) and the vertex of the same index (data term);
// per-thread sums, warp/block reduction, per-block partials, and the last CTA sums the
// partials in block order, so the result is deterministic (not bitwise equal to the
// reference's serial sum: the summation order differs, rel. error ~1e-15).
__device__ __forceinline__ double lumped_weight(int x, int y, int W, int H) {
  int cnt = 0;  // incident triangles (mesh.cpp:122-126: area/3 each)
  if (x > 0 && y > 0) cnt += 2;
  if (x < W - 1 && y > 0) cnt += 1;
  if (x > 0 && y < H - 1) cnt += 1;
  if (x < W - 1 && y < H - 1) cnt += 2;
  double s = 0.0;
  for (int k = 0; k < cnt; ++k) s += 0.5 / 3.0;
  return s;
}

__global__ void k_energy(const double* __restrict__ t10, const double* __restrict__ alpha,
                         const double* __restrict__ lambda, const double* __restrict__ u3, int W,
                         int H, int nc, double* __restrict__ part, double* __restrict__ out,
                         unsigned* __restrict__ counter) {
  const int cw = W - 1, ch = H - 1;
  const size_t n = static_cast<size_t>(W) * H;
  const double* u1 = u3;
  const double* u2 = u3 + n;
  const double* mt = u3 + 2 * n;
  const long long ncell = static_cast<long long>(cw) * ch;
  const long long nwork = ncell > static_cast<long long>(n) ? ncell : static_cast<long long>(n);
  double eg = 0.0, ed = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < nwork;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (i < ncell) {
      const int x = static_cast<int>(i % cw), y = static_cast<int>(i / cw);
#pragma unroll
      for (int up = 0; up < 2; ++up) {
        const Grad g = tri_grad(u1, u2, mt, W, x, y, up, nc);
        double s = alpha[2 * i + up] * (g.g[0] * g.g[0] + g.g[1] * g.g[1] + g.g[2] * g.g[2] +
                                        g.g[3] * g.g[3]);
        if (nc == 3) s += lambda[2 * i + up] * (g.g[4] * g.g[4] + g.g[5] * g.g[5]);
        eg += 0.5 * s;  // area 1/2
      }
    }
    if (i < static_cast<long long>(n)) {
      const int x = static_cast<int>(i % W), y = static_cast<int>(i / W);
      // nodal_terms (assembly.cpp:19-28) and the reference's loop order
      double A[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, F[3] = {0, 0, 0};
      A[0] = t10[i], A[1] = t10[n + i], A[3] = t10[n + i], A[4] = t10[3 * n + i];
      F[0] = t10[6 * n + i], F[1] = t10[7 * n + i];
      if (nc == 3) {
        A[2] = t10[2 * n + i], A[5] = t10[4 * n + i];
        A[6] = t10[2 * n + i], A[7] = t10[4 * n + i], A[8] = t10[5 * n + i];
        F[2] = t10[8 * n + i];
      }
      const double U[3] = {u1[i], u2[i], nc == 3 ? mt[i] : 0.0};
      double quad = 0.0, lin = 0.0;
      for (int c = 0; c < nc; ++c) {
        for (int c2 = 0; c2 < nc; ++c2) quad += U[c] * A[c * 3 + c2] * U[c2];
        lin += F[c] * U[c];
      }
      ed += lumped_weight(x, y, W, H) * (quad - 2.0 * lin + t10[9 * n + i]);
    }
  }
  __shared__ double sm[2][32];
  for (int off = 16; off; off >>= 1) {
    eg += __shfl_xor_sync(~0u, eg, off);
    ed += __shfl_xor_sync(~0u, ed, off);
  }
  if ((threadIdx.x & 31) == 0) sm[0][threadIdx.x >> 5] = eg, sm[1][threadIdx.x >> 5] = ed;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) a += sm[0][w], b += sm[1][w];
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    if (t == gridDim.x - 1) {
      double sg = 0.0, sd = 0.0;
      for (unsigned k = 0; k < gridDim.x; ++k) sg += __ldcg(part + 2 * k), sd += __ldcg(part + 2 * k + 1);
      *out = 0.5 * (sg + sd);
      *counter = 0;
    }
  }
}

}  // namespace

void energy(const double* t10, const double* alpha, const double* lambda, const double* u3,
            int W, int H, int nc, double* out_dev, double* scratch, unsigned* counter,
            cudaStream_t st) {
  k_energy<<<kRedBlocks, kRedThreads, 0, st>>>(t10, alpha, lambda, u3, W, H, nc, scratch,
                                               out_dev, counter);
  FFB_LAUNCHED();
}

void error_indicator(const double* t10, const double* alpha, const double* lambda,
                     const double* u3, int W, int H, int nc, double* eta, double* eta_max_dev,
                     double* scratch, unsigned* counter, cudaStream_t st) {
  k_indicator<<<kRedBlocks, kRedThreads, 0, st>>>(t10, alpha, lambda, u3, W, H, nc, eta,
                                                  scratch, eta_max_dev, counter);
  FFB_LAUNCHED();
}

void update_alpha(double* alpha_out, const double* alpha, const double* eta,
                  const double* eta_max_dev, long long ntri, double kappa, double thr,
                  double alpha_th, cudaStream_t st) {
  k_update_alpha<<<kRedBlocks, kRedThreads, 0, st>>>(alpha_out, alpha, eta, eta_max_dev, ntri,
                                                     kappa, thr, alpha_th);
  FFB_LAUNCHED();
}

}  // namespace ffb
