// K7/K8: the conjugate-gradient iteration around the additive-Schwarz preconditioner.
//
// Same recurrence and stopping rule as the reference's cg_solve (src/linsolve.cpp:298-361):
// true relative residual ||r||/||b|| <= tol checked after the x/r update, warm start,
// "indefinite" failure when p.Ap <= 0, max_iters. The Jacobi preconditioner is replaced
// by the symmetric additive Schwarz operator M^-1 = sum_i R_i^T A_i^-1 R_i (the
// reference's RAS is nonsymmetric and cannot precondition CG).
//
// Per iteration: spmv_p (p = z + beta p fused into the matrix-free operator, p.Ap), update
// (x, r, r.r), asm (band solves, band.cu), combine (z = sum of the subdomain solutions, r.z).
//
// Multi-GPU layout (one rank per GPU, capi.cpp): rank r owns a band of subdomain ROWS
// [j0, j1) and the pixel rows [y0, y1) of their cores. Every kernel works on the owned rows;
// the halos a rank needs are neighbour rows exchanged between the kernels (r on the rows its
// subdomains' free rectangles reach into, p/z on one row, and the partial sums of z on the
// rows its subdomains cover in the neighbour's band).
//
// Reductions are WORLD-INDEPENDENT: the reduction unit is a subdomain row j (its core rows,
// full width) processed by a fixed number kCU of CTAs with a fixed thread -> pixel map; the
// unit's value is the sum of its CTAs' partials in CTA order (computed by the last CTA to
// finish), and the global value the sum of the units in j order (k_scalar, after an
// all-reduce of the unit values when world > 1: every unit is non-zero on exactly one rank,
// so the all-reduce is exact). The z combine sums the subdomains covering a pixel row-pair
// by row-pair, (z_{j,i} + z_{j,i+1}) + (z_{j+1,i} + z_{j+1,i+1}), so a row-pair computed on
// the neighbouring rank enters the same expression. Hence every scalar, iterate and the
// iteration count are bitwise identical for any number of GPUs (at equal subdomain-solve
// cluster size, which orders the sums inside the line solves), and run to run.
// Once converged (or failed) every kernel returns at entry, so the host may enqueue
// several iterations ahead and only reads the control block between chunks.
#include "ffb_internal.cuh"

#include <algorithm>

namespace ffb {

namespace {

constexpr int T = kRedThreads;

__device__ __forceinline__ double block_sum(double v, double* sm) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_down_sync(~0u, v, off);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (T >> 5); ++i) s += sm[i];
  return s;  // valid in thread 0
}

// thread 0 of every block calls this after writing its partial; returns true in the last
// block, which then owns the final fixed-order sum.
__device__ __forceinline__ bool arrive_last(unsigned* counter) {
  __threadfence();
  const unsigned t = atomicAdd(counter, 1u);
  return t == gridDim.x - 1;
}

enum Stage { kStInit = 0, kStPap, kStRr, kStRz };

// the scalar recurrences of cg_solve (linsolve.cpp:314-357) once a reduction is complete;
// s2 only for kStInit (r.r next to b.b)
__device__ void apply_stage(PcgCtl* ctl, int stage, double s, double s2) {
  switch (stage) {
    case kStInit:
      ctl->bb = s;
      ctl->rr = s2;
      ctl->normb = sqrt(s);
      ctl->k = 0;
      ctl->iters = 0;
      ctl->err = 0;
      if (s == 0.0) {  // linsolve.cpp:321-324
        ctl->zero_rhs = 1;
        ctl->res = 0.0;
        ctl->done = 1;
      } else {
        ctl->res = sqrt(s2) / ctl->normb;
        // a NaN residual can never pass the test: stop at once (the host reports
        // "no convergence ... relative residual nan") instead of iterating to max_iters
        ctl->done = (ctl->res <= ctl->tol || ctl->res != ctl->res) ? 1 : 0;
      }
      break;
    case kStPap:
      ctl->pAp = s;
      break;
    case kStRr:
      ctl->rr = s;
      ctl->res = sqrt(s) / ctl->normb;
      ctl->iters = ctl->k;
      if (ctl->res <= ctl->tol || ctl->k >= ctl->max_iters || ctl->res != ctl->res) ctl->done = 1;
      break;
    case kStRz:
      ctl->rz_old = ctl->rz;
      ctl->rz = s;
      ctl->k += 1;
      break;
  }
}

// Last CTA of a reduction kernel: unit values ur[j] (j in the rank's units) as the CTA-order
// sum of part[], then, if `finish` (world == 1), the j-order total and the scalar update.
// part2/ur2 carry a second simultaneous reduction (k_init) or are null.
__device__ void finish_units(const RankRows& g, int py, const double* part, double* ur,
                             const double* part2, double* ur2, int finish, PcgCtl* ctl,
                             int stage) {
  const int nu = g.j1 - g.j0;
  for (int u = threadIdx.x; u < nu; u += blockDim.x) {
    double a = 0.0, b = 0.0;
    for (int c = 0; c < kCU; ++c) {
      a += __ldcg(part + u * kCU + c);
      if (part2) b += __ldcg(part2 + u * kCU + c);
    }
    ur[g.j0 + u] = a;
    if (ur2) ur2[g.j0 + u] = b;
  }
  if (!finish) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int j = 0; j < py; ++j) {
      a += ur[j];
      if (ur2) b += ur2[j];
    }
    apply_stage(ctl, stage, a, b);
  }
}

// (unit, CTA-in-unit) of this block; the unit's pixels are its core rows, full width
struct UnitRange {
  long long v0;  // first pixel
  int n;         // pixels
  int c;         // CTA index within the unit
  int u;         // unit index relative to j0
};
__device__ __forceinline__ UnitRange unit_of_block(const RankRows& g, const int* __restrict__ ys,
                                                   int W) {
  UnitRange r;
  r.u = blockIdx.x / kCU;
  r.c = blockIdx.x - r.u * kCU;
  const int j = g.j0 + r.u;
  r.v0 = static_cast<long long>(ys[j]) * W;
  r.n = (ys[j + 1] - ys[j]) * W;
  return r;
}

struct Vtx {
  int x, y;
  long long v;
};

// (A p)_c at vertex v, stencil order of the reference CSR row (assembly.cpp:240-249)
template <int NC>
__device__ __forceinline__ void apply_at(const double* __restrict__ coef, size_t n, int W, int H,
                                         const Vtx& q, const double* pc, const double* pd,
                                         const double* pl, const double* pr, const double* pu,
                                         double* out) {
  const long long v = q.v;
  double m[3][3];
  m[0][0] = coef[0 * n + v];
  m[0][1] = m[1][0] = coef[1 * n + v];
  m[1][1] = coef[3 * n + v];
  if (NC == 3) {
    m[0][2] = m[2][0] = coef[2 * n + v];
    m[1][2] = m[2][1] = coef[4 * n + v];
    m[2][2] = coef[5 * n + v];
  }
  double ehA = 0, ehL = 0, evA = 0, evL = 0, elA = 0, elL = 0, edA = 0, edL = 0;
  if (q.x < W - 1) { ehA = coef[6 * n + v]; if (NC == 3) ehL = coef[7 * n + v]; }
  if (q.y < H - 1) { evA = coef[8 * n + v]; if (NC == 3) evL = coef[9 * n + v]; }
  if (q.x > 0) { elA = coef[6 * n + v - 1]; if (NC == 3) elL = coef[7 * n + v - 1]; }
  if (q.y > 0) { edA = coef[8 * n + v - W]; if (NC == 3) edL = coef[9 * n + v - W]; }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double kd_ = c < 2 ? edA : edL, kl = c < 2 ? elA : elL;
    const double kr = c < 2 ? ehA : ehL, ku = c < 2 ? evA : evL;
    double s = 0.0;
    s += kd_ * pd[c];
    s += kl * pl[c];
#pragma unroll
    for (int c2 = 0; c2 < NC; ++c2) s += m[c][c2] * pc[c2];
    s += kr * pr[c];
    s += ku * pu[c];
    out[c] = s;
  }
}

template <int NC>
__device__ __forceinline__ void load3(const double* __restrict__ a, long long v, double* o) {
#pragma unroll
  for (int c = 0; c < NC; ++c) o[c] = a[v * NC + c];
}

// r = b - A x ; b.b ; r.r   (linsolve.cpp:314-327), on the owned rows
template <int NC>
__global__ void __launch_bounds__(T) k_init(const double* __restrict__ coef,
                                            const double* __restrict__ b,
                                            const double* __restrict__ x, double* __restrict__ r,
                                            int W, int H, RankRows g, const int* __restrict__ ys,
                                            int py, PcgCtl* ctl, double* part, double* ur,
                                            int finish) {
  __shared__ double sm[32];
  const size_t n = static_cast<size_t>(W) * H;
  const UnitRange ur_ = unit_of_block(g, ys, W);
  double bb = 0.0, rr = 0.0;
  for (int i = ur_.c * T + threadIdx.x; i < ur_.n; i += kCU * T) {
    const long long v = ur_.v0 + i;
    Vtx q{static_cast<int>(v % W), static_cast<int>(v / W), v};
    double pc[3], pd[3] = {0, 0, 0}, pl[3] = {0, 0, 0}, pr[3] = {0, 0, 0}, pu[3] = {0, 0, 0};
    load3<NC>(x, v, pc);
    if (q.y > 0) load3<NC>(x, v - W, pd);
    if (q.x > 0) load3<NC>(x, v - 1, pl);
    if (q.x < W - 1) load3<NC>(x, v + 1, pr);
    if (q.y < H - 1) load3<NC>(x, v + W, pu);
    double ax[3];
    apply_at<NC>(coef, n, W, H, q, pc, pd, pl, pr, pu, ax);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double bc = b[v * NC + c];
      const double rc = bc - ax[c];
      r[v * NC + c] = rc;
      bb += bc * bc;
      rr += rc * rc;
    }
  }
  bb = block_sum(bb, sm);
  rr = block_sum(rr, sm);
  __shared__ bool last;
  double* part2 = part + static_cast<long long>(gridDim.x);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = bb;
    part2[blockIdx.x] = rr;
    last = arrive_last(&ctl->counter[0]);
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) ctl->counter[0] = 0;
  finish_units(g, py, part, ur, part2, ur + py, finish, ctl, kStInit);
}

// S_j(v) = sum over the column-subdomains i of row j covering pixel (x, y), ascending i
template <int NC>
__device__ __forceinline__ void row_pair_sum(const SubInfo* __restrict__ subs, int px, int j,
                                             int ly, const AxisMap& cm,
                                             const double* __restrict__ zlocal, double* acc) {
  bool first = true;
#pragma unroll
  for (int ii = 0; ii < 2; ++ii) {
    const int i = ii ? cm.p1 : cm.p0;
    if (i < 0) continue;
    const int lx = ii ? cm.l1 : cm.l0;
    const SubInfo& s = subs[j * px + i];
    const long long vl = s.xfast ? static_cast<long long>(ly) * s.fw + lx
                                 : static_cast<long long>(lx) * s.fh + ly;
    const double* zl = zlocal + s.vec_off + vl * NC;
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = first ? zl[c] : acc[c] + zl[c];
    first = false;
  }
}

// The partial sums of this rank's subdomains on the neighbours' rows it covers: rows
// [fa0, fa1) above (covered by subdomain row j0 only) and [fb0, fb1) below (row j1 - 1 only),
// sent to rank - 1 / rank + 1 before their combine.
template <int NC>
__global__ void __launch_bounds__(T)
    k_zpart(const SubInfo* __restrict__ subs, const AxisMap* __restrict__ colmap,
            const AxisMap* __restrict__ rowmap, int px, const double* __restrict__ zlocal, int W,
            RankRows g, double* __restrict__ send_up, double* __restrict__ send_dn,
            const PcgCtl* ctl) {
  if (ctl->done | ctl->err) return;
  const int na = (g.fa1 - g.fa0) * W, nb = (g.fb1 - g.fb0) * W;
  for (int k = blockIdx.x * T + threadIdx.x; k < na + nb; k += gridDim.x * T) {
    const bool up = k < na;
    const int kk = up ? k : k - na;
    const int y = (up ? g.fa0 : g.fb0) + kk / W, x = kk % W;
    const int j = up ? g.j0 : g.j1 - 1;
    const AxisMap rm = rowmap[y];
    const int ly = rm.p0 == j ? rm.l0 : rm.l1;
    double acc[3];
    row_pair_sum<NC>(subs, px, j, ly, colmap[x], zlocal, acc);
    double* out = (up ? send_up : send_dn) + static_cast<long long>(kk) * NC;
#pragma unroll
    for (int c = 0; c < NC; ++c) out[c] = acc[c];
  }
}

// combine on the owned rows: z = S_j0 (+ S_j1) over the (<= 2) subdomain rows covering the
// pixel, ascending j; an S of a subdomain row owned by a neighbour comes from its k_zpart
// (recv_up: rows [ra0, ra1) from rank - 1; recv_dn: rows [rb0, rb1) from rank + 1). r.z.
// Two-level (world == 1 only): + the core's coarse value yc (coarse.cu).
template <int NC>
__global__ void __launch_bounds__(T) k_combine(const SubInfo* __restrict__ subs,
                                               const AxisMap* __restrict__ colmap,
                                               const AxisMap* __restrict__ rowmap, int px,
                                               const double* __restrict__ zlocal,
                                               const double* __restrict__ r,
                                               double* __restrict__ z, int W, RankRows g,
                                               const int* __restrict__ ys, int py,
                                               const double* __restrict__ recv_up,
                                               const double* __restrict__ recv_dn, PcgCtl* ctl,
                                               double* part, double* ur, int finish,
                                               const double* __restrict__ yc,
                                               const int* __restrict__ ccol,
                                               const int* __restrict__ crow) {
  if (ctl->done | ctl->err) return;
  __shared__ double sm[32];
  const UnitRange ur_ = unit_of_block(g, ys, W);
  double rz = 0.0;
  for (int i = ur_.c * T + threadIdx.x; i < ur_.n; i += kCU * T) {
    const long long v = ur_.v0 + i;
    const int x = static_cast<int>(v % W), y = static_cast<int>(v / W);
    const AxisMap cm = colmap[x], rm = rowmap[y];
    double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      const int j = jj ? rm.p1 : rm.p0;
      if (j < 0) continue;
      double s[3];
      if (j < g.j0) {
        const double* f = recv_up + (static_cast<long long>(y - g.ra0) * W + x) * NC;
#pragma unroll
        for (int c = 0; c < NC; ++c) s[c] = f[c];
      } else if (j >= g.j1) {
        const double* f = recv_dn + (static_cast<long long>(y - g.rb0) * W + x) * NC;
#pragma unroll
        for (int c = 0; c < NC; ++c) s[c] = f[c];
      } else {
        row_pair_sum<NC>(subs, px, j, jj ? rm.l1 : rm.l0, cm, zlocal, s);
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[c] = jj ? acc[c] + s[c] : s[c];
    }
    if (yc) {  // two-level: + Z A0^-1 Z^T r (coarse.cu), the core's coarse value
      const double* yv = yc + static_cast<long long>(ccol[x] + crow[y]) * NC;
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[c] += yv[c];
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      z[v * NC + c] = acc[c];
      rz += r[v * NC + c] * acc[c];
    }
  }
  rz = block_sum(rz, sm);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = rz;
    last = arrive_last(&ctl->counter[1]);
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) ctl->counter[1] = 0;
  finish_units(g, py, part, ur, nullptr, nullptr, finish, ctl, kStRz);
}

// p = z + beta p (beta = rz/rz_old, p = z on the first iteration); q = A p; p.q on the owned
// rows. p is also written on the (<= 1) halo row on each side, so the next iteration's
// stencil finds its old value there.
template <int NC>
__global__ void __launch_bounds__(T) k_spmv_p(const double* __restrict__ coef,
                                              const double* __restrict__ z, double* __restrict__ P0,
                                              double* __restrict__ P1, double* __restrict__ qv,
                                              int W, int H, RankRows g,
                                              const int* __restrict__ ys, int py, PcgCtl* ctl,
                                              double* part, double* ur, int finish) {
  if (ctl->done | ctl->err) return;
  __shared__ double sm[32];
  const int k = ctl->k;
  const double beta = k == 1 ? 0.0 : ctl->rz / ctl->rz_old;
  const double* __restrict__ pold = (k & 1) ? P1 : P0;
  double* __restrict__ pnew = (k & 1) ? P0 : P1;
  const size_t n = static_cast<size_t>(W) * H;
  auto pn = [&](long long w, double* o) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
      o[c] = k == 1 ? z[w * NC + c] : z[w * NC + c] + beta * pold[w * NC + c];
  };
  const UnitRange ur_ = unit_of_block(g, ys, W);
  double pq = 0.0;
  for (int i = ur_.c * T + threadIdx.x; i < ur_.n; i += kCU * T) {
    const long long v = ur_.v0 + i;
    Vtx q{static_cast<int>(v % W), static_cast<int>(v / W), v};
    double pc[3], pd[3] = {0, 0, 0}, pl[3] = {0, 0, 0}, pr[3] = {0, 0, 0}, pu[3] = {0, 0, 0};
    pn(v, pc);
    if (q.y > 0) pn(v - W, pd);
    if (q.x > 0) pn(v - 1, pl);
    if (q.x < W - 1) pn(v + 1, pr);
    if (q.y < H - 1) pn(v + W, pu);
    double ap[3];
    apply_at<NC>(coef, n, W, H, q, pc, pd, pl, pr, pu, ap);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      pnew[v * NC + c] = pc[c];
      qv[v * NC + c] = ap[c];
      pq += pc[c] * ap[c];
    }
  }
  // halo rows of p (outside the owned band, inside the image)
  const int hu = g.y0 > 0 ? 1 : 0, hd = g.y1 < H ? 1 : 0;
  for (int i = blockIdx.x * T + threadIdx.x; i < (hu + hd) * W; i += gridDim.x * T) {
    const int y = (i < hu * W) ? g.y0 - 1 : g.y1;
    const long long v = static_cast<long long>(y) * W + (i % W);
    double pc[3];
    pn(v, pc);
#pragma unroll
    for (int c = 0; c < NC; ++c) pnew[v * NC + c] = pc[c];
  }
  pq = block_sum(pq, sm);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = pq;
    last = arrive_last(&ctl->counter[2]);
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) ctl->counter[2] = 0;
  finish_units(g, py, part, ur, nullptr, nullptr, finish, ctl, kStPap);
}

// x += alpha p ; r -= alpha q ; r.r ; convergence test (linsolve.cpp:335-349), owned rows
template <int NC>
__global__ void __launch_bounds__(T) k_update(double* __restrict__ x, double* __restrict__ r,
                                              const double* __restrict__ P0,
                                              const double* __restrict__ P1,
                                              const double* __restrict__ qv, int W, RankRows g,
                                              const int* __restrict__ ys, int py, PcgCtl* ctl,
                                              double* part, double* ur, int finish) {
  if (ctl->done | ctl->err) return;
  __shared__ double sm[32];
  const int k = ctl->k;
  const double pAp = ctl->pAp;
  if (pAp <= 0.0) {  // linsolve.cpp:339
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctl->err = 1;
      ctl->err_it = k;
    }
    return;
  }
  const double alpha = ctl->rz / pAp;
  const double* __restrict__ p = (k & 1) ? P0 : P1;
  const UnitRange ur_ = unit_of_block(g, ys, W);
  double rr = 0.0;
  for (int i = ur_.c * T + threadIdx.x; i < ur_.n; i += kCU * T) {
    const long long v = ur_.v0 + i;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const long long e = v * NC + c;
      x[e] += alpha * p[e];
      const double ri = r[e] - alpha * qv[e];
      r[e] = ri;
      rr += ri * ri;
    }
  }
  rr = block_sum(rr, sm);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = rr;
    last = arrive_last(&ctl->counter[3]);
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) ctl->counter[3] = 0;
  finish_units(g, py, part, ur, nullptr, nullptr, finish, ctl, kStRr);
}

// after the all-reduce of the unit values (world > 1): the j-order total, the scalar update
__global__ void k_scalar(const double* __restrict__ ur, int py, int stage, PcgCtl* ctl) {
  if (ctl->done | ctl->err) return;
  double a = 0.0, b = 0.0;
  for (int j = 0; j < py; ++j) {
    a += ur[j];
    if (stage == kStInit) b += ur[py + j];
  }
  apply_stage(ctl, stage, a, b);
}

// warm start of the next adaptive pass: x <- x + theta (x - xprev), xprev <- old x
// (theta == 0: only the copy)
__global__ void k_extrapolate(double* __restrict__ x, double* __restrict__ xprev, long long n,
                              double theta) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double xc = x[i];
    if (theta != 0.0) x[i] = xc + theta * (xc - xprev[i]);
    xprev[i] = xc;
  }
}

}  // namespace

void vec_extrapolate(double* x, double* xprev, long long n, double theta, cudaStream_t st) {
  k_extrapolate<<<kRedBlocks, T, 0, st>>>(x, xprev, n, theta);
  FFB_LAUNCHED();
}

static int grid_of(const RankRows& g) { return (g.j1 - g.j0) * kCU; }

void pcg_init(int nc, const double* coef, const double* b, const double* x, double* r, int W,
              int H, const RankRows& g, const int* ys, int py, PcgCtl* ctl, double* part,
              double* ur, int finish, cudaStream_t st) {
  if (grid_of(g) == 0) return;
  if (nc == 3)
    k_init<3><<<grid_of(g), T, 0, st>>>(coef, b, x, r, W, H, g, ys, py, ctl, part, ur, finish);
  else
    k_init<2><<<grid_of(g), T, 0, st>>>(coef, b, x, r, W, H, g, ys, py, ctl, part, ur, finish);
  FFB_LAUNCHED();
}

void pcg_zpart(int nc, const SubInfo* subs, const AxisMap* colmap, const AxisMap* rowmap, int px,
               const double* zlocal, int W, const RankRows& g, double* send_up, double* send_dn,
               const PcgCtl* ctl, cudaStream_t st) {
  const int n = (g.fa1 - g.fa0 + g.fb1 - g.fb0) * W;
  if (n <= 0) return;
  const int grid = std::min((n + T - 1) / T, 4 * 148);
  if (nc == 3)
    k_zpart<3><<<grid, T, 0, st>>>(subs, colmap, rowmap, px, zlocal, W, g, send_up, send_dn, ctl);
  else
    k_zpart<2><<<grid, T, 0, st>>>(subs, colmap, rowmap, px, zlocal, W, g, send_up, send_dn, ctl);
  FFB_LAUNCHED();
}

void pcg_combine(int nc, const SubInfo* subs, const AxisMap* colmap, const AxisMap* rowmap,
                 int px, const double* zlocal, const double* r, double* z, int W,
                 const RankRows& g, const int* ys, int py, const double* recv_up,
                 const double* recv_dn, PcgCtl* ctl, double* part, double* ur, int finish,
                 cudaStream_t st, const double* yc, const int* ccol, const int* crow) {
  if (grid_of(g) == 0) return;
  if (nc == 3)
    k_combine<3><<<grid_of(g), T, 0, st>>>(subs, colmap, rowmap, px, zlocal, r, z, W, g, ys, py,
                                           recv_up, recv_dn, ctl, part, ur, finish, yc, ccol, crow);
  else
    k_combine<2><<<grid_of(g), T, 0, st>>>(subs, colmap, rowmap, px, zlocal, r, z, W, g, ys, py,
                                           recv_up, recv_dn, ctl, part, ur, finish, yc, ccol, crow);
  FFB_LAUNCHED();
}

void pcg_spmv_p(int nc, const double* coef, const double* z, double* P0, double* P1, double* q,
                int W, int H, const RankRows& g, const int* ys, int py, PcgCtl* ctl, double* part,
                double* ur, int finish, cudaStream_t st) {
  if (grid_of(g) == 0) return;
  if (nc == 3)
    k_spmv_p<3><<<grid_of(g), T, 0, st>>>(coef, z, P0, P1, q, W, H, g, ys, py, ctl, part, ur, finish);
  else
    k_spmv_p<2><<<grid_of(g), T, 0, st>>>(coef, z, P0, P1, q, W, H, g, ys, py, ctl, part, ur, finish);
  FFB_LAUNCHED();
}

void pcg_update(int nc, double* x, double* r, const double* P0, const double* P1,
                const double* q, int W, const RankRows& g, const int* ys, int py, PcgCtl* ctl,
                double* part, double* ur, int finish, cudaStream_t st) {
  if (grid_of(g) == 0) return;
  if (nc == 3)
    k_update<3><<<grid_of(g), T, 0, st>>>(x, r, P0, P1, q, W, g, ys, py, ctl, part, ur, finish);
  else
    k_update<2><<<grid_of(g), T, 0, st>>>(x, r, P0, P1, q, W, g, ys, py, ctl, part, ur, finish);
  FFB_LAUNCHED();
}

void pcg_scalar(const double* ur, int py, int stage, PcgCtl* ctl, cudaStream_t st) {
  k_scalar<<<1, 1, 0, st>>>(ur, py, stage, ctl);
  FFB_LAUNCHED();
}

int pcg_stage_init() { return kStInit; }
int pcg_stage_pap() { return kStPap; }
int pcg_stage_rr() { return kStRr; }
int pcg_stage_rz() { return kStRz; }

}  // namespace ffb
