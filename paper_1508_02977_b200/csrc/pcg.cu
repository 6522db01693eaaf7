// K7/K8: the conjugate-gradient iteration around the additive-Schwarz preconditioner.
//
// Same recurrence and stopping rule as the reference's cg_solve (src/linsolve.cpp:298-361):
// true relative residual ||r||/||b|| <= tol checked after the x/r update, warm start,
// "indefinite" failure when p.Ap <= 0, max_iters. The Jacobi preconditioner is replaced
// by the symmetric additive Schwarz operator M^-1 = sum_i R_i^T A_i^-1 R_i (the
// reference's RAS is nonsymmetric and cannot precondition CG).
//
// Four kernels per iteration, no host round trip: spmv_p (p = z + beta p fused into the
// matrix-free operator, p.Ap), update (x, r, r.r), asm (band solves, band.cu), combine
// (z = sum of subdomain solutions in ascending subdomain order, r.z). Scalars live in a
// device control block; every reduction writes per-CTA partials and the last CTA to
// finish sums them in a fixed order, so results are bitwise reproducible run to run.
// Once converged (or failed) every kernel returns at entry, so the host may enqueue
// several iterations ahead and only reads the control block between chunks.
#include "ffb_internal.cuh"

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

// fixed-order sum of gridDim.x partials by one block
__device__ __forceinline__ double final_sum(const double* part, int nparts, double* sm) {
  double v = 0.0;
  for (int i = threadIdx.x; i < nparts; i += T) v += __ldcg(part + i);
  return block_sum(v, sm);
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

// r = b - A x ; b.b ; r.r   (linsolve.cpp:314-327)
template <int NC>
__global__ void __launch_bounds__(T) k_init(const double* __restrict__ coef,
                                            const double* __restrict__ b,
                                            const double* __restrict__ x, double* __restrict__ r,
                                            int W, int H, PcgCtl* ctl, double* part) {
  __shared__ double sm[32];
  const size_t n = static_cast<size_t>(W) * H;
  double bb = 0.0, rr = 0.0;
  for (long long v = static_cast<long long>(blockIdx.x) * T + threadIdx.x;
       v < static_cast<long long>(n); v += static_cast<long long>(gridDim.x) * T) {
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
  if (threadIdx.x == 0) {
    part[blockIdx.x] = bb;
    part[gridDim.x + blockIdx.x] = rr;
    last = arrive_last(&ctl->counter[0]);
  }
  __syncthreads();
  if (!last) return;
  const double BB = final_sum(part, gridDim.x, sm);
  const double RR = final_sum(part + gridDim.x, gridDim.x, sm);
  if (threadIdx.x == 0) {
    ctl->counter[0] = 0;
    ctl->bb = BB;
    ctl->rr = RR;
    ctl->normb = sqrt(BB);
    ctl->k = 0;
    ctl->iters = 0;
    ctl->err = 0;
    if (BB == 0.0) {  // linsolve.cpp:321-324
      ctl->zero_rhs = 1;
      ctl->res = 0.0;
      ctl->done = 1;
    } else {
      ctl->res = sqrt(RR) / ctl->normb;
      ctl->done = ctl->res <= ctl->tol ? 1 : 0;
    }
  }
}

// combine: z = sum_i R_i^T z_i (ascending subdomain id), r.z; k++
// With a shard [s_lo, s_hi) (multi-GPU) only this rank's subdomains contribute and the
// result is a partial z that the host all-reduces before k_rz forms r.z.
template <int NC>
__global__ void __launch_bounds__(T) k_combine(const SubInfo* __restrict__ subs,
                                               const AxisMap* __restrict__ colmap,
                                               const AxisMap* __restrict__ rowmap, int px,
                                               const double* __restrict__ zlocal,
                                               const double* __restrict__ r,
                                               double* __restrict__ z, int W, int H,
                                               PcgCtl* ctl, double* part, int s_lo, int s_hi,
                                               int partial, const double* __restrict__ yc,
                                               const int* __restrict__ ccol,
                                               const int* __restrict__ crow) {
  if (ctl->done | ctl->err) return;
  __shared__ double sm[32];
  const size_t n = static_cast<size_t>(W) * H;
  double rz = 0.0;
  for (long long v = static_cast<long long>(blockIdx.x) * T + threadIdx.x;
       v < static_cast<long long>(n); v += static_cast<long long>(gridDim.x) * T) {
    const int x = static_cast<int>(v % W), y = static_cast<int>(v / W);
    const AxisMap cm = colmap[x], rm = rowmap[y];
    double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      const int j = jj ? rm.p1 : rm.p0;
      if (j < 0) continue;
      const int ly = jj ? rm.l1 : rm.l0;
#pragma unroll
      for (int ii = 0; ii < 2; ++ii) {
        const int i = ii ? cm.p1 : cm.p0;
        if (i < 0) continue;
        const int lx = ii ? cm.l1 : cm.l0;
        const int sid = j * px + i;
        if (sid < s_lo || sid >= s_hi) continue;
        const SubInfo& s = subs[sid];
        const long long vl = s.xfast ? static_cast<long long>(ly) * s.fw + lx
                                     : static_cast<long long>(lx) * s.fh + ly;
        const double* zl = zlocal + s.vec_off + vl * NC;
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] += zl[c];
      }
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
  if (partial) return;
  rz = block_sum(rz, sm);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = rz;
    last = arrive_last(&ctl->counter[1]);
  }
  __syncthreads();
  if (!last) return;
  const double RZ = final_sum(part, gridDim.x, sm);
  if (threadIdx.x == 0) {
    ctl->counter[1] = 0;
    ctl->rz_old = ctl->rz;
    ctl->rz = RZ;
    ctl->k += 1;
  }
}

// r.z of the all-reduced z (multi-GPU stage B); k++
__global__ void __launch_bounds__(T) k_rz(const double* __restrict__ r,
                                          const double* __restrict__ z, long long nvec,
                                          PcgCtl* ctl, double* part) {
  if (ctl->done | ctl->err) return;
  __shared__ double sm[32];
  double rz = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * T + threadIdx.x; i < nvec;
       i += static_cast<long long>(gridDim.x) * T)
    rz += r[i] * z[i];
  rz = block_sum(rz, sm);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = rz;
    last = arrive_last(&ctl->counter[1]);
  }
  __syncthreads();
  if (!last) return;
  const double RZ = final_sum(part, gridDim.x, sm);
  if (threadIdx.x == 0) {
    ctl->counter[1] = 0;
    ctl->rz_old = ctl->rz;
    ctl->rz = RZ;
    ctl->k += 1;
  }
}

// p = z + beta p (beta = rz/rz_old, p = z on the first iteration); q = A p; p.q
template <int NC>
__global__ void __launch_bounds__(T) k_spmv_p(const double* __restrict__ coef,
                                              const double* __restrict__ z, double* __restrict__ P0,
                                              double* __restrict__ P1, double* __restrict__ qv,
                                              int W, int H, PcgCtl* ctl, double* part) {
  if (ctl->done | ctl->err) return;
  __shared__ double sm[32];
  const int k = ctl->k;
  const double beta = k == 1 ? 0.0 : ctl->rz / ctl->rz_old;
  const double* __restrict__ pold = (k & 1) ? P1 : P0;
  double* __restrict__ pnew = (k & 1) ? P0 : P1;
  const size_t n = static_cast<size_t>(W) * H;
  double pq = 0.0;
  for (long long v = static_cast<long long>(blockIdx.x) * T + threadIdx.x;
       v < static_cast<long long>(n); v += static_cast<long long>(gridDim.x) * T) {
    Vtx q{static_cast<int>(v % W), static_cast<int>(v / W), v};
    auto pn = [&](long long w, double* o) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
        o[c] = k == 1 ? z[w * NC + c] : z[w * NC + c] + beta * pold[w * NC + c];
    };
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
  pq = block_sum(pq, sm);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = pq;
    last = arrive_last(&ctl->counter[2]);
  }
  __syncthreads();
  if (!last) return;
  const double PQ = final_sum(part, gridDim.x, sm);
  if (threadIdx.x == 0) {
    ctl->counter[2] = 0;
    ctl->pAp = PQ;
  }
}

// x += alpha p ; r -= alpha q ; r.r ; convergence test (linsolve.cpp:335-349)
template <int NC>
__global__ void __launch_bounds__(T) k_update(double* __restrict__ x, double* __restrict__ r,
                                              const double* __restrict__ P0,
                                              const double* __restrict__ P1,
                                              const double* __restrict__ qv, long long nvec,
                                              int max_iters, PcgCtl* ctl, double* part) {
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
  double rr = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * T + threadIdx.x; i < nvec;
       i += static_cast<long long>(gridDim.x) * T) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * qv[i];
    r[i] = ri;
    rr += ri * ri;
  }
  rr = block_sum(rr, sm);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = rr;
    last = arrive_last(&ctl->counter[3]);
  }
  __syncthreads();
  if (!last) return;
  const double RR = final_sum(part, gridDim.x, sm);
  if (threadIdx.x == 0) {
    ctl->counter[3] = 0;
    ctl->rr = RR;
    ctl->res = sqrt(RR) / ctl->normb;
    ctl->iters = k;
    if (ctl->res <= ctl->tol || k >= max_iters) ctl->done = 1;
  }
}

}  // namespace

void pcg_init(int nc, const double* coef, const double* b, const double* x, double* r, int W,
              int H, PcgCtl* ctl, double* part, cudaStream_t st) {
  if (nc == 3)
    k_init<3><<<kRedBlocks, T, 0, st>>>(coef, b, x, r, W, H, ctl, part);
  else
    k_init<2><<<kRedBlocks, T, 0, st>>>(coef, b, x, r, W, H, ctl, part);
  FFB_LAUNCHED();
}

void pcg_combine(int nc, const SubInfo* subs, const AxisMap* colmap, const AxisMap* rowmap,
                 int px, const double* zlocal, const double* r, double* z, int W, int H,
                 PcgCtl* ctl, double* part, int s_lo, int s_hi, int partial, cudaStream_t st,
                 const double* yc, const int* ccol, const int* crow) {
  if (nc == 3)
    k_combine<3><<<kRedBlocks, T, 0, st>>>(subs, colmap, rowmap, px, zlocal, r, z, W, H, ctl, part,
                                           s_lo, s_hi, partial, yc, ccol, crow);
  else
    k_combine<2><<<kRedBlocks, T, 0, st>>>(subs, colmap, rowmap, px, zlocal, r, z, W, H, ctl, part,
                                           s_lo, s_hi, partial, yc, ccol, crow);
  FFB_LAUNCHED();
}

void pcg_rz(const double* r, const double* z, long long nvec, PcgCtl* ctl, double* part,
            cudaStream_t st) {
  k_rz<<<kRedBlocks, T, 0, st>>>(r, z, nvec, ctl, part);
  FFB_LAUNCHED();
}

void pcg_spmv_p(int nc, const double* coef, const double* z, double* P0, double* P1, double* q,
                int W, int H, PcgCtl* ctl, double* part, cudaStream_t st) {
  if (nc == 3)
    k_spmv_p<3><<<kRedBlocks, T, 0, st>>>(coef, z, P0, P1, q, W, H, ctl, part);
  else
    k_spmv_p<2><<<kRedBlocks, T, 0, st>>>(coef, z, P0, P1, q, W, H, ctl, part);
  FFB_LAUNCHED();
}

void pcg_update(int nc, double* x, double* r, const double* P0, const double* P1,
                const double* q, long long nvec, int max_iters, PcgCtl* ctl, double* part,
                cudaStream_t st) {
  if (nc == 3)
    k_update<3><<<kRedBlocks, T, 0, st>>>(x, r, P0, P1, q, nvec, max_iters, ctl, part);
  else
    k_update<2><<<kRedBlocks, T, 0, st>>>(x, r, P0, P1, q, nvec, max_iters, ctl, part);
  FFB_LAUNCHED();
}

}  // namespace ffb
