// C-ABI of flowfem_b200 (include/flowfem_b200.h) and the host orchestration of the hot
// path: run_on_frames (src/pipeline.cpp:38-78) under the converged-pass protocol, with the
// Schwarz-preconditioned CG of pcg.cu/band.cu as the linear solve.
//
// There is no CPU fallback: every numerical step runs in this library's CUDA kernels, and a
// missing or unusable device is an error.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/flowfem_b200.h"
#include "comm.hpp"
#include "ffb_internal.cuh"
#include "partition.hpp"

namespace ffb {

namespace {
thread_local std::string g_err;
std::atomic<long long> g_launches{0};
}  // namespace

void fail(const std::string& msg) { throw Error(msg); }

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  (void)file;
  (void)line;
  fail(std::string("cuda: ") + cudaGetErrorString(e) + " (" + what + ")");
}

void note_launch(long long n) { g_launches += n; }

// fill kernels live in operator.cu's translation unit family; declared here
void fill(double* p, double v, long long n, cudaStream_t st);
void debug_prof(unsigned long long* out, int reset);

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  T* ensure(size_t m) {
    if (m > n || !p) {
      release();
      const cudaError_t e = cudaMalloc(&p, std::max<size_t>(m, 1) * sizeof(T));
      if (e != cudaSuccess) {
        p = nullptr;
        cudaGetLastError();
        fail("cuda: out of device memory allocating " + std::to_string(m * sizeof(T)) +
             " bytes");
      }
      n = m;
    }
    return p;
  }
};

struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
};

}  // namespace ffb

using namespace ffb;

struct ffb_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  cudaStream_t own_st = nullptr;
  // problem on the device
  int W = 0, H = 0;
  size_t N = 0;
  long long ntri = 0;
  DBuf<double> t10, alpha, lambda, coef, b, x, r, z, p0, p1, q, eta, part, tmp, work, frames;
  DBuf<double> eta_hist;
  DBuf<double> xprev;  // the previous pass's solution (FFB_EXTRAP)
  DBuf<double> red;  // reduction scratch of the indicator / energy / compose kernels
  DBuf<int> bad_diag;
  DBuf<unsigned> counter;
  DBuf<PcgCtl> ctl;
  PcgCtl* h_ctl = nullptr;
  long long terms_version = 0, alpha_version = 0;
  long long coef_key_a = -1, coef_key_t = -1;
  int coef_nc = 0;
  long long rhs_key_t = -1;
  int rhs_nc = 0;
  long long factor_key_a = -1, factor_key_t = -1;
  // partition
  bool have_part = false;
  int part_px = 0, part_py = 0, part_ov = -1, part_nc = 0;
  Partition decomp;
  int nbf = 32, kd_max = 0, ccl = 1;
  // multi-GPU (comm.hpp): this rank's row band of subdomains; s_lo/s_hi = its subdomains
  std::unique_ptr<Comm> comm;
  RankRows rows{};
  int up = -1, dn = -1;  // nearest non-empty ranks above / below (-1: none)
  std::vector<size_t> gather_off, gather_cnt;  // owned rows of every rank, in doubles / W nc
  int s_lo = 0, s_hi = 0;
  // persistent ring solve (balance_chains): CTAs, and the task queue + forward-done counters
  int n_cta = 0;
  DBuf<int> qsync;
  DBuf<double> ur, urs, zs_up, zs_dn, zr_up, zr_dn;
  int stage_nc = 0, stage_max_iters = 0;
  double stage_tol = 0;
  SolvePlan plan{};
  std::vector<SubInfo> subs;
  DBuf<SubInfo> d_subs;
  DBuf<AxisMap> d_col, d_row;
  DBuf<double> fac, fac_t, dscratch, ylocal, zlocal, rlocal, xlocal, G0, G1, incs;
  // opt-in (ffb_set_factor_storage 32 / FFB_FACTOR_F32=1): the row-group tile solve streams a
  // single-precision copy of the line inverses (half the bytes per application); the
  // factorisation, the products and every CG vector stay in double
  int factor_bits = 64;
  DBuf<float> fac32;
  DBuf<int> own_col, own_row;
  // two-level coarse space (coarse.cu): core cuts, coarse node maps, A0 band + inverse
  bool coarse = true;
  int cbw = 0, n0 = 0, coarse_nc = 0;
  long long coarse_key_a = -1, coarse_key_t = -1;
  DBuf<int> d_xs, d_ys, d_ccol, d_crow, d_cbad;
  DBuf<double> cAB, cAinv, cgv, cyv;
  // linsolve boundary on an explicit CSR system (ffb_csr_*)
  DBuf<int> csr_rp, csr_ci, csr_perm, csr_iperm, csr_bad;
  DBuf<double> csr_v, csr_b, csr_x, csr_r, csr_z, csr_p, csr_Ap, csr_diag, csr_part, csr_AB;
  DBuf<CgCtl> cgctl;
  DBuf<int> a_f2v, a_v2f, a_rp;  // assemble(): the CSR pattern of the last system
  DBuf<double> a_g;
  // literal loop, CG subdomain mode: reference-order vectors + per-subdomain control blocks
  DBuf<double> b_x, b_b, b_r, b_z, b_p, b_Ap, b_part;
  DBuf<CgCtl> b_ctl;
  DBuf<double> alpha_fact;  // alpha of the resident factorisation (incremental refactor)
  DBuf<int2> d_changed;
  long long fact_key_t_full = -1;  // terms version / partition of the last full factorisation
  int fact_valid = 0;
  bool incremental = true;
  DBuf<int> d_bad;
  double factor_doubles = 0, apply_doubles = 0, sum_n = 0, factor_flops = 0;
  // asm kernel timing: a pool of event pairs, created on first use and reused (no event
  // creation inside a timed solve once the pool is warm)
  std::vector<EventPair> asm_events;
  size_t asm_used = 0;
  double asm_ms_total = 0;
  long long asm_launches_timed = 0;
  bool time_asm = false;

  ~ffb_ctx() {
    for (auto& e : asm_events) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    if (h_ctl) cudaFreeHost(h_ctl);
    if (own_st) cudaStreamDestroy(own_st);
  }
};

// SparseCholesky (linsolve.hpp:32-48) on the device: analyze = the reference's RCM ordering
// (bit-exact, host integer work) and the band width; factorize = band Cholesky of the
// permuted matrix on the device; solve = permuted forward/backward substitution.
struct ffb_chol {
  ffb_ctx* c = nullptr;
  int n = 0, nc = 3, bw = 0;
  long long nnz = 0;
  bool factored = false;
  DBuf<int> perm, iperm, rp, ci, bad;
  DBuf<double> v, AB, t, b;
};

namespace {

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  } catch (...) {
    g_err = "unknown error";
    return 1;
  }
}

void check_ctx(ffb_ctx* c) {
  if (!c) fail("ffb: null context");
  FFB_CUDA(cudaSetDevice(c->device));
}

void check_dims(int W, int H, const char* who) {
  if (W < 2 || H < 2) fail(std::string(who) + ": frames must be at least 2x2");
}

void set_problem(ffb_ctx* c, int W, int H) {
  if (c->W == W && c->H == H) return;
  c->W = W;
  c->H = H;
  c->N = static_cast<size_t>(W) * H;
  c->ntri = 2LL * (W - 1) * (H - 1);
  c->have_part = false;
  c->coef_key_a = c->coef_key_t = c->rhs_key_t = c->factor_key_a = c->factor_key_t = -1;
}

void upload(double* d, const double* h, size_t n, cudaStream_t st) {
  FFB_CUDA(cudaMemcpyAsync(d, h, n * sizeof(double), cudaMemcpyHostToDevice, st));
}
void download(double* h, const double* d, size_t n, cudaStream_t st) {
  FFB_CUDA(cudaMemcpyAsync(h, d, n * sizeof(double), cudaMemcpyDeviceToHost, st));
}
void sync(ffb_ctx* c) { FFB_CUDA(cudaStreamSynchronize(c->st)); }

// s0,s1 (2N) <- smooth(f0), smooth(f1); t10 <- data terms (imaging.cpp:33-138)
void frames_to_terms_dev(ffb_ctx* c, const double* f0, const double* f1, double sigma,
                         double rho) {
  const int W = c->W, H = c->H;
  const size_t N = c->N;
  double* s = c->work.ensure(2 * N);
  double* tmp = c->tmp.ensure(10 * N);
  smooth_planes(f0, s, tmp, W, H, 1, sigma, c->st);
  smooth_planes(f1, s + N, tmp, W, H, 1, sigma, c->st);
  double* t10 = c->t10.ensure(10 * N);
  double* tmp2 = c->coef.ensure(10 * N);  // large-radius path only; coefficients rebuilt after
  c->coef_key_a = c->coef_key_t = -1;
  data_terms(s, s + N, t10, tmp, tmp2, W, H, rho, c->st);
  c->terms_version++;
}

void ensure_coef(ffb_ctx* c, int nc) {
  if (c->coef_key_a == c->alpha_version && c->coef_key_t == c->terms_version && c->coef_nc == nc)
    return;
  c->coef.ensure(kCoefPlanes * c->N);
  int* bad = c->bad_diag.ensure(1);
  FFB_CUDA(cudaMemsetAsync(bad, 0x7f, sizeof(int), c->st));
  build_coef(c->t10.p, c->alpha.p, c->lambda.p, c->W, c->H, nc, c->coef.p, bad, c->st);
  int hbad = 0;
  FFB_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  if (hbad != 0x7f7f7f7f) fail("linsolve.cg: non-positive diagonal at row " + std::to_string(hbad));
  c->coef_key_a = c->alpha_version;
  c->coef_key_t = c->terms_version;
  c->coef_nc = nc;
}

void ensure_rhs(ffb_ctx* c, int nc) {
  if (c->rhs_key_t == c->terms_version && c->rhs_nc == nc) return;
  build_rhs(c->t10.p, c->W, c->H, nc, c->b.ensure(3 * c->N), c->st);
  c->rhs_key_t = c->terms_version;
  c->rhs_nc = nc;
}

// Row band of `rank`: subdomain rows [j0, j1) = [rank py / world, (rank+1) py / world), the
// core rows they own, the rows their free rectangles reach into the neighbours' bands, and
// the rows of this band the neighbours' subdomains cover (SURVEY §8e exchange sets).
RankRows rank_rows(const Partition& P, int rank, int world) {
  const int px = P.px, py = P.py;
  RankRows g{};
  g.j0 = static_cast<int>(static_cast<long long>(rank) * py / world);
  g.j1 = static_cast<int>(static_cast<long long>(rank + 1) * py / world);
  g.y0 = P.ys[g.j0];
  g.y1 = P.ys[g.j1];
  g.fa0 = g.fa1 = g.y0;
  g.fb0 = g.fb1 = g.y1;
  g.ra0 = g.ra1 = g.y0;
  g.rb0 = g.rb1 = g.y1;
  if (g.j1 == g.j0) return g;  // an empty rank (world > py)
  const Rect top = free_rect(P, g.j0 * px), bot = free_rect(P, (g.j1 - 1) * px);
  g.fa0 = std::min(top.y0, g.y0);
  g.fb1 = std::max(bot.y1, g.y1);
  if (g.j0 > 0) g.ra1 = std::min(free_rect(P, (g.j0 - 1) * px).y1, g.y1);
  if (g.j1 < py) g.rb0 = std::max(free_rect(P, g.j1 * px).y0, g.y0);
  if (g.fa1 - g.fa0 > 0 && g.j0 == 0) fail("schwarz: rank rows: free rows above the image");
  return g;
}

// Persistent ring solve with one CTA per chain (band.cu k_line_solve<M, true>): when the
// rank has more chains than SMs, one CTA per SM pulls the forward chains of every subdomain
// and then the backward chains from a queue, so the SMs stay busy through what would be a
// partly empty last round of one-chain-per-CTA launches (c4: 512 chains per sweep on 148 SMs
// = 3.46 rounds). FFB_NO_BALANCE=1 keeps the two launches per application.
void balance_chains(ffb_ctx* c) {
  c->n_cta = 0;
  if (c->plan.tile || c->ccl != 1 || std::getenv("FFB_NO_BALANCE")) return;
  int nsm = 0;
  FFB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
  const int nsub = c->s_hi - c->s_lo;
  if (nsm < 1 || 2 * nsub <= nsm) return;
  c->n_cta = nsm;
  c->qsync.ensure(nsub + 1);
}

void ensure_partition(ffb_ctx* c, int px, int py, int ov, int nc) {
  if (c->have_part && c->part_px == px && c->part_py == py && c->part_ov == ov &&
      c->part_nc == nc)
    return;
  c->have_part = false;
  c->factor_key_a = c->factor_key_t = -1;
  c->fact_valid = 0;
  const int W = c->W, H = c->H;
  c->decomp = build_partition(W, H, px, py, ov);
  const int np = px * py;
  std::vector<Rect> fr(np);
  int kd_max = 0;
  for (int p = 0; p < np; ++p) {
    fr[p] = free_rect(c->decomp, p);
    const int fw = fr[p].w(), fh = fr[p].h();
    kd_max = std::max(kd_max, nc * std::min(fw, fh));
  }
  c->kd_max = kd_max;
  c->nbf = kd_max > 512 ? 16 : 32;
  c->incremental = !std::getenv("FFB_FULL_REFACTOR");
  if (const char* e = std::getenv("FFB_NB")) {
    const int v = std::atoi(e);
    if (v == 16 || v == 32) c->nbf = v;
  }
  c->subs.assign(np, SubInfo{});
  // this rank's band of subdomain rows (all of them on a single GPU): subdomains
  // [s_lo, s_hi) are factored and solved here
  {
    const int rank = c->comm ? c->comm->rank : 0, world = c->comm ? c->comm->world : 1;
    c->rows = rank_rows(c->decomp, rank, world);
    c->s_lo = c->rows.j0 * px;
    c->s_hi = c->rows.j1 * px;
    c->up = c->dn = -1;
    c->gather_off.assign(world, 0);
    c->gather_cnt.assign(world, 0);
    const bool live = c->rows.j1 > c->rows.j0;  // a rank without subdomains exchanges nothing
    for (int q = 0; q < world; ++q) {
      const RankRows gq = rank_rows(c->decomp, q, world);
      c->gather_off[q] = static_cast<size_t>(gq.y0) * W * nc;
      c->gather_cnt[q] = static_cast<size_t>(gq.y1 - gq.y0) * W * nc;
      if (live && gq.j1 > gq.j0 && q < rank) c->up = q;
      if (live && gq.j1 > gq.j0 && q > rank && c->dn < 0) c->dn = q;
    }
  }
  // CTAs per subdomain solve (one thread-block cluster), from THIS rank's subdomains: enough
  // that ~128 SMs take part (2 chains per subdomain)
  {
    const int nown = std::max(1, c->s_hi - c->s_lo);
    c->ccl = 1;
    while (c->ccl < 8 && 2 * nown * c->ccl * 2 <= 160) c->ccl *= 2;
    if (const char* e = std::getenv("FFB_CLUSTER")) {
      const int v = std::atoi(e);
      if (v == 1 || v == 2 || v == 4 || v == 8) c->ccl = v;
    }
    c->plan = solve_plan(kd_max, c->ccl);
  }
  long long fac_off = 0, vec_off = 0, fac32_off = 0;
  double fd = 0, ad = 0, sn = 0, ff = 0;
  for (int p = 0; p < np; ++p) {
    SubInfo& s = c->subs[p];
    s.fx0 = fr[p].x0, s.fy0 = fr[p].y0, s.fw = fr[p].w(), s.fh = fr[p].h();
    if (s.fw < 1 || s.fh < 1) fail("schwarz.build_partition: empty subdomain");
    s.xfast = s.fw <= s.fh ? 1 : 0;
    s.S = s.xfast ? s.fw : s.fh;
    s.L = s.xfast ? s.fh : s.fw;
    s.kd = nc * s.S;
    const long long n = static_cast<long long>(s.kd) * s.L;
    if (n > (1LL << 30)) fail("schwarz: subdomain too large");
    s.n = static_cast<int>(n);
    s.line_sz = packed_line_size(s.kd);
    s.m = (s.L - 1) / 2;  // the middle line of the twisted factorisation
    s.fac_off = fac_off;
    s.vec_off = vec_off;
    s.fac32_off = fac32_off;
    if (p < c->s_lo || p >= c->s_hi) continue;  // another rank's subdomain: no storage here
    fac32_off += (((s.line_sz + 3) & ~3LL) * s.L + 31) / 32 * 32;
    fac_off += (s.line_sz * s.L + 31) / 32 * 32;
    vec_off += (n + 31) / 32 * 32;
    fd += static_cast<double>(s.line_sz) * s.L;
    ff += static_cast<double>(n) * s.kd * s.kd;  // 2 flops x n kd^2 / 2 FMAs
    ad += static_cast<double>(s.line_sz) * (2 * s.L - 1);  // forward all, backward L-1 lines
    sn += static_cast<double>(n);
  }
  c->factor_doubles = fd;
  c->factor_flops = ff;
  balance_chains(c);
  c->apply_doubles = ad;
  c->sum_n = sn;
  // free-rectangle membership along each axis (free rect of part (i,j) = X_i x Y_j)
  std::vector<AxisMap> col(W, AxisMap{-1, 0, -1, 0}), row(H, AxisMap{-1, 0, -1, 0});
  for (int i = 0; i < px; ++i) {
    const Rect& f = fr[i];
    for (int x = f.x0; x < f.x1; ++x) {
      AxisMap& m = col[x];
      if (m.p0 < 0) m.p0 = i, m.l0 = x - f.x0;
      else if (m.p1 < 0) m.p1 = i, m.l1 = x - f.x0;
      else fail("schwarz: more than two overlapping parts along x");
    }
  }
  for (int j = 0; j < py; ++j) {
    const Rect& f = fr[j * px];
    for (int y = f.y0; y < f.y1; ++y) {
      AxisMap& m = row[y];
      if (m.p0 < 0) m.p0 = j, m.l0 = y - f.y0;
      else if (m.p1 < 0) m.p1 = j, m.l1 = y - f.y0;
      else fail("schwarz: more than two overlapping parts along y");
    }
  }
  for (int x = 0; x < W; ++x)
    if (col[x].p0 < 0) fail("schwarz: column not covered by any subdomain");
  for (int y = 0; y < H; ++y)
    if (row[y].p0 < 0) fail("schwarz: row not covered by any subdomain");
  c->d_subs.ensure(np);
  c->d_col.ensure(W);
  c->d_row.ensure(H);
  FFB_CUDA(cudaMemcpyAsync(c->d_subs.p, c->subs.data(), np * sizeof(SubInfo),
                           cudaMemcpyHostToDevice, c->st));
  FFB_CUDA(cudaMemcpyAsync(c->d_col.p, col.data(), W * sizeof(AxisMap), cudaMemcpyHostToDevice,
                           c->st));
  FFB_CUDA(cudaMemcpyAsync(c->d_row.p, row.data(), H * sizeof(AxisMap), cudaMemcpyHostToDevice,
                           c->st));
  c->fac.ensure(fac_off);
  if (c->plan.tile) c->fac_t.ensure(fac_off);  // tile-major copy for the register-tiled solve
  if (c->factor_bits == 32 && c->plan.rt) c->fac32.ensure(fac32_off + 32);
  else c->fac32.release();
  c->dscratch.ensure(factor_scratch_doubles(c->s_hi - c->s_lo, kd_max));
  c->ylocal.ensure(vec_off);
  c->zlocal.ensure(vec_off);
  c->d_bad.ensure(np);
  // coarse space: core cuts and the coarse node of every pixel's core, the shorter subdomain
  // axis fastest (A0's bandwidth is then nc * min(px, py))
  {
    // opt-in (FFB_COARSE=1): measured to cost iterations on every config (c4 400 -> 488,
    // c3 260 -> 338, c2 176 -> 226, c5 214 -> 259; profiles/r2_coarse_space.txt)
    const char* e = std::getenv("FFB_COARSE");
    c->coarse = e && std::atoi(e) == 1;
    c->coarse_key_a = c->coarse_key_t = -1;
    const Partition& P = c->decomp;
    std::vector<int> ccol(W), crow(H);
    const bool yfast = py <= px;
    for (int x = 0; x < W; ++x) {
      const int ix = int(std::upper_bound(P.xs.begin(), P.xs.end(), x) - P.xs.begin()) - 1;
      ccol[x] = yfast ? ix * py : ix;
    }
    for (int y = 0; y < H; ++y) {
      const int iy = int(std::upper_bound(P.ys.begin(), P.ys.end(), y) - P.ys.begin()) - 1;
      crow[y] = yfast ? iy : iy * px;
    }
    c->cbw = nc * (yfast ? py : px);
    c->n0 = nc * np;
    FFB_CUDA(cudaMemcpyAsync(c->d_xs.ensure(px + 1), P.xs.data(), (px + 1) * sizeof(int),
                             cudaMemcpyHostToDevice, c->st));
    FFB_CUDA(cudaMemcpyAsync(c->d_ys.ensure(py + 1), P.ys.data(), (py + 1) * sizeof(int),
                             cudaMemcpyHostToDevice, c->st));
    FFB_CUDA(cudaMemcpyAsync(c->d_ccol.ensure(W), ccol.data(), W * sizeof(int),
                             cudaMemcpyHostToDevice, c->st));
    FFB_CUDA(cudaMemcpyAsync(c->d_crow.ensure(H), crow.data(), H * sizeof(int),
                             cudaMemcpyHostToDevice, c->st));
  }
  sync(c);
  c->have_part = true;
  c->part_px = px, c->part_py = py, c->part_ov = ov, c->part_nc = nc;
}

void ensure_factor(ffb_ctx* c, int nc) {
  if (!c->have_part) fail("schwarz: no partition set");
  if (c->part_nc != nc) ensure_partition(c, c->part_px, c->part_py, c->part_ov, nc);
  if (c->factor_key_a == c->alpha_version && c->factor_key_t == c->terms_version) return;
  ensure_coef(c, nc);
  const int np = c->s_hi - c->s_lo;
  FFB_CUDA(cudaMemsetAsync(c->d_bad.p, 0x7f, np * sizeof(int), c->st));
  // Only alpha changed since the last (successful) factorisation of this partition and these
  // terms: refactor each chain from the first line the change touches (exact).
  const bool incr = c->incremental && c->fact_valid && c->factor_key_t == c->terms_version &&
                    c->alpha_fact.p != nullptr;
  const int2* changed = nullptr;
  c->fact_valid = 0;  // until this factorisation has succeeded
  if (incr) {
    int2* ch = c->d_changed.ensure(np);
    changed_lines(c->d_subs.p + c->s_lo, np, c->alpha.p, c->alpha_fact.p, c->W, c->H, ch, c->st);
    changed = ch;
  }
  line_factor(c->d_subs.p + c->s_lo, np, c->ccl, c->nbf, c->kd_max, c->coef.p, c->N, c->W, nc,
              c->fac.p, c->dscratch.p, static_cast<long long>(c->kd_max) * c->kd_max, c->d_bad.p,
              c->st, changed, c->plan.tile ? c->fac_t.p : nullptr);
  if (c->fac32.p)
    factor_to_f32(c->d_subs.p + c->s_lo, np, c->fac.p, c->fac32.p, changed, c->st);
  FFB_CUDA(cudaMemcpyAsync(c->alpha_fact.ensure(c->ntri), c->alpha.p, c->ntri * sizeof(double),
                           cudaMemcpyDeviceToDevice, c->st));
  std::vector<int> bad(np);
  FFB_CUDA(cudaMemcpyAsync(bad.data(), c->d_bad.p, np * sizeof(int), cudaMemcpyDeviceToHost,
                           c->st));
  sync(c);
  for (int p = 0; p < np; ++p)
    if (bad[p] != 0x7f7f7f7f)
      fail("linsolve.cholesky: breakdown at pivot " + std::to_string(bad[p]) + " of subdomain " +
           std::to_string(p + c->s_lo) + ": matrix is not positive definite");
  c->factor_key_a = c->alpha_version;
  c->factor_key_t = c->terms_version;
  c->fact_valid = 1;
}

// A0 = Z^T A Z of the current operator, factored and inverted on the device (coarse.cu)
void ensure_coarse(ffb_ctx* c, int nc) {
  if (!c->coarse) return;
  if (c->coarse_key_a == c->alpha_version && c->coarse_key_t == c->terms_version &&
      c->coarse_nc == nc)
    return;
  ensure_coef(c, nc);
  const int px = c->part_px, py = c->part_py;
  c->n0 = nc * px * py;
  c->cbw = nc * std::min(px, py);
  int* bad = c->d_cbad.ensure(1);
  FFB_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(int), c->st));
  coarse_build(c->coef.p, c->W, c->H, nc, c->d_xs.p, c->d_ys.p, px, py, c->d_ccol.p, c->d_crow.p,
               c->cbw, c->cAB.ensure(static_cast<size_t>(c->n0) * (c->cbw + 1)),
               c->cAinv.ensure(static_cast<size_t>(c->n0) * c->n0), bad, c->st);
  c->cgv.ensure(c->n0);
  c->cyv.ensure(c->n0);
  int hbad = -1;
  FFB_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  if (hbad >= 0)
    fail("linsolve.cholesky: breakdown at pivot " + std::to_string(hbad) +
         " of the coarse problem: matrix is not positive definite");
  c->coarse_key_a = c->alpha_version;
  c->coarse_key_t = c->terms_version;
  c->coarse_nc = nc;
}

// y = A0^-1 Z^T r for the combine kernel (nullptr without a coarse space; single GPU only)
const double* coarse_term(ffb_ctx* c, int nc, const double* r, const PcgCtl* ctl) {
  if (!c->coarse || (c->comm && c->comm->world > 1)) return nullptr;
  coarse_apply(r, c->W, nc, c->d_xs.p, c->d_ys.p, c->part_px, c->part_py, c->d_ccol.p,
               c->d_crow.p, c->cAinv.p, c->cgv.p, c->cyv.p, ctl, c->st);
  return c->cyv.p;
}

// the factor layout the subdomain solve streams: the tile-major copy for the register-tiled
// kernel, else the packed rows
const double* solve_factor(const ffb_ctx* c) { return c->plan.tile ? c->fac_t.p : c->fac.p; }

void launch_asm(ffb_ctx* c, int nc, const double* rvec, const int* flags) {
  EventPair* ev = nullptr;
  if (c->time_asm) {
    if (c->asm_used == c->asm_events.size()) {
      EventPair e;
      FFB_CUDA(cudaEventCreate(&e.a));
      FFB_CUDA(cudaEventCreate(&e.b));
      c->asm_events.push_back(e);
    }
    ev = &c->asm_events[c->asm_used++];
    FFB_CUDA(cudaEventRecord(ev->a, c->st));
  }
  line_solve(c->d_subs.p + c->s_lo, c->s_hi - c->s_lo, c->plan, solve_factor(c), c->coef.p, c->N, rvec,
             c->ylocal.p, c->zlocal.p, c->W, nc, flags, c->st, nullptr,
             c->n_cta ? c->qsync.p : nullptr, c->n_cta, c->fac32.p);
  if (ev) FFB_CUDA(cudaEventRecord(ev->b, c->st));
}

void harvest_asm_events(ffb_ctx* c) {
  for (size_t k = 0; k < c->asm_used; ++k) {
    const EventPair& e = c->asm_events[k];
    float ms = 0;
    FFB_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
    // kernels that returned at entry (converged) take ~2 us; count real applications only
    if (ms > 0.02f) {
      c->asm_ms_total += ms;
      c->asm_launches_timed++;
    }
  }
  c->asm_used = 0;
}

struct PcgResult {
  int iters;
  double res;
};

// Schwarz-preconditioned CG on the resident system, x warm or zero.
// rows [a, b) of an interleaved nc-component vector as an exchange slice
Xfer rows_xfer(double* v, int W, int nc, int a, int b, int peer, int send) {
  return Xfer{peer, send, v + static_cast<size_t>(a) * W * nc,
              static_cast<size_t>(std::max(0, b - a)) * W * nc};
}

// One scalar reduction's completion: world 1 finished it inside the kernel (finish = 1);
// otherwise all-reduce the unit values and sum them in unit order on every rank.
void reduce_scalar(ffb_ctx* c, int stage, int nvals) {
  if (!c->comm || c->comm->world == 1) return;
  // out of place: ur keeps zeros outside this rank's units, urs receives the sum
  double* urs = c->urs.ensure(2 * static_cast<size_t>(c->part_py));
  c->comm->allreduce_sum(c->ur.p, urs, static_cast<size_t>(nvals) * c->part_py, c->st);
  pcg_scalar(urs, c->part_py, stage, c->ctl.p, c->st);
}

// z = M^-1 r on the owned rows: r halo -> subdomain solves -> partial sums for the
// neighbours -> combine (+ r.z) -> z halo (one row), SURVEY §8e steps 1-3
void precondition(ffb_ctx* c, int nc, const int* flags, int fin) {
  const bool multi = c->comm && c->comm->world > 1;
  const RankRows& g = c->rows;
  const int W = c->W;
  double* r = c->r.p;
  double* z = c->z.p;
  PcgCtl* ctl = c->ctl.p;
  if (multi) {  // r on the rows my subdomains reach into; mine to the neighbours
    Xfer x[4];
    int n = 0;
    if (c->up >= 0) {
      x[n++] = rows_xfer(r, W, nc, g.ra0, g.ra1, c->up, 1);
      x[n++] = rows_xfer(r, W, nc, g.fa0, g.fa1, c->up, 0);
    }
    if (c->dn >= 0) {
      x[n++] = rows_xfer(r, W, nc, g.rb0, g.rb1, c->dn, 1);
      x[n++] = rows_xfer(r, W, nc, g.fb0, g.fb1, c->dn, 0);
    }
    c->comm->exchange(x, n, c->st);
  }
  launch_asm(c, nc, r, flags);
  const double* yc = multi ? nullptr : coarse_term(c, nc, r, ctl);
  if (multi) {  // this rank's subdomain sums on the neighbours' rows, theirs on mine
    pcg_zpart(nc, c->d_subs.p, c->d_col.p, c->d_row.p, c->part_px, c->zlocal.p, W, g, c->zs_up.p,
              c->zs_dn.p, ctl, c->st);
    Xfer x[4];
    int n = 0;
    if (c->up >= 0) {
      x[n++] = Xfer{c->up, 1, c->zs_up.p, static_cast<size_t>(g.fa1 - g.fa0) * W * nc};
      x[n++] = Xfer{c->up, 0, c->zr_up.p, static_cast<size_t>(g.ra1 - g.ra0) * W * nc};
    }
    if (c->dn >= 0) {
      x[n++] = Xfer{c->dn, 1, c->zs_dn.p, static_cast<size_t>(g.fb1 - g.fb0) * W * nc};
      x[n++] = Xfer{c->dn, 0, c->zr_dn.p, static_cast<size_t>(g.rb1 - g.rb0) * W * nc};
    }
    c->comm->exchange(x, n, c->st);
  }
  pcg_combine(nc, c->d_subs.p, c->d_col.p, c->d_row.p, c->part_px, c->zlocal.p, r, z, W, g,
              c->d_ys.p, c->part_py, c->zr_up.p, c->zr_dn.p, ctl, c->part.p, c->ur.p, fin, c->st,
              yc, c->d_ccol.p, c->d_crow.p);
  reduce_scalar(c, pcg_stage_rz(), 1);
  if (multi) {  // one row of z each side for the next operator application
    Xfer x[4];
    int n = 0;
    if (c->up >= 0) {
      x[n++] = rows_xfer(z, W, nc, g.y0, g.y0 + 1, c->up, 1);
      x[n++] = rows_xfer(z, W, nc, g.y0 - 1, g.y0, c->up, 0);
    }
    if (c->dn >= 0) {
      x[n++] = rows_xfer(z, W, nc, g.y1 - 1, g.y1, c->dn, 1);
      x[n++] = rows_xfer(z, W, nc, g.y1, g.y1 + 1, c->dn, 0);
    }
    c->comm->exchange(x, n, c->st);
  }
}

// Schwarz-preconditioned CG on the resident system, x warm or zero. With a communicator the
// rank works on its row band (pcg.cu) and x is all-gathered at the end, so every rank holds
// the whole solution; the iterates are bitwise those of the single-GPU solve.
PcgResult pcg(ffb_ctx* c, int nc, double tol, int max_iters, bool warm) {
  ensure_coef(c, nc);
  ensure_rhs(c, nc);
  ensure_factor(c, nc);
  ensure_coarse(c, nc);
  const size_t N = c->N;
  const long long nvec = static_cast<long long>(N) * nc;
  const bool multi = c->comm && c->comm->world > 1;
  const int fin = multi ? 0 : 1;
  const RankRows& g = c->rows;
  const int W = c->W, py = c->part_py;
  double* x = c->x.ensure(3 * N);
  double* r = c->r.ensure(3 * N);
  double* z = c->z.ensure(3 * N);
  double* P0 = c->p0.ensure(3 * N);
  double* P1 = c->p1.ensure(3 * N);
  double* q = c->q.ensure(3 * N);
  c->part.ensure(2 * static_cast<size_t>(std::max(1, g.j1 - g.j0)) * kCU);
  double* ur = c->ur.ensure(2 * static_cast<size_t>(py));
  FFB_CUDA(cudaMemsetAsync(ur, 0, 2 * py * sizeof(double), c->st));  // zero off this rank's units
  const size_t row = static_cast<size_t>(W) * nc;
  c->zs_up.ensure(std::max(1, g.fa1 - g.fa0) * row);
  c->zs_dn.ensure(std::max(1, g.fb1 - g.fb0) * row);
  c->zr_up.ensure(std::max(1, g.ra1 - g.ra0) * row);
  c->zr_dn.ensure(std::max(1, g.rb1 - g.rb0) * row);
  PcgCtl* ctl = c->ctl.ensure(1);
  if (!c->h_ctl) FFB_CUDA(cudaMallocHost(&c->h_ctl, sizeof(PcgCtl)));
  if (!warm) FFB_CUDA(cudaMemsetAsync(x, 0, nvec * sizeof(double), c->st));
  if (max_iters <= 0) max_iters = static_cast<int>(std::min<long long>(10 * nvec, 1 << 30));
  std::memset(c->h_ctl, 0, sizeof(PcgCtl));
  c->h_ctl->tol = tol;
  c->h_ctl->max_iters = max_iters;
  FFB_CUDA(cudaMemcpyAsync(ctl, c->h_ctl, sizeof(PcgCtl), cudaMemcpyHostToDevice, c->st));
  const int* flags = &ctl->done;
  pcg_init(nc, c->coef.p, c->b.p, x, r, W, c->H, g, c->d_ys.p, py, ctl, c->part.p, ur, fin, c->st);
  reduce_scalar(c, pcg_stage_init(), 2);
  precondition(c, nc, flags, fin);
  const int chunk = 8;
  for (;;) {
    for (int it = 0; it < chunk; ++it) {
      pcg_spmv_p(nc, c->coef.p, z, P0, P1, q, W, c->H, g, c->d_ys.p, py, ctl, c->part.p, ur, fin,
                 c->st);
      reduce_scalar(c, pcg_stage_pap(), 1);
      pcg_update(nc, x, r, P0, P1, q, W, g, c->d_ys.p, py, ctl, c->part.p, ur, fin, c->st);
      reduce_scalar(c, pcg_stage_rr(), 1);
      precondition(c, nc, flags, fin);
    }
    FFB_CUDA(cudaMemcpyAsync(c->h_ctl, ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    if (c->time_asm) harvest_asm_events(c);
    if (c->h_ctl->done || c->h_ctl->err) break;
  }
  const PcgCtl& h = *c->h_ctl;
  if (h.err)
    fail("linsolve.cg: indefinite matrix detected at iteration " + std::to_string(h.err_it));
  if (h.zero_rhs) {
    FFB_CUDA(cudaMemsetAsync(x, 0, nvec * sizeof(double), c->st));
    return {0, 0.0};
  }
  if (multi)  // every rank's owned rows of x to every rank
    c->comm->allgather_rows(x, c->gather_off.data(), c->gather_cnt.data(), c->st);
  if (!(h.res <= tol)) {
    char buf[160];
    std::snprintf(buf, sizeof buf,
                  "linsolve.cg: no convergence after %d iterations, relative residual %f",
                  h.iters, h.res);
    fail(buf);
  }
  return {h.iters, h.res};
}

void ensure_reg(ffb_ctx* c) {
  c->alpha.ensure(c->ntri);
  c->lambda.ensure(c->ntri);
}

// run_on_frames, converged-pass protocol: n_passes x {solve, indicator,
// update} + final solve; frames and u3 on the device.
void run_dev(ffb_ctx* c, int W, int H, const double* f0, const double* f1,
             const ffb_run_config* cfg, double* d_u3, ffb_run_stats* stats) {
  if (!cfg) fail("cli.run: null config");
  check_dims(W, H, "cli.run");
  set_problem(c, W, H);
  const int nc = cfg->illumination ? 3 : 2;
  const int n_passes = cfg->adapt ? std::max(0, cfg->n_passes) : 0;
  if (n_passes + 1 > FFB_MAX_SOLVES) fail("cli.run: too many adaptive passes");
  cudaEvent_t ev[6];
  for (auto& e : ev) FFB_CUDA(cudaEventCreate(&e));
  FFB_CUDA(cudaEventRecord(ev[0], c->st));
  frames_to_terms_dev(c, f0, f1, cfg->sigma, cfg->rho);
  ensure_reg(c);
  fill(c->alpha.p, cfg->alpha0, c->ntri, c->st);
  fill(c->lambda.p, cfg->lambda0, c->ntri, c->st);
  c->alpha_version++;
  c->fact_valid = 0;
  const Split sp = choose_split(W, H, cfg->parts);
  ensure_partition(c, sp.px, sp.py, cfg->overlap, nc);
  FFB_CUDA(cudaEventRecord(ev[1], c->st));
  // alpha_th NaN = unset (std::optional, pipeline.cpp:71); explicit values, 0 included, are the floor
  const double alpha_th = std::isnan(cfg->alpha_th) ? cfg->alpha0 / 100.0 : cfg->alpha_th;
  double* eh = c->eta_hist.ensure(FFB_MAX_SOLVES);
  double* eta = c->eta.ensure(c->ntri);
  double* blockmax = c->red.ensure(4 * kRedBlocks);
  unsigned* counter = c->counter.ensure(1);
  FFB_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), c->st));
  double ms_factor = 0, ms_pcg = 0, ms_adapt = 0, ms_factor0 = 0;
  // Warm start of pass p >= 2: x_{p-1} + theta (x_{p-1} - x_{p-2}), theta = 0.75 — the
  // solution moves the same way from pass to pass as alpha keeps shrinking in the same places
  // (measured: c4 400 -> 378 PCG iterations per chain, c3 260 -> 242; theta 0.5 / 1.0 / 1.5,
  // profiles/r2_warm_start.txt). Each pass still converges to tol, so the result is the same
  // to the solve tolerance. FFB_EXTRAP=theta overrides, FFB_EXTRAP=-1 warm-starts plainly.
  const double extrap = std::getenv("FFB_EXTRAP") ? std::atof(std::getenv("FFB_EXTRAP")) : 0.75;
  long long total_it = 0;
  c->asm_ms_total = 0;
  c->asm_launches_timed = 0;
  c->time_asm = stats != nullptr;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->parts_x = sp.px;
    stats->parts_y = sp.py;
    stats->n_solves = n_passes + 1;
  }
  for (int pass = 0; pass <= n_passes; ++pass) {
    FFB_CUDA(cudaEventRecord(ev[2], c->st));
    ensure_factor(c, nc);
    FFB_CUDA(cudaEventRecord(ev[3], c->st));
    if (pass > 0 && extrap >= 0.0)  // warm start: the last solution, extrapolated
      vec_extrapolate(c->x.p, c->xprev.ensure(3 * c->N), static_cast<long long>(c->N) * nc,
                      pass > 1 ? extrap : 0.0, c->st);
    const PcgResult pr = pcg(c, nc, cfg->tol, cfg->max_iters, pass > 0);
    FFB_CUDA(cudaEventRecord(ev[4], c->st));
    total_it += pr.iters;
    if (stats) {
      stats->iters[pass] = pr.iters;
      stats->residual[pass] = pr.res;
    }
    if (pass < n_passes) {
      double* u3 = c->work.ensure(3 * c->N);
      inter_to_planes(c->x.p, u3, static_cast<long long>(c->N), nc, c->st);
      error_indicator(c->t10.p, c->alpha.p, c->lambda.p, u3, W, H, nc, eta, eh + pass,
                      blockmax, counter, c->st);
      update_alpha(c->alpha.p, c->alpha.p, eta, eh + pass, c->ntri, cfg->kappa,
                   cfg->eta_threshold, alpha_th, c->st);
      c->alpha_version++;
    }
    FFB_CUDA(cudaEventRecord(ev[5], c->st));
    sync(c);
    float a = 0, b = 0, d = 0;
    FFB_CUDA(cudaEventElapsedTime(&a, ev[2], ev[3]));
    FFB_CUDA(cudaEventElapsedTime(&b, ev[3], ev[4]));
    FFB_CUDA(cudaEventElapsedTime(&d, ev[4], ev[5]));
    if (pass == 0) ms_factor0 = a;  // the full factorisation (later passes are incremental)
    ms_factor += a, ms_pcg += b, ms_adapt += d;
  }
  inter_to_planes(c->x.p, d_u3, static_cast<long long>(c->N), nc, c->st);
  FFB_CUDA(cudaEventRecord(ev[5], c->st));
  sync(c);
  c->time_asm = false;
  if (stats) {
    float t_terms = 0, t_total = 0;
    FFB_CUDA(cudaEventElapsedTime(&t_terms, ev[0], ev[1]));
    FFB_CUDA(cudaEventElapsedTime(&t_total, ev[0], ev[5]));
    if (n_passes > 0)
      FFB_CUDA(cudaMemcpy(stats->eta_max, eh, n_passes * sizeof(double), cudaMemcpyDeviceToHost));
    stats->pcg_iterations = total_it;
    stats->ms_terms = t_terms;
    stats->ms_factor = ms_factor;
    stats->ms_pcg = ms_pcg;
    stats->ms_adapt = ms_adapt;
    stats->ms_total = t_total;
    // algorithmic bytes of one PCG iteration: the packed line inverses streamed forward
    // (all lines) and backward (all but the last) + the vector kernels (coefficients
    // 80 B/px, ~14 vector passes of nc doubles)
    stats->factor_doubles = c->apply_doubles;
    stats->iter_bytes = 8.0 * c->apply_doubles + (80.0 + 14.0 * 8.0 * nc) * c->N;
    stats->ms_asm_per_iter =
        c->asm_launches_timed ? c->asm_ms_total / c->asm_launches_timed : 0.0;
    stats->ms_factor_full = ms_factor0;
    stats->factor_flops = c->factor_flops;
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

}  // namespace

// ===================================================================== C-ABI
extern "C" {

const char* ffb_last_error(void) { return g_err.c_str(); }
int ffb_abi_version(void) { return FFB_ABI_VERSION; }
long long ffb_kernel_launches(void) { return g_launches.load(); }

int ffb_create(ffb_ctx** out, int device) {
  return guard([&] {
    if (!out) fail("ffb: null output pointer");
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      fail("ffb: no CUDA device available (this library has no CPU fallback)");
    }
    if (device < 0 || device >= n) fail("ffb: device index out of range");
    cudaDeviceProp prop{};
    FFB_CUDA(cudaGetDeviceProperties(&prop, device));
    // the library ships sm_100a cubins only (no PTX): refuse other devices up front instead of
    // failing at the first launch with "no kernel image"
    if (prop.major != 10 || prop.minor != 0)
      fail("ffb: requires a compute capability 10.0 (B200, sm_100a) device; found " +
           std::to_string(prop.major) + "." + std::to_string(prop.minor));
    auto c = std::make_unique<ffb_ctx>();
    c->device = device;
    if (const char* e = std::getenv("FFB_FACTOR_F32")) c->factor_bits = std::atoi(e) ? 32 : 64;
    FFB_CUDA(cudaSetDevice(device));
    FFB_CUDA(cudaStreamCreateWithFlags(&c->own_st, cudaStreamNonBlocking));
    c->st = c->own_st;
    *out = c.release();
  });
}

int ffb_destroy(ffb_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->st);
    delete ctx;
  });
}

// development probe: clock64 phase accumulators of the factor/solve kernels (zeros unless
// built with FFB_PROFILE=1); not part of the public header
int ffb_debug_prof(unsigned long long* out64, int reset) {
  return guard([&] { debug_prof(out64, reset); });
}

// development probe: which subdomain-solve kernel the resident partition uses (1 the
// register-tiled k_line_solve_tile, 2 the row-group tile ring k_line_solve_rt, 0 the
// row-batch ring k_line_solve, -1 none yet)
int ffb_debug_solve_kernel(ffb_ctx* c) {
  if (!c || !c->have_part) return -1;
  return c->plan.tile ? 1 : (c->plan.rt ? 2 : 0);
}

// development probe (host only, no device needed): the subdomain-solve plan for a widest
// line of kd_max unknowns on C-CTA clusters — tile (1: register-tiled, 2: row-group tile
// ring, 0: row-batch ring), its dynamic
// shared memory and, for the tiled kernel, the per-CTA line stage in doubles
int ffb_debug_solve_plan(int kd_max, int C, int* tile, long long* smem, int* stage) {
  return guard([&] {
    const SolvePlan pl = solve_plan(kd_max, C);
    if (tile) *tile = pl.tile ? 1 : (pl.rt ? 2 : 0);
    if (smem) *smem = static_cast<long long>(pl.smem);
    if (stage) *stage = pl.tile ? pl.stage_doubles : 0;
  });
}

// development probe: average time of `n` applications of the Schwarz preconditioner with
// the context's resident factorisation (after a solve), on the current residual vector
int ffb_debug_time_asm(ffb_ctx* c, int nc, int n, int dbg, double* ms) {
  return guard([&] {
    check_ctx(c);
    if (!c->have_part || !c->r.p) fail("ffb_debug_time_asm: no resident factorisation");
    cudaEvent_t a, b;
    FFB_CUDA(cudaEventCreate(&a));
    FFB_CUDA(cudaEventCreate(&b));
    set_solve_dbg(dbg);
    launch_asm(c, nc, c->r.p, nullptr);
    FFB_CUDA(cudaEventRecord(a, c->st));
    for (int i = 0; i < n; ++i) launch_asm(c, nc, c->r.p, nullptr);
    FFB_CUDA(cudaEventRecord(b, c->st));
    FFB_CUDA(cudaEventSynchronize(b));
    float t = 0;
    FFB_CUDA(cudaEventElapsedTime(&t, a, b));
    *ms = t / n;
    set_solve_dbg(0);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

int ffb_set_factor_storage(ffb_ctx* c, int bits) {
  return guard([&] {
    check_ctx(c);
    if (bits != 64 && bits != 32) fail("ffb_set_factor_storage: bits must be 64 or 32");
    if (bits == c->factor_bits) return;
    sync(c);
    c->factor_bits = bits;
    if (c->have_part) {  // rebuild the resident partition's storage; the next solve refactors
      c->have_part = false;
      ensure_partition(c, c->part_px, c->part_py, c->part_ov, c->part_nc);
    }
  });
}

int ffb_get_factor_storage(ffb_ctx* c, int* bits, int* in_use) {
  return guard([&] {
    check_ctx(c);
    if (bits) *bits = c->factor_bits;
    if (in_use) *in_use = c->fac32.p ? 32 : 64;  // 32 only where the row-group tile solve runs
  });
}

int ffb_set_stream(ffb_ctx* c, void* stream, int own) {
  return guard([&] {
    check_ctx(c);
    FFB_CUDA(cudaStreamSynchronize(c->st));
    c->st = own ? c->own_st : static_cast<cudaStream_t>(stream);
  });
}

int ffb_gaussian_smooth(ffb_ctx* c, int W, int H, const double* in, double sigma, double* out) {
  return guard([&] {
    check_ctx(c);
    if (W < 1 || H < 1) fail("imaging.gaussian_smooth: empty image");
    const size_t N = static_cast<size_t>(W) * H;
    double* d = c->work.ensure(2 * N);
    double* tmp = c->tmp.ensure(N);
    upload(d, in, N, c->st);
    smooth_planes(d, d + N, tmp, W, H, 1, sigma, c->st);
    download(out, d + N, N, c->st);
    sync(c);
  });
}

int ffb_compute_derivatives(ffb_ctx* c, int W, int H, const double* f0, const double* f1,
                            double* fx, double* fy, double* ft, double* f) {
  return guard([&] {
    check_ctx(c);
    check_dims(W, H, "imaging.compute_derivatives");
    const size_t N = static_cast<size_t>(W) * H;
    double* d = c->tmp.ensure(6 * N);
    upload(d, f0, N, c->st);
    upload(d + N, f1, N, c->st);
    derivatives4(d, d + N, d + 2 * N, d + 3 * N, d + 4 * N, d + 5 * N, W, H, c->st);
    download(fx, d + 2 * N, N, c->st);
    download(fy, d + 3 * N, N, c->st);
    download(ft, d + 4 * N, N, c->st);
    download(f, d + 5 * N, N, c->st);
    sync(c);
  });
}

int ffb_build_data_terms(ffb_ctx* c, int W, int H, const double* fx, const double* fy,
                         const double* ft, const double* f, double rho, double* out10) {
  return guard([&] {
    check_ctx(c);
    const size_t N = static_cast<size_t>(W) * H;
    double* in4 = c->work.ensure(4 * N);
    double* t10 = c->tmp.ensure(10 * N);
    double* scratch = c->frames.ensure(20 * N);  // large-radius path only
    upload(in4, fx, N, c->st);
    upload(in4 + N, fy, N, c->st);
    upload(in4 + 2 * N, ft, N, c->st);
    upload(in4 + 3 * N, f, N, c->st);
    data_terms_from4(in4, in4 + N, in4 + 2 * N, in4 + 3 * N, t10, scratch,
                     scratch + 10 * N, W, H, rho, c->st);
    download(out10, t10, 10 * N, c->st);
    sync(c);
  });
}

int ffb_frames_to_terms(ffb_ctx* c, int W, int H, const double* f0, const double* f1,
                        double sigma, double rho, double* out10) {
  return guard([&] {
    check_ctx(c);
    check_dims(W, H, "imaging.compute_derivatives");
    set_problem(c, W, H);
    double* fr = c->frames.ensure(2 * c->N);
    upload(fr, f0, c->N, c->st);
    upload(fr + c->N, f1, c->N, c->st);
    frames_to_terms_dev(c, fr, fr + c->N, sigma, rho);
    download(out10, c->t10.p, 10 * c->N, c->st);
    sync(c);
  });
}

int ffb_enumerate_splits(int W, int H, int n_parts, int* px, int* py, double* ratio, int cap) {
  int count = -1;
  if (guard([&] {
        const auto all = enumerate_splits(W, H, n_parts);
        count = 0;
        for (const auto& s : all) {
          if (count >= cap) break;
          px[count] = s.px, py[count] = s.py, ratio[count] = s.ratio;
          ++count;
        }
      }))
    return -1;
  return count;
}

int ffb_choose_split(int W, int H, int n_parts, int* px, int* py, double* ratio) {
  return guard([&] {
    const Split s = choose_split(W, H, n_parts);
    *px = s.px, *py = s.py, *ratio = s.ratio;
  });
}

long ffb_build_partition(int W, int H, int px, int py, int ov, int* buf, long cap) {
  long need = -1;
  if (guard([&] {
        const std::vector<int> flat = flatten(build_partition(W, H, px, py, ov));
        need = static_cast<long>(flat.size());
        if (buf && cap >= need) std::memcpy(buf, flat.data(), flat.size() * sizeof(int));
      }))
    return -1;
  return need;
}

int ffb_assign_workers(int n_workers, int n_parts, int* out) {
  return guard([&] {
    const auto a = assign_workers(n_workers, n_parts);
    std::memcpy(out, a.data(), a.size() * sizeof(int));
  });
}

int ffb_assemble_apply(ffb_ctx* c, int W, int H, const double* t10, const double* alpha,
                       const double* lambda, int nc, const double* x3, double* y3, double* b3) {
  return guard([&] {
    check_ctx(c);
    if (nc != 2 && nc != 3) fail("assembly.assemble: components must be 2 or 3");
    check_dims(W, H, "mesh.build_pixel_mesh");
    set_problem(c, W, H);
    const size_t N = c->N;
    upload(c->t10.ensure(10 * N), t10, 10 * N, c->st);
    c->terms_version++;
    ensure_reg(c);
    upload(c->alpha.p, alpha, c->ntri, c->st);
    upload(c->lambda.p, lambda, c->ntri, c->st);
    c->alpha_version++;
    c->coef.ensure(kCoefPlanes * N);
    build_coef(c->t10.p, c->alpha.p, c->lambda.p, W, H, nc, c->coef.p, nullptr, c->st);
    c->coef_key_a = c->alpha_version, c->coef_key_t = c->terms_version, c->coef_nc = nc;
    double* w = c->work.ensure(3 * N);
    double* xi = c->x.ensure(3 * N);
    double* yi = c->q.ensure(3 * N);
    upload(w, x3, 3 * N, c->st);
    planes_to_inter(w, xi, static_cast<long long>(N), nc, c->st);
    apply_op(c->coef.p, W, H, nc, xi, yi, c->st);
    inter_to_planes(yi, w, static_cast<long long>(N), nc, c->st);
    download(y3, w, 3 * N, c->st);
    sync(c);
    build_rhs(c->t10.p, W, H, nc, yi, c->st);
    inter_to_planes(yi, w, static_cast<long long>(N), nc, c->st);
    download(b3, w, 3 * N, c->st);
    sync(c);
  });
}

int ffb_error_indicator(ffb_ctx* c, int W, int H, const double* t10, const double* alpha,
                        const double* lambda, const double* u3, int nc, double* eta,
                        double* eta_max) {
  return guard([&] {
    check_ctx(c);
    check_dims(W, H, "adapt.error_indicator");
    set_problem(c, W, H);
    const size_t N = c->N;
    upload(c->t10.ensure(10 * N), t10, 10 * N, c->st);
    c->terms_version++;
    ensure_reg(c);
    upload(c->alpha.p, alpha, c->ntri, c->st);
    upload(c->lambda.p, lambda, c->ntri, c->st);
    c->alpha_version++;
    double* u = c->work.ensure(3 * N);
    upload(u, u3, 3 * N, c->st);
    double* e = c->eta.ensure(c->ntri);
    double* em = c->eta_hist.ensure(FFB_MAX_SOLVES);
    unsigned* counter = c->counter.ensure(1);
    FFB_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), c->st));
    error_indicator(c->t10.p, c->alpha.p, c->lambda.p, u, W, H, nc, e, em,
                    c->red.ensure(4 * kRedBlocks), counter, c->st);
    if (eta) download(eta, e, c->ntri, c->st);
    download(eta_max, em, 1, c->st);
    sync(c);
  });
}

int ffb_update_alpha(ffb_ctx* c, int ntri, const double* alpha, const double* eta,
                     double eta_max, double kappa, double eta_thr, double alpha_th,
                     double* alpha_out) {
  return guard([&] {
    check_ctx(c);
    double* d = c->tmp.ensure(3 * static_cast<size_t>(ntri) + 1);
    upload(d, alpha, ntri, c->st);
    upload(d + ntri, eta, ntri, c->st);
    upload(d + 3 * static_cast<size_t>(ntri), &eta_max, 1, c->st);
    update_alpha(d + 2 * static_cast<size_t>(ntri), d, d + ntri, d + 3 * static_cast<size_t>(ntri),
                 ntri, kappa, eta_thr, alpha_th, c->st);
    download(alpha_out, d + 2 * static_cast<size_t>(ntri), ntri, c->st);
    sync(c);
  });
}

int ffb_set_terms(ffb_ctx* c, int W, int H, const double* t10) {
  return guard([&] {
    check_ctx(c);
    check_dims(W, H, "mesh.build_pixel_mesh");
    set_problem(c, W, H);
    upload(c->t10.ensure(10 * c->N), t10, 10 * c->N, c->st);
    c->terms_version++;
    sync(c);
  });
}

int ffb_set_frames(ffb_ctx* c, int W, int H, const double* f0, const double* f1, double sigma,
                   double rho) {
  return guard([&] {
    check_ctx(c);
    check_dims(W, H, "imaging.compute_derivatives");
    set_problem(c, W, H);
    double* fr = c->frames.ensure(2 * c->N);
    upload(fr, f0, c->N, c->st);
    upload(fr + c->N, f1, c->N, c->st);
    frames_to_terms_dev(c, fr, fr + c->N, sigma, rho);
    sync(c);
  });
}

int ffb_set_reg(ffb_ctx* c, const double* alpha, const double* lambda) {
  return guard([&] {
    check_ctx(c);
    if (!c->W) fail("assembly.assemble: no problem set");
    ensure_reg(c);
    upload(c->alpha.p, alpha, c->ntri, c->st);
    upload(c->lambda.p, lambda, c->ntri, c->st);
    c->alpha_version++;
    c->fact_valid = 0;  // lambda may have changed too: no incremental refactorisation
    sync(c);
  });
}

int ffb_get_reg(ffb_ctx* c, double* alpha, double* lambda) {
  return guard([&] {
    check_ctx(c);
    if (!c->alpha.p) fail("assembly.assemble: no regularization set");
    if (alpha) download(alpha, c->alpha.p, c->ntri, c->st);
    if (lambda) download(lambda, c->lambda.p, c->ntri, c->st);
    sync(c);
  });
}

int ffb_set_partition(ffb_ctx* c, int px, int py, int overlap) {
  return guard([&] {
    check_ctx(c);
    if (!c->W) fail("schwarz.schwarz_solve: no problem set");
    ensure_partition(c, px, py, overlap, 3);
  });
}

int ffb_pcg_solve(ffb_ctx* c, int nc, double tol, int max_iters, int warm, double* u3,
                  int* iters, double* residual) {
  return guard([&] {
    check_ctx(c);
    if (nc != 2 && nc != 3) fail("assembly.assemble: components must be 2 or 3");
    if (!c->alpha.p) fail("assembly.assemble: no regularization set");
    if (!c->have_part) fail("schwarz.schwarz_solve: no partition set");
    if (warm) {
      double* w = c->work.ensure(3 * c->N);
      upload(w, u3, 3 * c->N, c->st);
      planes_to_inter(w, c->x.ensure(3 * c->N), static_cast<long long>(c->N), nc, c->st);
    }
    const PcgResult r = pcg(c, nc, tol, max_iters, warm != 0);
    double* w = c->work.ensure(3 * c->N);
    inter_to_planes(c->x.p, w, static_cast<long long>(c->N), nc, c->st);
    download(u3, w, 3 * c->N, c->st);
    sync(c);
    if (iters) *iters = r.iters;
    if (residual) *residual = r.res;
  });
}

// ---- multi-GPU: communicators (comm.hpp) --------------------------------------------
int ffb_comm_nccl_id(unsigned char* id128) {
  return guard([&] {
    if (!id128) fail("schwarz.comm: null id buffer");
    nccl_unique_id(id128);
  });
}

int ffb_comm_init_nccl(ffb_ctx* c, int rank, int world, const unsigned char* id128) {
  return guard([&] {
    check_ctx(c);
    if (world < 1 || rank < 0 || rank >= world) fail("schwarz.comm: invalid rank/world");
    c->comm = world == 1 ? nullptr : make_nccl_comm(rank, world, id128);
    c->have_part = false;  // the row band changes with the communicator
    c->factor_key_a = c->factor_key_t = -1;
    c->fact_valid = 0;
  });
}

int ffb_comm_local_hub(int world, ffb_local_hub** hub) {
  return guard([&] {
    if (!hub) fail("schwarz.comm: null hub pointer");
    *hub = reinterpret_cast<ffb_local_hub*>(local_hub_create(world));
  });
}

int ffb_comm_local_hub_destroy(ffb_local_hub* hub) {
  return guard([&] { local_hub_destroy(reinterpret_cast<LocalHub*>(hub)); });
}

int ffb_comm_init_local(ffb_ctx* c, ffb_local_hub* hub, int rank) {
  return guard([&] {
    check_ctx(c);
    c->comm = make_local_comm(reinterpret_cast<LocalHub*>(hub), rank);
    c->have_part = false;
    c->factor_key_a = c->factor_key_t = -1;
    c->fact_valid = 0;
  });
}

int ffb_comm_info(ffb_ctx* c, int* rank, int* world, int* rows) {
  return guard([&] {
    check_ctx(c);
    if (rank) *rank = c->comm ? c->comm->rank : 0;
    if (world) *world = c->comm ? c->comm->world : 1;
    if (rows) {
      if (!c->have_part) fail("schwarz.comm: no partition set");
      const RankRows& g = c->rows;
      const int v[12] = {g.y0, g.y1, g.j0, g.j1, g.fa0, g.fa1, g.fb0, g.fb1, g.ra0, g.ra1, g.rb0, g.rb1};
      std::memcpy(rows, v, sizeof v);
    }
  });
}

int ffb_comm_rows(int W, int H, int px, int py, int ov, int rank, int world, int* rows) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) fail("schwarz.comm: invalid rank/world");
    const RankRows g = rank_rows(build_partition(W, H, px, py, ov), rank, world);
    const int v[12] = {g.y0, g.y1, g.j0, g.j1, g.fa0, g.fa1, g.fb0, g.fb1, g.ra0, g.ra1, g.rb0, g.rb1};
    std::memcpy(rows, v, sizeof v);
  });
}

// ---- the reference's literal Schwarz loop (schwarz.cpp:162-319) ----------------------
int ffb_schwarz_run(ffb_ctx* c, const ffb_schwarz_options* o, double* u3, ffb_schwarz_stats* stats) {
  return guard([&] {
    check_ctx(c);
    if (!o) fail("schwarz.schwarz_solve: null options");
    const int nc = o->components, n_iters = o->n_iters;
    if (nc != 2 && nc != 3) fail("assembly.assemble: components must be 2 or 3");
    if (!c->alpha.p) fail("assembly.assemble: no regularization set");
    if (!c->have_part) fail("schwarz.schwarz_solve: no partition set");
    if (c->comm && c->comm->world > 1)
      fail("schwarz.schwarz_solve: the literal loop runs on one GPU (no communicator)");
    if (n_iters < 0) fail("schwarz.schwarz_solve: n_iters must be >= 0");
    if (o->method != FFB_SOLVE_CHOLESKY && o->method != FFB_SOLVE_CG)
      fail("schwarz.schwarz_solve: unknown solver method");
    const bool use_cg = o->method == FFB_SOLVE_CG;
    if (c->part_nc != nc) ensure_partition(c, c->part_px, c->part_py, c->part_ov, nc);
    ensure_coef(c, nc);
    ensure_rhs(c, nc);
    const size_t N = c->N;
    const int np = static_cast<int>(c->subs.size());
    const long long vec_len = c->ylocal.n;
    int max_n = 0;
    for (const SubInfo& sd : c->subs) max_n = std::max(max_n, sd.n);
    double* rl = c->rlocal.ensure(vec_len);
    double* xl = c->xlocal.ensure(vec_len);
    double* G = c->G0.ensure(3 * N);
    double* Gn = c->G1.ensure(3 * N);
    double* inc = c->incs.ensure(std::max(n_iters, 1));
    double* em = c->eta_hist.ensure(std::max(n_iters, FFB_MAX_SOLVES));
    double* eta = c->eta.ensure(c->ntri);
    double* blockmax = c->red.ensure(4 * kRedBlocks);
    unsigned* counter = c->counter.ensure(1);
    // CG mode: persistent warm start x_prev (schwarz.cpp:250-253), reference-order vectors
    const int maxch = ras_cg_chunks(max_n);
    double *bx = nullptr, *bb = nullptr, *br = nullptr, *bz = nullptr, *bp = nullptr,
           *bAp = nullptr, *bpart = nullptr;
    CgCtl* bctl = nullptr;
    std::vector<CgCtl> hctl;
    if (use_cg) {
      bx = c->b_x.ensure(vec_len);
      bb = c->b_b.ensure(vec_len);
      br = c->b_r.ensure(vec_len);
      bz = c->b_z.ensure(vec_len);
      bp = c->b_p.ensure(vec_len);
      bAp = c->b_Ap.ensure(vec_len);
      bpart = c->b_part.ensure(static_cast<size_t>(maxch) * np);
      bctl = c->b_ctl.ensure(np);
      hctl.resize(np);
      FFB_CUDA(cudaMemsetAsync(bx, 0, vec_len * sizeof(double), c->st));  // no x_prev yet
    }
    FFB_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), c->st));
    FFB_CUDA(cudaMemsetAsync(G, 0, 3 * N * sizeof(double), c->st));  // G = 0 (schwarz.cpp:190)
    // owner (core) of every column / row (schwarz.cpp:87-91)
    {
      const Partition& P = c->decomp;
      std::vector<int> oc(c->W), orow(c->H);
      for (int x = 0; x < c->W; ++x)
        oc[x] = int(std::upper_bound(P.xs.begin(), P.xs.end(), x) - P.xs.begin()) - 1;
      for (int y = 0; y < c->H; ++y)
        orow[y] = int(std::upper_bound(P.ys.begin(), P.ys.end(), y) - P.ys.begin()) - 1;
      FFB_CUDA(cudaMemcpyAsync(c->own_col.ensure(c->W), oc.data(), c->W * sizeof(int),
                               cudaMemcpyHostToDevice, c->st));
      FFB_CUDA(cudaMemcpyAsync(c->own_row.ensure(c->H), orow.data(), c->H * sizeof(int),
                               cudaMemcpyHostToDevice, c->st));
      sync(c);
    }
    const int n_adapt = o->adapt ? std::max(0, o->n_adapt) : 0;
    int n_upd = 0;
    for (int iter = 0; iter < n_iters; ++iter) {
      const auto t0 = std::chrono::steady_clock::now();
      ensure_coef(c, nc);
      ras_rhs(c->d_subs.p, np, c->coef.p, c->b.p, G, N, c->W, c->H, nc, rl, c->st);
      const double* dl = nullptr;
      if (use_cg) {  // cg_solve per subdomain, warm-started from x_prev (schwarz.cpp:248-252)
        ras_perm(c->d_subs.p, np, nc, rl, bb, 1, c->st);
        ras_cg_begin(c->d_subs.p, np, maxch, c->coef.p, N, c->W, nc, o->cg_tolerance,
                     o->cg_max_iters, bb, bx, br, bz, bp, bAp, bpart, bctl, c->st);
        for (;;) {
          FFB_CUDA(cudaMemcpyAsync(hctl.data(), bctl, np * sizeof(CgCtl), cudaMemcpyDeviceToHost,
                                   c->st));
          sync(c);
          bool all = true;
          for (const CgCtl& h : hctl) all = all && h.done;
          if (all) break;
          ras_cg_iterations(c->d_subs.p, np, maxch, c->coef.p, N, c->W, nc, 16, bx, br, bz, bp,
                            bAp, bpart, bctl, c->st);
        }
        for (const CgCtl& h : hctl) {
          if (h.err == 2)
            fail("linsolve.cg: indefinite matrix detected at iteration " + std::to_string(h.it));
          if (!h.zero && h.res > o->cg_tolerance)
            fail("linsolve.cg: no convergence after " + std::to_string(h.it) +
                 " iterations, relative residual " + std::to_string(h.res));
        }
        ras_cg_zero(c->d_subs.p, np, bx, bctl, c->st);
        ras_perm(c->d_subs.p, np, nc, bx, xl, 0, c->st);
      } else {
        ensure_factor(c, nc);  // refactors iff alpha changed (schwarz.cpp:238-241)
        line_solve(c->d_subs.p, np, c->plan, solve_factor(c), c->coef.p, N, nullptr, c->ylocal.p,
                   c->zlocal.p, c->W, nc, nullptr, c->st, rl, c->n_cta ? c->qsync.p : nullptr,
                   c->n_cta);
        // x += A^-1 (rhs - A x): one step of iterative refinement (schwarz.cpp:242-247)
        vec_copy(xl, c->zlocal.p, vec_len, c->st);
        ras_residual(c->d_subs.p, np, c->coef.p, N, c->W, nc, rl, xl, rl, c->st);
        line_solve(c->d_subs.p, np, c->plan, solve_factor(c), c->coef.p, N, nullptr, c->ylocal.p,
                   c->zlocal.p, c->W, nc, nullptr, c->st, rl, c->n_cta ? c->qsync.p : nullptr,
                   c->n_cta);
        dl = c->zlocal.p;
      }
      ras_compose(c->own_col.p, c->own_row.p, c->d_subs.p, c->part_px, xl, dl, G, Gn, c->W, c->H,
                  nc, blockmax, inc + iter, counter, c->st);
      std::swap(G, Gn);
      if (iter < n_adapt) {  // schwarz.cpp:303-311
        double* u = c->work.ensure(3 * N);
        inter_to_planes(G, u, static_cast<long long>(N), nc, c->st);
        error_indicator(c->t10.p, c->alpha.p, c->lambda.p, u, c->W, c->H, nc, eta, em + n_upd,
                        blockmax, counter, c->st);
        update_alpha(c->alpha.p, c->alpha.p, eta, em + n_upd, c->ntri, o->kappa,
                     o->eta_threshold, o->alpha_th, c->st);
        c->alpha_version++;
        if (stats && stats->alpha_history && o->record_alpha_history)
          download(stats->alpha_history + static_cast<size_t>(n_upd) * c->ntri, c->alpha.p,
                   c->ntri, c->st);
        ++n_upd;
      }
      if (stats && stats->seconds) {  // wall time per iteration (schwarz.cpp:312-316)
        sync(c);
        stats->seconds[iter] =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      }
    }
    double* u = c->work.ensure(3 * N);
    inter_to_planes(G, u, static_cast<long long>(N), nc, c->st);
    if (u3) download(u3, u, 3 * N, c->st);
    if (stats && stats->increments && n_iters > 0) download(stats->increments, inc, n_iters, c->st);
    if (stats && stats->eta_max && n_upd > 0) download(stats->eta_max, em, n_upd, c->st);
    if (stats) stats->n_updates = n_upd;
    sync(c);
  });
}

int ffb_schwarz_solve(ffb_ctx* c, int n_iters, int nc, int adapt, int n_adapt, double kappa,
                      double eta_thr, double alpha_th, int refine, double* u3,
                      double* increments, double* eta_max) {
  if (!refine) {
    g_err = "schwarz.schwarz_solve: the Cholesky subdomain path always refines (schwarz.cpp:242-247)";
    return 1;
  }
  ffb_schwarz_options o{};
  o.n_iters = n_iters, o.workers = 1, o.components = nc, o.adapt = adapt, o.n_adapt = n_adapt;
  o.kappa = kappa, o.eta_threshold = eta_thr, o.alpha_th = alpha_th;
  o.method = FFB_SOLVE_CHOLESKY, o.cg_tolerance = 1e-10;
  ffb_schwarz_stats st{};
  st.increments = increments, st.eta_max = eta_max;
  return ffb_schwarz_run(c, &o, u3, &st);
}

// energy (assembly.cpp:201-238) of a host state, as a device reduction
int ffb_energy(ffb_ctx* c, int W, int H, const double* t10, const double* alpha,
               const double* lambda, const double* u3, int nc, double* e) {
  return guard([&] {
    check_ctx(c);
    if (nc != 2 && nc != 3) fail("assembly.energy: components must be 2 or 3");
    check_dims(W, H, "mesh.build_pixel_mesh");
    if (!e) fail("assembly.energy: null output");
    set_problem(c, W, H);
    const size_t N = c->N;
    upload(c->t10.ensure(10 * N), t10, 10 * N, c->st);
    c->terms_version++;
    ensure_reg(c);
    upload(c->alpha.p, alpha, c->ntri, c->st);
    upload(c->lambda.p, lambda, c->ntri, c->st);
    c->alpha_version++;
    c->fact_valid = 0;
    double* u = c->work.ensure(3 * N);
    upload(u, u3, 3 * N, c->st);
    double* out = c->eta_hist.ensure(FFB_MAX_SOLVES);
    unsigned* counter = c->counter.ensure(1);
    FFB_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), c->st));
    energy(c->t10.p, c->alpha.p, c->lambda.p, u, W, H, nc, out, c->red.ensure(4 * kRedBlocks),
           counter, c->st);
    download(e, out, 1, c->st);
    sync(c);
  });
}

// energy of the resident solution (the last solve's x) with the resident terms and reg
int ffb_energy_resident(ffb_ctx* c, int nc, double* e) {
  return guard([&] {
    check_ctx(c);
    if (!c->x.p || !c->alpha.p || !c->t10.p) fail("assembly.energy: no solution on the device");
    if (!e) fail("assembly.energy: null output");
    double* u = c->work.ensure(3 * c->N);
    inter_to_planes(c->x.p, u, static_cast<long long>(c->N), nc, c->st);
    double* out = c->eta_hist.ensure(FFB_MAX_SOLVES);
    unsigned* counter = c->counter.ensure(1);
    FFB_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), c->st));
    energy(c->t10.p, c->alpha.p, c->lambda.p, u, c->W, c->H, nc, out,
           c->red.ensure(4 * kRedBlocks), counter, c->st);
    download(e, out, 1, c->st);
    sync(c);
  });
}

int ffb_adapt(ffb_ctx* c, int nc, double kappa, double eta_thr, double alpha_th,
              double* eta_max) {
  return guard([&] {
    check_ctx(c);
    if (!c->x.p) fail("adapt.error_indicator: no solution on the device");
    double* u3 = c->work.ensure(3 * c->N);
    inter_to_planes(c->x.p, u3, static_cast<long long>(c->N), nc, c->st);
    double* em = c->eta_hist.ensure(FFB_MAX_SOLVES);
    unsigned* counter = c->counter.ensure(1);
    FFB_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), c->st));
    double* eta = c->eta.ensure(c->ntri);
    error_indicator(c->t10.p, c->alpha.p, c->lambda.p, u3, c->W, c->H, nc, eta, em,
                    c->red.ensure(4 * kRedBlocks), counter, c->st);
    update_alpha(c->alpha.p, c->alpha.p, eta, em, c->ntri, kappa, eta_thr, alpha_th, c->st);
    c->alpha_version++;
    if (eta_max) download(eta_max, em, 1, c->st);
    sync(c);
  });
}

int ffb_run_on_frames(ffb_ctx* c, int W, int H, const double* f0, const double* f1,
                      const ffb_run_config* cfg, double* u3, double* alpha,
                      ffb_run_stats* stats) {
  return guard([&] {
    check_ctx(c);
    check_dims(W, H, "cli.run");
    const size_t N = static_cast<size_t>(W) * H;
    double* fr = c->frames.ensure(5 * N);
    upload(fr, f0, N, c->st);
    upload(fr + N, f1, N, c->st);
    run_dev(c, W, H, fr, fr + N, cfg, fr + 2 * N, stats);
    download(u3, fr + 2 * N, 3 * N, c->st);
    if (alpha) download(alpha, c->alpha.p, c->ntri, c->st);
    sync(c);
  });
}

int ffb_run_on_frames_dev(ffb_ctx* c, int W, int H, const double* d_f0, const double* d_f1,
                          const ffb_run_config* cfg, double* d_u3, ffb_run_stats* stats) {
  return guard([&] {
    check_ctx(c);
    run_dev(c, W, H, d_f0, d_f1, cfg, d_u3, stats);
  });
}

/* ---- linsolve boundary on an explicit CSR SparseSystem (linsolve.hpp:26-62) ---------- */
}  // extern "C"

namespace {

CsrDev upload_csr(ffb_ctx* c, int n, const int* row_ptr, const int* cols, const double* vals) {
  if (n < 0) fail("linsolve: negative system size");
  if (n > 0 && (!row_ptr || !cols || !vals)) fail("linsolve: null CSR array");
  const long long nnz = n > 0 ? row_ptr[n] : 0;
  int* rp = c->csr_rp.ensure(n + 1);
  int* ci = c->csr_ci.ensure(nnz);
  double* v = c->csr_v.ensure(nnz);
  FFB_CUDA(cudaMemcpyAsync(rp, row_ptr, (n + 1) * sizeof(int), cudaMemcpyHostToDevice, c->st));
  if (nnz) {
    FFB_CUDA(cudaMemcpyAsync(ci, cols, nnz * sizeof(int), cudaMemcpyHostToDevice, c->st));
    upload(v, vals, nnz, c->st);
  }
  return CsrDev{n, rp, ci, v};
}

// cg_solve (linsolve.cpp:298-361) on the device, bit for bit; b, x device vectors of A.n
void run_cg(ffb_ctx* c, const CsrDev& A, const double* b, const double* warm_h, double tol,
            int max_iters, double* x, int* iters, double* res) {
  const int n = A.n;
  double* diag = c->csr_diag.ensure(n);
  int* bad = c->csr_bad.ensure(1);
  FFB_CUDA(cudaMemsetAsync(bad, 0x7f, sizeof(int), c->st));
  csr_diag(A, diag, bad, c->st);
  int bad_h = 0;
  FFB_CUDA(cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  if (bad_h != 0x7f7f7f7f) fail("linsolve.cg: non-positive diagonal at row " + std::to_string(bad_h));
  CgCtl h{};
  h.tol = tol;
  h.max_iters = max_iters > 0 ? max_iters : 10LL * n;
  CgCtl* ctl = c->cgctl.ensure(1);
  FFB_CUDA(cudaMemcpyAsync(ctl, &h, sizeof(CgCtl), cudaMemcpyHostToDevice, c->st));
  double* part = c->csr_part.ensure(dot_chunks(n));
  double *r = c->csr_r.ensure(n), *z = c->csr_z.ensure(n), *p = c->csr_p.ensure(n),
         *Ap = c->csr_Ap.ensure(n);
  det_dot(b, b, n, part, ctl, c->st);
  cg_scalar(part, n, cg_stage_normb(), ctl, c->st);
  if (warm_h)
    upload(x, warm_h, n, c->st);
  else
    FFB_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), c->st));
  csr_spmv(A, x, Ap, ctl, c->st);
  cg_init(n, b, Ap, diag, r, z, p, ctl, c->st);
  det_dot(r, z, n, part, ctl, c->st);
  cg_scalar(part, n, cg_stage_init_rz(), ctl, c->st);
  det_dot(r, r, n, part, ctl, c->st);
  cg_scalar(part, n, cg_stage_init_res(), ctl, c->st);
  for (;;) {
    FFB_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(CgCtl), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    if (h.done) break;
    for (int k = 0; k < 16; ++k) cg_iteration(A, x, r, z, p, Ap, diag, part, ctl, c->st);
  }
  if (h.zero) {
    FFB_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), c->st));
    h.it = 0, h.res = 0.0;
  }
  if (iters) *iters = static_cast<int>(h.it);
  if (res) *res = h.res;
  if (h.err == 2)
    fail("linsolve.cg: indefinite matrix detected at iteration " + std::to_string(h.it));
  if (!h.zero && h.res > tol)
    fail("linsolve.cg: no convergence after " + std::to_string(h.it) +
         " iterations, relative residual " + std::to_string(h.res));
}

}  // namespace

extern "C" {

// assemble (assembly.hpp:59-61, assembly.cpp:32-166) as an explicit CSR SparseSystem: the
// pattern (free vertices, row lengths) is host integer work as in the reference, the values
// and the eliminated right-hand side come from the device coefficient planes (bitwise).
// Call with row_ptr == NULL for n and nnz, then with arrays of n+1 / nnz / nnz / n and
// vert_to_free[W*H] / free_to_vert[n/nc] (either may be NULL).
int ffb_assemble_system(ffb_ctx* c, int W, int H, const double* t10, const double* alpha,
                        const double* lambda, int nc, int n_dir, const int* dir_vertices,
                        const double* dir_values, int* n_out, long long* nnz_out, int* row_ptr,
                        int* cols, double* vals, double* rhs, int* vert_to_free,
                        int* free_to_vert) {
  return guard([&] {
    if (nc != 2 && nc != 3) fail("assembly.assemble: components must be 2 or 3");
    check_dims(W, H, "mesh.build_pixel_mesh");
    const int nv = W * H;
    std::vector<int> v2f(nv, 0);
    std::vector<double> g;
    if (n_dir > 0) {
      g.assign(static_cast<size_t>(nv) * nc, 0.0);
      for (int k = 0; k < n_dir; ++k) {
        const int v = dir_vertices[k];
        if (v < 0 || v >= nv) fail("assembly.assemble: Dirichlet vertex out of range");
        v2f[v] = -1;
        for (int cc = 0; cc < nc; ++cc) g[static_cast<size_t>(v) * nc + cc] = dir_values[k * nc + cc];
      }
    }
    std::vector<int> f2v;
    for (int v = 0; v < nv; ++v) {
      if (v2f[v] == 0) {
        v2f[v] = static_cast<int>(f2v.size());
        f2v.push_back(v);
      } else {
        v2f[v] = -1;
      }
    }
    const int nf = static_cast<int>(f2v.size());
    std::vector<int> rp(static_cast<size_t>(nf) * nc + 1, 0);
    for (int f = 0; f < nf; ++f) {
      const int v = f2v[f], x = v % W, y = v / W;
      const int nb[6][2] = {{x - 1, y - 1}, {x, y - 1}, {x - 1, y}, {x + 1, y}, {x, y + 1}, {x + 1, y + 1}};
      int cnt = 0;
      for (const auto& q : nb)
        if (q[0] >= 0 && q[0] < W && q[1] >= 0 && q[1] < H && v2f[q[1] * W + q[0]] >= 0) ++cnt;
      for (int cc = 0; cc < nc; ++cc) rp[f * nc + cc + 1] = cnt + nc;
    }
    for (size_t r = 0; r + 1 < rp.size(); ++r) rp[r + 1] += rp[r];
    *n_out = nf * nc;
    *nnz_out = rp.back();
    if (!row_ptr) return;
    check_ctx(c);
    set_problem(c, W, H);
    const size_t N = c->N;
    upload(c->t10.ensure(10 * N), t10, 10 * N, c->st);
    c->terms_version++;
    ensure_reg(c);
    upload(c->alpha.p, alpha, c->ntri, c->st);
    upload(c->lambda.p, lambda, c->ntri, c->st);
    c->alpha_version++;
    c->fact_valid = 0;
    c->coef.ensure(kCoefPlanes * N);
    build_coef(c->t10.p, c->alpha.p, c->lambda.p, W, H, nc, c->coef.p, nullptr, c->st);
    c->coef_key_a = c->alpha_version, c->coef_key_t = c->terms_version, c->coef_nc = nc;
    int* d_f2v = c->a_f2v.ensure(std::max(nf, 1));
    int* d_v2f = c->a_v2f.ensure(nv);
    int* d_rp = c->a_rp.ensure(rp.size());
    double* d_g = c->a_g.ensure(std::max<size_t>(g.size(), 1));
    if (nf) FFB_CUDA(cudaMemcpyAsync(d_f2v, f2v.data(), nf * sizeof(int), cudaMemcpyHostToDevice, c->st));
    FFB_CUDA(cudaMemcpyAsync(d_v2f, v2f.data(), nv * sizeof(int), cudaMemcpyHostToDevice, c->st));
    FFB_CUDA(cudaMemcpyAsync(d_rp, rp.data(), rp.size() * sizeof(int), cudaMemcpyHostToDevice, c->st));
    if (!g.empty()) upload(d_g, g.data(), g.size(), c->st);
    const long long nnz = rp.back();
    int* d_cols = c->csr_ci.ensure(std::max<long long>(nnz, 1));
    double* d_vals = c->csr_v.ensure(std::max<long long>(nnz, 1));
    double* d_rhs = c->csr_b.ensure(std::max(nf * nc, 1));
    csr_fill(c->coef.p, c->t10.p, W, H, nc, nf, d_f2v, d_v2f, d_rp, g.empty() ? nullptr : d_g,
             d_cols, d_vals, d_rhs, c->st);
    std::copy(rp.begin(), rp.end(), row_ptr);
    if (nnz) {
      FFB_CUDA(cudaMemcpyAsync(cols, d_cols, nnz * sizeof(int), cudaMemcpyDeviceToHost, c->st));
      download(vals, d_vals, nnz, c->st);
    }
    if (nf) download(rhs, d_rhs, static_cast<size_t>(nf) * nc, c->st);
    sync(c);
    if (vert_to_free) std::copy(v2f.begin(), v2f.end(), vert_to_free);
    if (free_to_vert) std::copy(f2v.begin(), f2v.end(), free_to_vert);
  });
}

int ffb_csr_spmv(ffb_ctx* c, int n, const int* row_ptr, const int* cols, const double* vals,
                 const double* x, double* y) {
  return guard([&] {
    check_ctx(c);
    const CsrDev A = upload_csr(c, n, row_ptr, cols, vals);
    if (n == 0) return;
    double* xd = c->csr_x.ensure(n);
    double* yd = c->csr_r.ensure(n);
    upload(xd, x, n, c->st);
    csr_spmv(A, xd, yd, nullptr, c->st);
    download(y, yd, n, c->st);
    sync(c);
  });
}

int ffb_rcm_order(int n, int components, const int* row_ptr, const int* cols, int* perm) {
  return guard([&] {
    if (n < 0 || !row_ptr || (n > 0 && (!cols || !perm))) fail("linsolve.rcm_order: bad arguments");
    const std::vector<int> p = rcm_order(n, components, row_ptr, cols);
    std::copy(p.begin(), p.end(), perm);
  });
}

int ffb_csr_cg_solve(ffb_ctx* c, int n, const int* row_ptr, const int* cols, const double* vals,
                     const double* rhs, double tol, int max_iters, const double* warm, double* x,
                     int* iters, double* res) {
  return guard([&] {
    check_ctx(c);
    const CsrDev A = upload_csr(c, n, row_ptr, cols, vals);
    if (n == 0) {
      if (iters) *iters = 0;
      if (res) *res = 0.0;
      return;
    }
    double* b = c->csr_b.ensure(n);
    double* xd = c->csr_x.ensure(n);
    upload(b, rhs, n, c->st);
    run_cg(c, A, b, warm, tol, max_iters, xd, iters, res);
    download(x, xd, n, c->st);
    sync(c);
  });
}

int ffb_csr_solve(ffb_ctx* c, int n, int components, const int* row_ptr, const int* cols,
                  const double* vals, const double* rhs, int method, double tol, int max_iters,
                  const double* warm, double* x, int* iters, double* res) {
  return guard([&] {
    check_ctx(c);
    if (method != FFB_SOLVE_CHOLESKY && method != FFB_SOLVE_CG) fail("linsolve.solve: unknown method");
    bool all_zero = true;
    for (int i = 0; i < n && all_zero; ++i) all_zero = rhs[i] == 0.0;
    if (all_zero) {  // linsolve.cpp:365-372
      std::fill(x, x + n, 0.0);
      if (iters) *iters = 0;
      if (res) *res = 0.0;
      return;
    }
    const CsrDev A = upload_csr(c, n, row_ptr, cols, vals);
    double* b = c->csr_b.ensure(n);
    double* xd = c->csr_x.ensure(n);
    upload(b, rhs, n, c->st);
    if (method == FFB_SOLVE_CG) {
      run_cg(c, A, b, warm, tol, max_iters, xd, iters, res);
      download(x, xd, n, c->st);
      sync(c);
      return;
    }
    // direct: RCM (bit-exact with the reference's analyse) -> band Cholesky -> solve,
    // one refinement step, residual report (linsolve.cpp:377-397)
    const std::vector<int> perm = rcm_order(n, components, row_ptr, cols);
    std::vector<int> iperm(n);
    for (int k = 0; k < n; ++k) iperm[perm[k]] = k;
    int bw = 0;
    for (int r = 0; r < n; ++r)
      for (int q = row_ptr[r]; q < row_ptr[r + 1]; ++q)
        bw = std::max(bw, std::abs(iperm[r] - iperm[cols[q]]));
    int* dperm = c->csr_perm.ensure(n);
    int* diperm = c->csr_iperm.ensure(n);
    FFB_CUDA(cudaMemcpyAsync(dperm, perm.data(), n * sizeof(int), cudaMemcpyHostToDevice, c->st));
    FFB_CUDA(cudaMemcpyAsync(diperm, iperm.data(), n * sizeof(int), cudaMemcpyHostToDevice, c->st));
    const size_t nab = static_cast<size_t>(n) * (bw + 1);
    double* AB = c->csr_AB.ensure(nab);
    FFB_CUDA(cudaMemsetAsync(AB, 0, nab * sizeof(double), c->st));
    band_scatter(A, diperm, bw, AB, c->st);
    int* bad = c->csr_bad.ensure(1);
    FFB_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(int), c->st));
    band_cholesky(n, bw, AB, bad, c->st);
    int bad_h = -1;
    FFB_CUDA(cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    if (bad_h >= 0)
      fail("linsolve.cholesky: breakdown at pivot " + std::to_string(bad_h) + " (unknown " +
           std::to_string(perm[bad_h]) + "): matrix is not positive definite");
    double* t = c->csr_z.ensure(n);
    double* Ax = c->csr_Ap.ensure(n);
    double* r = c->csr_r.ensure(n);
    gather(n, dperm, b, t, c->st);
    band_solve(n, bw, AB, t, c->st);
    scatter(n, dperm, t, xd, false, c->st);
    csr_spmv(A, xd, Ax, nullptr, c->st);
    vec_sub(n, b, Ax, r, c->st);
    gather(n, dperm, r, t, c->st);
    band_solve(n, bw, AB, t, c->st);
    scatter(n, dperm, t, xd, true, c->st);
    if (res) {
      csr_spmv(A, xd, Ax, nullptr, c->st);
      double* rep = c->csr_part.ensure(1);
      residual_report(n, b, Ax, rep, c->st);
      download(res, rep, 1, c->st);
    }
    if (iters) *iters = 0;
    download(x, xd, n, c->st);
    sync(c);
  });
}

int ffb_chol_create(ffb_ctx* c, ffb_chol** out) {
  return guard([&] {
    check_ctx(c);
    if (!out) fail("linsolve.cholesky: null output");
    auto h = std::make_unique<ffb_chol>();
    h->c = c;
    *out = h.release();
  });
}

int ffb_chol_destroy(ffb_chol* h) {
  return guard([&] {
    if (!h) return;
    cudaSetDevice(h->c->device);
    delete h;
  });
}

int ffb_chol_analyze(ffb_chol* h, int n, int components, const int* row_ptr, const int* cols) {
  return guard([&] {
    if (!h) fail("linsolve.cholesky: null handle");
    check_ctx(h->c);
    const std::vector<int> perm = rcm_order(n, components, row_ptr, cols);  // rcm.cpp, bit-exact
    std::vector<int> iperm(n);
    for (int k = 0; k < n; ++k) iperm[perm[k]] = k;
    int bw = 0;
    for (int r = 0; r < n; ++r)
      for (int q = row_ptr[r]; q < row_ptr[r + 1]; ++q)
        bw = std::max(bw, std::abs(iperm[r] - iperm[cols[q]]));
    cudaStream_t st = h->c->st;
    h->n = n, h->nc = components, h->bw = bw, h->nnz = n > 0 ? row_ptr[n] : 0;
    h->factored = false;
    FFB_CUDA(cudaMemcpyAsync(h->perm.ensure(std::max(n, 1)), perm.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
    FFB_CUDA(cudaMemcpyAsync(h->iperm.ensure(std::max(n, 1)), iperm.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
    FFB_CUDA(cudaMemcpyAsync(h->rp.ensure(n + 1), row_ptr, (n + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
    if (h->nnz)
      FFB_CUDA(cudaMemcpyAsync(h->ci.ensure(h->nnz), cols, h->nnz * sizeof(int), cudaMemcpyHostToDevice, st));
    FFB_CUDA(cudaStreamSynchronize(st));
  });
}

int ffb_chol_factorize(ffb_chol* h, int n, const double* vals) {
  return guard([&] {
    if (!h || !h->perm.p) fail("linsolve.cholesky: factorize before analyze");
    check_ctx(h->c);
    if (n != h->n) fail("linsolve.cholesky: matrix size changed since analyze");
    cudaStream_t st = h->c->st;
    if (n == 0) {
      h->factored = true;
      return;
    }
    upload(h->v.ensure(std::max<long long>(h->nnz, 1)), vals, h->nnz, st);
    const size_t nab = static_cast<size_t>(n) * (h->bw + 1);
    double* AB = h->AB.ensure(nab);
    FFB_CUDA(cudaMemsetAsync(AB, 0, nab * sizeof(double), st));
    const CsrDev A{n, h->rp.p, h->ci.p, h->v.p};
    band_scatter(A, h->iperm.p, h->bw, AB, st);
    int* bad = h->bad.ensure(1);
    FFB_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(int), st));
    band_cholesky(n, h->bw, AB, bad, st);
    int bad_h = -1;
    FFB_CUDA(cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    FFB_CUDA(cudaStreamSynchronize(st));
    h->factored = false;
    if (bad_h >= 0) {
      int u = 0;
      FFB_CUDA(cudaMemcpy(&u, h->perm.p + bad_h, sizeof(int), cudaMemcpyDeviceToHost));
      fail("linsolve.cholesky: breakdown at pivot " + std::to_string(bad_h) + " (unknown " +
           std::to_string(u) + "): matrix is not positive definite");
    }
    h->factored = true;
  });
}

int ffb_chol_solve(ffb_chol* h, int n, const double* b, double* x) {
  return guard([&] {
    if (!h || !h->factored) fail("linsolve.cholesky: solve before factorize");
    check_ctx(h->c);
    if (n != h->n) fail("linsolve.cholesky: rhs size mismatch");
    if (n == 0) return;
    cudaStream_t st = h->c->st;
    double* db = h->b.ensure(n);
    double* t = h->t.ensure(n);
    upload(db, b, n, st);
    gather(n, h->perm.p, db, t, st);
    band_solve(n, h->bw, h->AB.p, t, st);
    scatter(n, h->perm.p, t, db, false, st);
    download(x, db, n, st);
    FFB_CUDA(cudaStreamSynchronize(st));
  });
}

int ffb_chol_info(ffb_chol* h, int* bandwidth, long long* factor_nonzeros) {
  return guard([&] {
    if (!h) fail("linsolve.cholesky: null handle");
    if (bandwidth) *bandwidth = h->bw;
    if (factor_nonzeros) {  // stored lower band including the diagonal
      long long s = 0;
      for (int i = 0; i < h->n; ++i) s += std::min(i, h->bw) + 1;
      *factor_nonzeros = s;
    }
  });
}

// the caller's Partition (flat format of include/flowfem_b200.h): must be the grid
// build_partition(W, H, px, py, ov) makes — the device layout follows that grid
int ffb_set_partition_flat(ffb_ctx* c, const int* flat, long len) {
  return guard([&] {
    check_ctx(c);
    if (!c->W) fail("schwarz.schwarz_solve: no problem set");
    if (!flat || len < 6) fail("schwarz.schwarz_solve: bad partition");
    if (flat[0] != c->W || flat[1] != c->H)
      fail("schwarz.schwarz_solve: partition does not match the mesh");
    const std::vector<int> want = flatten(build_partition(flat[0], flat[1], flat[2], flat[3], flat[4]));
    if (static_cast<long>(want.size()) != len || !std::equal(want.begin(), want.end(), flat))
      fail("schwarz.schwarz_solve: only partitions made by build_partition are supported");
    ensure_partition(c, flat[2], flat[3], flat[4], c->part_nc ? c->part_nc : 3);
  });
}

/* ---- I/O and evaluation (image_io.cpp, metrics.cpp) ---------------------------------- */
int ffb_load_image(const char* path, int* W, int* H, double* out) {
  return guard([&] {
    if (!path || !W || !H) fail("imaging.load_image: null argument");
    int w = 0, h = 0;
    const std::vector<double> img = load_image(path, w, h);
    if (out) {
      if (*W != w || *H != h) fail("imaging.load_image: output buffer size does not match " + std::string(path));
      std::copy(img.begin(), img.end(), out);
    }
    *W = w, *H = h;
  });
}

int ffb_save_pgm(const char* path, int W, int H, const double* img) {
  return guard([&] {
    if (!path || !img || W <= 0 || H <= 0) fail("imaging.save_pgm: bad arguments");
    save_pgm(path, W, H, img);
  });
}

int ffb_read_flo(const char* path, int* W, int* H, float* u, float* v) {
  return guard([&] {
    if (!path || !W || !H) fail("metrics.read_flo: null argument");
    int w = 0, h = 0;
    std::vector<float> uu, vv;
    read_flo(path, w, h, uu, vv);
    if (u && v) {
      if (*W != w || *H != h) fail("metrics.read_flo: output buffer size does not match " + std::string(path));
      std::copy(uu.begin(), uu.end(), u);
      std::copy(vv.begin(), vv.end(), v);
    }
    *W = w, *H = h;
  });
}

int ffb_write_flo(const char* path, int W, int H, const float* u, const float* v) {
  return guard([&] {
    if (!path || !u || !v || W <= 0 || H <= 0) fail("metrics.write_flo: bad arguments");
    write_flo(path, W, H, u, v);
  });
}

int ffb_compute_metrics(ffb_ctx* c, int W, int H, const double* u1, const double* u2,
                        const float* tu, const float* tv, double* aae_deg, double* ee,
                        long long* valid) {
  return guard([&] {
    check_ctx(c);
    check_dims(W, H, "metrics.compute_metrics");
    const size_t n = static_cast<size_t>(W) * H;
    double* d = c->work.ensure(2 * n + 2 * ((n + 1) / 2) + 3 * kRedBlocks + 4);
    double* du1 = d;
    double* du2 = d + n;
    float* dtu = reinterpret_cast<float*>(d + 2 * n);
    float* dtv = dtu + n;
    double* part = d + 2 * n + 2 * ((n + 1) / 2);
    double* out = part + 3 * kRedBlocks;
    unsigned* counter = c->counter.ensure(1);
    upload(du1, u1, n, c->st);
    upload(du2, u2, n, c->st);
    FFB_CUDA(cudaMemcpyAsync(dtu, tu, n * sizeof(float), cudaMemcpyHostToDevice, c->st));
    FFB_CUDA(cudaMemcpyAsync(dtv, tv, n * sizeof(float), cudaMemcpyHostToDevice, c->st));
    FFB_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), c->st));
    flow_metrics(du1, du2, dtu, dtv, static_cast<long long>(n), part, counter, out, c->st);
    double h[3];
    download(h, out, 3, c->st);
    sync(c);
    const long long k = static_cast<long long>(h[2]);
    *valid = k;
    *aae_deg = k > 0 ? h[0] / static_cast<double>(k) * 180.0 / M_PI : 0.0;
    *ee = k > 0 ? h[1] / static_cast<double>(k) : 0.0;
  });
}

}  // extern "C"
