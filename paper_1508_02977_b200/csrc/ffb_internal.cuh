// Internal declarations shared by the flowfem_b200 translation units.
// Reference paths are relative to /root/reference/proj.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

namespace ffb {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

[[noreturn]] void fail(const std::string& msg);
void cuda_check(cudaError_t e, const char* what, const char* file, int line);
void note_launch(long long n = 1);

#define FFB_CUDA(x) ::ffb::cuda_check((x), #x, __FILE__, __LINE__)
#define FFB_LAUNCHED() \
  do {                 \
    ::ffb::note_launch(); \
    FFB_CUDA(cudaPeekAtLastError()); \
  } while (0)

constexpr int kMaxTaps = 129;  // radius <= 64

struct Taps {
  int r;
  double w[kMaxTaps];
};
// gauss_kernel (src/imaging.cpp:19-29), computed on the host with std::exp
Taps make_taps(double sigma);

// ---- imaging kernels (imaging.cu) ---------------------------------------------------
// separable smoothing of `planes` planes (stride W*H) in -> out, tmp is scratch of the
// same size; sigma <= 0 copies.
void smooth_planes(const double* in, double* out, double* tmp, int W, int H, int planes,
                   double sigma, cudaStream_t st);
// the ten rho-smoothed data-term planes from the smoothed frames (derivatives + products +
// smoothing in one tiled kernel); prod and tmp (10 N each) are used only by the
// large-radius / unsmoothed path
void data_terms(const double* s0, const double* s1, double* t10, double* prod, double* tmp,
                int W, int H, double rho, cudaStream_t st);
void derivatives4(const double* s0, const double* s1, double* fx, double* fy, double* ft,
                  double* f, int W, int H, cudaStream_t st);
// the same from given derivative planes (build_data_terms)
void data_terms_from4(const double* fx, const double* fy, const double* ft, const double* f,
                      double* t10, double* prod, double* tmp, int W, int H, double rho,
                      cudaStream_t st);

// ---- operator (operator.cu) -----------------------------------------------------------
// Per-vertex coefficient planes (SoA, each N = W*H):
//   0..5  m11 m12 m13 m22 m23 m33  (lumped data block + stiffness diagonal)
//   6..7  eh_a eh_l : coupling (x,y)-(x+1,y) for alpha / lambda weights
//   8..9  ev_a ev_l : coupling (x,y)-(x,y+1)
constexpr int kCoefPlanes = 10;
void build_coef(const double* t10, const double* alpha, const double* lambda, int W, int H,
                int nc, double* coef, int* bad_diag, cudaStream_t st);
void build_rhs(const double* t10, int W, int H, int nc, double* b, cudaStream_t st);
void apply_op(const double* coef, int W, int H, int nc, const double* x, double* y,
              cudaStream_t st);
void planes_to_inter(const double* p3, double* x, long long N, int nc, cudaStream_t st);
// assemble()'s CSR rows of the free vertices (pattern from the host, values on the device)
void csr_fill(const double* coef, const double* t10, int W, int H, int nc, int n_free,
              const int* free_to_vert, const int* vert_to_free, const int* row_ptr,
              const double* g, int* cols, double* vals, double* rhs, cudaStream_t st);
void inter_to_planes(const double* x, double* p3, long long N, int nc, cudaStream_t st);

// ---- subdomain factor / solve (band.cu) -----------------------------------------------
// Subdomain i of the partition: the free vertices of its extended rectangle (ext minus
// the artificial Dirichlet ring, schwarz.cpp:93-112), ordered line by line along the long
// (slow) side; a line holds the S vertices of the short (fast) side x nc components.
struct SubInfo {
  int fx0, fy0, fw, fh;  // free rectangle (global pixel coordinates)
  int xfast;             // 1: x is the fast axis (line = one row), 0: y is (line = one column)
  int S;                 // fast extent (vertices per line)
  int L;                 // slow extent (number of lines)
  int kd;                // unknowns per line, nc*S
  int n;                 // L*kd scalar unknowns
  int m;                 // twisted split: chain 0 lines 0..m-1, chain 1 L-1..m+1, middle m
  long long line_sz;     // doubles per line of the packed factor (packed_line_size(kd))
  long long fac_off;     // offset (doubles) of the subdomain's factor
  long long vec_off;     // offset (doubles) into the per-subdomain vectors
  long long fac32_off;   // offset (floats) of the subdomain in the single-precision factor copy
};

struct AxisMap {  // free-rectangle membership along one axis (<= 2 parts)
  int p0, l0, p1, l1;  // part index along the axis and local coordinate; p1 = -1 if none
};

long long packed_line_size(int kd);
size_t factor_scratch_doubles(int nsub, int kd_max);
void line_factor(const SubInfo* d_subs, int nsub, int C, int nb, int kd_max, const double* coef,
                 size_t N, int W, int nc, double* fac, double* scratch, long long scratch_stride,
                 int* d_bad, cudaStream_t st, const int2* changed = nullptr,
                 double* fac_t = nullptr);
void changed_lines(const SubInfo* d_subs, int nsub, const double* alpha, const double* alpha_fact,
                   int W, int H, int2* changed, cudaStream_t st);
struct SolvePlan {
  int stages, cap, maxm, C, kd_max, tile, row_cost, ncs, stage_doubles;
  int rt;  // row-group tile ring kernel (k_line_solve_rt)
  size_t smem;
};
SolvePlan solve_plan(int kd_max, int C);
void line_solve(const SubInfo* d_subs, int nsub, const SolvePlan& pl, const double* fac,
                const double* coef, size_t N, const double* r, double* ylocal, double* zlocal,
                int W, int nc, const int* flags, cudaStream_t st,
                const double* rlocal = nullptr, int* qsync = nullptr, int n_cta = 0,
                const float* fac32 = nullptr);
// opt-in single-precision copy of the line inverses streamed by k_line_solve_rt<., float>
void factor_to_f32(const SubInfo* d_subs, int nsub, const double* fac, float* fac32,
                   const int2* changed, cudaStream_t st);

// ---- literal Schwarz iteration (ras.cu) ---------------------------------------------------
void ras_rhs(const SubInfo* d_subs, int nsub, const double* coef, const double* b,
             const double* G, size_t N, int W, int H, int nc, double* rl, cudaStream_t st);
void ras_residual(const SubInfo* d_subs, int nsub, const double* coef, size_t N, int W, int nc,
                  const double* rl, const double* xl, double* res, cudaStream_t st);
void ras_compose(const int* own_col, const int* own_row, const SubInfo* d_subs, int px,
                 const double* xl, const double* dl, const double* G, double* Gnew, int W, int H,
                 int nc, double* blockmax, double* inc_out, unsigned* counter, cudaStream_t st);
void vec_copy(double* dst, const double* src, long long n, cudaStream_t st);
// CG subdomain solves of the literal loop (SolveMethod::ConjugateGradient,
// schwarz.cpp:248-252): the reference's cg_solve per subdomain, all subdomains in lockstep,
// vectors in the reference's unknown order (ras_perm converts from / to the line layout)
struct CgCtl;
void ras_perm(const SubInfo* d_subs, int nsub, int nc, const double* src, double* dst, int to_ref,
              cudaStream_t st);
int ras_cg_chunks(int max_n);
void ras_cg_begin(const SubInfo* d_subs, int nsub, int maxch, const double* coef, size_t N, int W,
                  int nc, double tol, long long max_iters, const double* b, double* x, double* r,
                  double* z, double* p, double* Ap, double* partial, CgCtl* ctl, cudaStream_t st);
void ras_cg_iterations(const SubInfo* d_subs, int nsub, int maxch, const double* coef, size_t N,
                       int W, int nc, int k, double* x, double* r, double* z, double* p,
                       double* Ap, double* partial, CgCtl* ctl, cudaStream_t st);
void ras_cg_zero(const SubInfo* d_subs, int nsub, double* x, const CgCtl* ctl, cudaStream_t st);

// ---- PCG control block (solver.cu) ----------------------------------------------------
struct PcgCtl {
  double rz, rz_old, pAp, rr, bb, normb, res, tol;
  int k;       // combines completed
  int iters;   // CG iterations completed
  int done;    // converged (or zero rhs)
  int err;     // 1: indefinite (pAp <= 0)
  int err_it;
  int zero_rhs;
  int max_iters;
  int pad;
  unsigned counter[4];
};

// Row-band geometry of one rank (capi.cpp rank_rows): the reduction units are subdomain
// rows; rank r owns subdomain rows [j0, j1) and the pixel rows [y0, y1) of their cores.
constexpr int kCU = 296;  // CTAs per reduction unit (2 x 148 SMs), fixed for any world size
struct RankRows {
  int y0, y1;    // owned pixel rows
  int j0, j1;    // owned subdomain rows (reduction units)
  int fa0, fa1;  // rows above y0 that my subdomains' free rectangles cover
  int fb0, fb1;  // rows below y1 that my subdomains cover
  int ra0, ra1;  // my rows covered by the subdomains of the rank above
  int rb0, rb1;  // my rows covered by the subdomains of the rank below
};

// part >= 2 * (j1 - j0) * kCU doubles; ur: 2 * py doubles (unit values, zero outside the
// rank's units); finish = 1 when world == 1 (the last CTA completes the scalar update),
// else the caller all-reduces ur and runs pcg_scalar.
void pcg_init(int nc, const double* coef, const double* b, const double* x, double* r, int W,
              int H, const RankRows& g, const int* ys, int py, PcgCtl* ctl, double* part,
              double* ur, int finish, cudaStream_t st);
void pcg_zpart(int nc, const SubInfo* subs, const AxisMap* colmap, const AxisMap* rowmap, int px,
               const double* zlocal, int W, const RankRows& g, double* send_up, double* send_dn,
               const PcgCtl* ctl, cudaStream_t st);
void pcg_combine(int nc, const SubInfo* subs, const AxisMap* colmap, const AxisMap* rowmap,
                 int px, const double* zlocal, const double* r, double* z, int W,
                 const RankRows& g, const int* ys, int py, const double* recv_up,
                 const double* recv_dn, PcgCtl* ctl, double* part, double* ur, int finish,
                 cudaStream_t st, const double* yc = nullptr, const int* ccol = nullptr,
                 const int* crow = nullptr);
void pcg_spmv_p(int nc, const double* coef, const double* z, double* P0, double* P1, double* q,
                int W, int H, const RankRows& g, const int* ys, int py, PcgCtl* ctl, double* part,
                double* ur, int finish, cudaStream_t st);
void pcg_update(int nc, double* x, double* r, const double* P0, const double* P1,
                const double* q, int W, const RankRows& g, const int* ys, int py, PcgCtl* ctl,
                double* part, double* ur, int finish, cudaStream_t st);
void pcg_scalar(const double* ur, int py, int stage, PcgCtl* ctl, cudaStream_t st);
// x <- x + theta (x - xprev), xprev <- old x (the warm start of the next adaptive pass)
void vec_extrapolate(double* x, double* xprev, long long n, double theta, cudaStream_t st);
int pcg_stage_init();
int pcg_stage_pap();
int pcg_stage_rr();
int pcg_stage_rz();

// ---- two-level coarse space (coarse.cu) ---------------------------------------------------
// xs[px+1], ys[py+1]: core cuts; ccol[W] + crow[H]: coarse node of the core of pixel (x,y);
// AB: (nc px py) x (bw+1) band scratch; Ainv: n0 x n0; bad: Cholesky breakdown (-1 none)
void coarse_build(const double* coef, int W, int H, int nc, const int* xs, const int* ys, int px,
                  int py, const int* ccol, const int* crow, int bw, double* AB, double* Ainv,
                  int* bad, cudaStream_t st);
void coarse_apply(const double* r, int W, int nc, const int* xs, const int* ys, int px, int py,
                  const int* ccol, const int* crow, const double* Ainv, double* g, double* y,
                  const PcgCtl* ctl, cudaStream_t st);
void pcg_rz(const double* r, const double* z, long long nvec, PcgCtl* ctl, double* part,
            cudaStream_t st);
void pcg_spmv_p(int nc, const double* coef, const double* z, double* P0, double* P1, double* q,
                int W, int H, PcgCtl* ctl, double* part, cudaStream_t st);
void pcg_update(int nc, double* x, double* r, const double* P0, const double* P1,
                const double* q, long long nvec, int max_iters, PcgCtl* ctl, double* part,
                cudaStream_t st);

// ---- adaptation (adapt.cu) ------------------------------------------------------------
void error_indicator(const double* t10, const double* alpha, const double* lambda,
                     const double* u3, int W, int H, int nc, double* eta, double* eta_max_dev,
                     double* scratch, unsigned* counter, cudaStream_t st);
void update_alpha(double* alpha_out, const double* alpha, const double* eta,
                  const double* eta_max_dev, long long ntri, double kappa, double thr,
                  double alpha_th, cudaStream_t st);

// a25 energy (assembly.cpp:201-238): scratch >= 2 * kRedBlocks doubles, counter zeroed
void energy(const double* t10, const double* alpha, const double* lambda, const double* u3,
            int W, int H, int nc, double* out_dev, double* scratch, unsigned* counter,
            cudaStream_t st);

// reductions
constexpr int kRedBlocks = 592;  // 4 x 148 SMs
constexpr int kRedThreads = 256;

void set_solve_dbg(int v);  // development probe flags of the solve kernel (band.cu)

// ---- flow metrics (metrics.cu): out = (sum angular error, sum endpoint error, valid);
// part >= 3 * kRedBlocks doubles, counter zero-initialised (reset by the kernel)
void flow_metrics(const double* u1, const double* u2, const float* tu, const float* tv,
                  long long n, double* part, unsigned* counter, double* out, cudaStream_t st);

// ---- linsolve boundary on an explicit CSR system (linsolve.cu) ----------------------
struct CsrDev {
  int n;
  const int* rp;
  const int* ci;
  const double* v;
};
// device-side state of cg_solve (linsolve.cpp:298-361)
struct CgCtl {
  double tol, normb, rz, res, alpha, beta;
  long long it, max_iters;
  int done, zero, err;  // err 2: indefinite (pAp <= 0)
};
void csr_spmv(const CsrDev& A, const double* x, double* y, const CgCtl* ctl, cudaStream_t st);
void csr_diag(const CsrDev& A, double* diag, int* bad_row, cudaStream_t st);
int dot_chunks(long long n);
void det_dot(const double* a, const double* b, long long n, double* partial, const CgCtl* ctl,
             cudaStream_t st);
void cg_scalar(const double* partial, long long n, int stage, CgCtl* ctl, cudaStream_t st);
int cg_stage_normb();
int cg_stage_init_rz();
int cg_stage_init_res();
void cg_init(int n, const double* b, const double* Ap, const double* diag, double* r, double* z,
             double* p, const CgCtl* c, cudaStream_t st);
void cg_iteration(const CsrDev& A, double* x, double* r, double* z, double* p, double* Ap,
                  const double* diag, double* partial, CgCtl* c, cudaStream_t st);
void band_scatter(const CsrDev& A, const int* iperm, int bw, double* AB, cudaStream_t st);
void band_cholesky(int n, int bw, double* AB, int* bad, cudaStream_t st);
void band_solve(int n, int bw, const double* AB, double* x, cudaStream_t st);
void gather(int n, const int* idx, const double* src, double* dst, cudaStream_t st);
void scatter(int n, const int* idx, const double* src, double* dst, bool add, cudaStream_t st);
void vec_sub(int n, const double* b, const double* y, double* r, cudaStream_t st);
void residual_report(int n, const double* b, const double* Ax, double* out, cudaStream_t st);

}  // namespace ffb
