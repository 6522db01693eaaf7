/* flowfem_b200 — C-ABI of the B200-native adaptive-alpha Horn–Schunck + illumination
 * solver (arXiv 1508.02977 hot path). Plain C: pointers, sizes, status codes; no torch
 * or C++ types cross this boundary.
 *
 * Every entry point replaces a function of the reference library `flowfem`
 * (/root/reference/proj/include/flowfem/*.hpp); the citation is given per function.
 * Reference paths below are relative to /root/reference/proj.
 *
 * Conventions (identical to the test oracle, oracle/flowfem_port.h):
 *   - images / vertex fields: row-major H x W doubles, vertex id = y*W + x
 *     (include/flowfem/mesh.hpp:35);
 *   - "terms10": the ten DataTerms planes a11,a12,a13,a22,a23,a33,f1,f2,f3,c
 *     (include/flowfem/imaging.hpp:61-67), each W*H, back to back;
 *   - per-triangle fields: 2*(W-1)*(H-1) doubles, lower/upper triangle of cell (x,y)
 *     at 2*(y*(W-1)+x) and +1 (src/mesh.cpp:29-35);
 *   - "planes3": u1, u2, mt planes back to back, each W*H (FlowState,
 *     include/flowfem/assembly.hpp:11-22); with 2 components mt is written as 0;
 *   - flat partition format (Partition, include/flowfem/schwarz.hpp:23-48):
 *       [W, H, px, py, ov, np,
 *        per part p: core.x0 y0 x1 y1, ext.x0 y0 x1 y1, n_boundary, n_neighbors   (10 ints),
 *        then per part p: boundary[n_boundary],
 *                         per neighbor: part, band.x0 y0 x1 y1, n_gamma, gamma[n_gamma]]
 *
 * Errors: every call returns 0 on success and non-zero on failure; ffb_last_error()
 * returns the message of the calling thread's last failure, prefixed with the
 * reference module the way the reference's std::runtime_error messages are
 * ("linsolve.cg: …", "schwarz.build_partition: …", "imaging.compute_derivatives: …").
 * Host buffers are owned by the caller; device state is owned by the context.
 * One host thread per context; one context per GPU (one process per GPU).
 */
#ifndef FLOWFEM_B200_H
#define FLOWFEM_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define FFB_ABI_VERSION 2

typedef struct ffb_ctx ffb_ctx;

/* flowfem::RunConfig (include/flowfem/pipeline.hpp:15-33), solver-relevant fields. */
typedef struct ffb_run_config {
  double sigma;          /* pre-smoothing of both frames (imaging.cpp:33) */
  double rho;            /* data-term smoothing (imaging.cpp:108) */
  double alpha0;         /* uniform_reg (assembly.cpp:9-14) */
  double lambda0;
  int illumination;      /* 1 -> 3 components (u1,u2,mt), 0 -> 2 */
  int parts;             /* choose_split(W,H,parts) (schwarz.cpp:32-44) */
  int overlap;           /* build_partition overlap (schwarz.cpp:54) */
  int adapt;             /* AdaptConfig::enabled */
  int n_passes;          /* AdaptConfig::n_adapt: alpha updates; n_passes+1 solves */
  double kappa;          /* update_alpha (adapt.cpp:101-112) */
  double eta_threshold;
  double alpha_th;       /* NaN -> alpha0/100 (unset std::optional, pipeline.cpp:71) */
  double tol;            /* SolverConfig::cg_tolerance, true relative residual */
  int max_iters;         /* 0 -> 10 * unknowns (linsolve.cpp:333) */
} ffb_run_config;

#define FFB_MAX_SOLVES 64

typedef struct ffb_run_stats {
  int parts_x, parts_y;
  int n_solves;                         /* n_passes + 1 */
  int iters[FFB_MAX_SOLVES];            /* PCG iterations per solve */
  double residual[FFB_MAX_SOLVES];      /* final ||b-Ax||/||b|| per solve */
  double eta_max[FFB_MAX_SOLVES];       /* per alpha update */
  long long pcg_iterations;             /* sum of iters */
  double ms_terms, ms_factor, ms_pcg, ms_adapt, ms_total; /* CUDA-event phase times */
  double factor_doubles;                /* doubles of the packed line inverses one
                                           preconditioner application streams */
  double iter_bytes;                    /* algorithmic HBM bytes per PCG iteration */
  double ms_asm_per_iter;               /* mean duration of the subdomain-solve kernel */
  double ms_factor_full;                /* the first pass's (full) factorisation */
  double factor_flops;                  /* algorithmic flops of one full factorisation,
                                           sum_i n_i kd_i^2 (n kd^2 / 2 FMAs per subdomain) */
} ffb_run_stats;

/* ---- library ---------------------------------------------------------------------- */
const char* ffb_last_error(void);
int ffb_abi_version(void);
/* number of device kernels this library launched since load (evidence counter) */
long long ffb_kernel_launches(void);

/* ---- context (one GPU) ------------------------------------------------------------ */
int ffb_create(ffb_ctx** ctx, int device);
int ffb_destroy(ffb_ctx* ctx);
/* Launch on the caller's CUDA stream (cudaStream_t passed as void*; 0 is the legacy
 * default stream) when own == 0, or on the context's own stream when own != 0. Lets a host
 * framework order the solve with its own work and bracket it with its own events. */
int ffb_set_stream(ffb_ctx* ctx, void* stream, int own);
/* Storage of the subdomain factors the preconditioner streams (no reference counterpart: the
 * reference's SparseCholesky, linsolve.hpp:32-48, keeps doubles). 64 (default): the packed
 * line inverses in double. 32: opt-in — the solve kernel of the wide-line regime
 * (k_line_solve_rt: c3, c4) streams a single-precision COPY of them, half the bytes per
 * application; the factorisation, the products, the CG vectors and the stopping test on the
 * true residual stay in double, so the converged fields meet the same 1e-8 bar
 * (tests/test_gpu_fullsize.py). Environment FFB_FACTOR_F32=1 selects 32 at ffb_create.
 * ffb_get_factor_storage: the requested width and the one in use with the resident partition
 * (64 where another solve kernel runs). */
int ffb_set_factor_storage(ffb_ctx* ctx, int bits);
int ffb_get_factor_storage(ffb_ctx* ctx, int* bits, int* in_use);

/* ---- imaging: include/flowfem/imaging.hpp ----------------------------------------- */
/* gaussian_smooth (imaging.hpp:42-44, imaging.cpp:33-63) */
int ffb_gaussian_smooth(ffb_ctx* ctx, int W, int H, const double* in, double sigma,
                        double* out);
/* compute_derivatives (imaging.hpp:54-56, imaging.cpp:65-106) */
int ffb_compute_derivatives(ffb_ctx* ctx, int W, int H, const double* f0, const double* f1,
                            double* fx, double* fy, double* ft, double* f);
/* build_data_terms (imaging.hpp:69, imaging.cpp:108-138) */
int ffb_build_data_terms(ffb_ctx* ctx, int W, int H, const double* fx, const double* fy,
                         const double* ft, const double* f, double rho, double* out10);
/* run_on_frames' imaging prefix: smooth x2 -> derivatives -> data terms (pipeline.cpp:49-52) */
int ffb_frames_to_terms(ffb_ctx* ctx, int W, int H, const double* f0, const double* f1,
                        double sigma, double rho, double* out10);

/* ---- decomposition: include/flowfem/schwarz.hpp (host-only, bit-exact) ------------- */
/* enumerate_splits (schwarz.hpp:16, schwarz.cpp:16-30); returns count written or -1 */
int ffb_enumerate_splits(int W, int H, int n_parts, int* px, int* py, double* ratio, int cap);
/* choose_split (schwarz.hpp:19, schwarz.cpp:32-44) */
int ffb_choose_split(int W, int H, int n_parts, int* px, int* py, double* ratio);
/* build_partition (schwarz.hpp:52, schwarz.cpp:54-128): returns the flat length
 * (writes when cap suffices) or -1 */
long ffb_build_partition(int W, int H, int px, int py, int ov, int* buf, long cap);
/* assign_workers (schwarz.hpp:56, schwarz.cpp:46-52) */
int ffb_assign_workers(int n_workers, int n_parts, int* out);

/* ---- linsolve boundary: include/flowfem/linsolve.hpp ---------------
 * An explicit SparseSystem in CSR form (assembly.hpp:43-53): n scalar unknowns, both
 * triangles stored, row_ptr[n+1] / cols[nnz] / vals[nnz], free vertex major, component minor.
 * Host buffers in and out; the arithmetic runs on the device. */
#define FFB_SOLVE_CHOLESKY 0 /* SolveMethod::DirectCholesky (linsolve.hpp:10) */
#define FFB_SOLVE_CG 1       /* SolveMethod::ConjugateGradient */
/* y = A x in CSR order (spmv, assembly.hpp:76, assembly.cpp:240-249); bitwise */
int ffb_csr_spmv(ffb_ctx* ctx, int n, const int* row_ptr, const int* cols, const double* vals,
                 const double* x, double* y);
/* rcm_order (linsolve.hpp:22-24, linsolve.cpp:37-83): perm[new] = old; bit-exact */
int ffb_rcm_order(int n, int components, const int* row_ptr, const int* cols, int* perm);
/* cg_solve (linsolve.hpp:53-56, linsolve.cpp:298-361): Jacobi-PCG, det_dot reductions,
 * true-residual stop at tol, max_iters 0 -> 10 n, optional warm start; bitwise equal to the
 * reference's iterates, iteration count and residual. Errors: "linsolve.cg: ..." */
int ffb_csr_cg_solve(ffb_ctx* ctx, int n, const int* row_ptr, const int* cols,
                     const double* vals, const double* rhs, double tol, int max_iters,
                     const double* warm, double* x, int* iters, double* res);
/* solve (linsolve.hpp:58-62, linsolve.cpp:363-399): zero right-hand side -> zero vector;
 * FFB_SOLVE_CG -> cg_solve; FFB_SOLVE_CHOLESKY -> band Cholesky of the RCM-ordered matrix
 * on the device, one step of iterative refinement, res = ||b - A x|| / ||b||.
 * Errors: "linsolve.cholesky: breakdown at pivot k (unknown u): ..." */
int ffb_csr_solve(ffb_ctx* ctx, int n, int components, const int* row_ptr, const int* cols,
                  const double* vals, const double* rhs, int method, double tol, int max_iters,
                  const double* warm, double* x, int* iters, double* res);

/* assemble (assembly.hpp:59-61, assembly.cpp:32-166) as an explicit CSR SparseSystem with an
 * optional Dirichlet set (n_dir vertices, nc values each): pattern on the host, values and the
 * eliminated right-hand side from the device operator, bitwise equal to the reference. Call
 * with row_ptr == NULL for n and nnz, then with row_ptr[n+1], cols[nnz], vals[nnz], rhs[n]
 * and (optional) vert_to_free[W*H], free_to_vert[n/nc]. */
int ffb_assemble_system(ffb_ctx* ctx, int W, int H, const double* t10, const double* alpha,
                        const double* lambda, int nc, int n_dir, const int* dir_vertices,
                        const double* dir_values, int* n, long long* nnz, int* row_ptr,
                        int* cols, double* vals, double* rhs, int* vert_to_free,
                        int* free_to_vert);
/* SparseCholesky (linsolve.hpp:32-48): analyze = the reference's RCM order (bit-exact) + band
 * width; factorize = band Cholesky of the permuted matrix on the device ("linsolve.cholesky:
 * breakdown at pivot k (unknown u): matrix is not positive definite"); solve = permuted
 * substitutions on the device. Handles belong to a context. */
typedef struct ffb_chol ffb_chol;
int ffb_chol_create(ffb_ctx* ctx, ffb_chol** chol);
int ffb_chol_destroy(ffb_chol* chol);
int ffb_chol_analyze(ffb_chol* chol, int n, int components, const int* row_ptr, const int* cols);
int ffb_chol_factorize(ffb_chol* chol, int n, const double* vals);
int ffb_chol_solve(ffb_chol* chol, int n, const double* b, double* x);
/* band width of the permuted matrix and stored factor entries (lower band) */
int ffb_chol_info(ffb_chol* chol, int* bandwidth, long long* factor_nonzeros);

/* ---- I/O and evaluation: include/flowfem/imaging.hpp, metrics.hpp ---
 * load_image (imaging.hpp, image_io.cpp:136-145): binary PGM (8/16 bit) or non-interlaced
 * PNG, normalised to [0,1] (RGB -> 0.299 R + 0.587 G + 0.114 B). Call with out == NULL to
 * get W, H; then with *W, *H set and out of W*H doubles. */
int ffb_load_image(const char* path, int* W, int* H, double* out);
/* save_pgm (image_io.cpp:147-160): clamp to [0,1], 8-bit */
int ffb_save_pgm(const char* path, int W, int H, const double* img);
/* read_flo / write_flo (metrics.hpp:28-29, metrics.cpp:22-64): Middlebury .flo, float32
 * u, v planes of W*H; read with u == v == NULL for the size first */
int ffb_read_flo(const char* path, int* W, int* H, float* u, float* v);
int ffb_write_flo(const char* path, int W, int H, const float* u, const float* v);
/* compute_metrics (metrics.hpp:41, metrics.cpp:75-100) as a device reduction: average
 * angular error [deg] and endpoint error over pixels with valid truth (|u|,|v| <= 1e9) */
int ffb_compute_metrics(ffb_ctx* ctx, int W, int H, const double* u1, const double* u2,
                        const float* tu, const float* tv, double* aae_deg, double* ee,
                        long long* valid);

/* ---- operator: include/flowfem/assembly.hpp --------------------------------------- */
/* y = A x and b of the unconstrained global system: assemble (assembly.hpp:59-61,
 * assembly.cpp:32-166) followed by spmv (assembly.hpp:76, assembly.cpp:240-249), computed
 * matrix-free on the device. x3/y3/b3 are planes3. */
int ffb_assemble_apply(ffb_ctx* ctx, int W, int H, const double* t10, const double* alpha,
                       const double* lambda, int nc, const double* x3, double* y3, double* b3);

/* ---- adaptation: include/flowfem/adapt.hpp ----------------------------------------- */
/* error_indicator (adapt.hpp:20-23, adapt.cpp:9-99); eta may be NULL */
int ffb_error_indicator(ffb_ctx* ctx, int W, int H, const double* t10, const double* alpha,
                        const double* lambda, const double* u3, int nc, double* eta,
                        double* eta_max);
/* update_alpha (adapt.hpp:34-35, adapt.cpp:101-112) */
int ffb_update_alpha(ffb_ctx* ctx, int ntri, const double* alpha, const double* eta,
                     double eta_max, double kappa, double eta_thr, double alpha_th,
                     double* alpha_out);

/* ---- stateful solver: the Schwarz-preconditioned solve of the global system -------- */
/* Replaces the linear solve inside the adaptive loop (linsolve.hpp:53-62 on the global
 * system; schwarz_solve's subdomain factorizations, schwarz.cpp:228-252). The system
 * stays on the device between calls. */
int ffb_set_terms(ffb_ctx* ctx, int W, int H, const double* t10);
int ffb_set_frames(ffb_ctx* ctx, int W, int H, const double* f0, const double* f1,
                   double sigma, double rho);
int ffb_set_reg(ffb_ctx* ctx, const double* alpha, const double* lambda);
int ffb_get_reg(ffb_ctx* ctx, double* alpha, double* lambda);
int ffb_set_partition(ffb_ctx* ctx, int px, int py, int overlap);
/* the caller's Partition in the flat format above (schwarz_solve's `const Partition&`); it
 * must be the grid build_partition makes for its (W, H, px, py, ov) */
int ffb_set_partition_flat(ffb_ctx* ctx, const int* flat, long len);
/* Additive-Schwarz-preconditioned CG to ||b-Au||/||b|| <= tol (true residual,
 * linsolve.cpp:314-356). u3 (planes3): warm start on input if warm != 0, solution on
 * output. Refactors the subdomain band factors iff alpha changed since the last factor. */
int ffb_pcg_solve(ffb_ctx* ctx, int nc, double tol, int max_iters, int warm, double* u3,
                  int* iters, double* residual);
/* error_indicator + update_alpha on the resident state (adapt.cpp:9-112) */
int ffb_adapt(ffb_ctx* ctx, int nc, double kappa, double eta_thr, double alpha_th,
              double* eta_max);

/* SchwarzOptions (schwarz.hpp:59-66) with its AdaptConfig (adapt.hpp:24-30) and
 * SolverConfig (linsolve.hpp:12-17) flattened. */
typedef struct ffb_schwarz_options {
  int n_iters;              /* 10 */
  int workers;              /* accepted for signature parity; the device ignores it (results are
                               independent of workers in the reference too) */
  int components;           /* 3, or 2 without the illumination field */
  int adapt;                /* AdaptConfig::enabled */
  int n_adapt;              /* AdaptConfig::n_adapt: iterations that update alpha */
  double kappa, eta_threshold, alpha_th;
  int method;               /* FFB_SOLVE_CHOLESKY | FFB_SOLVE_CG (SolverConfig::method) */
  int cg_max_iters;         /* SolverConfig::cg_max_iters, 0 -> 10 n */
  double cg_tolerance;      /* SolverConfig::cg_tolerance */
  int record_alpha_history; /* SchwarzOptions::record_alpha_history */
} ffb_schwarz_options;

/* SchwarzStats (schwarz.hpp:68-73): caller-owned arrays, each may be NULL. */
typedef struct ffb_schwarz_stats {
  double* increments;    /* [n_iters] max-norm change of the composed field */
  double* seconds;       /* [n_iters] wall time per iteration (adds one sync per iteration) */
  double* eta_max;       /* [min(n_adapt, n_iters)] indicator max per alpha update */
  double* alpha_history; /* [min(n_adapt, n_iters) * ntri] alpha after each update, when
                            record_alpha_history != 0 */
  int n_updates;         /* out: alpha updates performed */
} ffb_schwarz_stats;

/* schwarz_solve (schwarz.hpp:79-81, schwarz.cpp:162-319): the reference's own synchronous
 * restricted-additive-Schwarz loop on the resident terms / reg / partition — per iteration
 * every subdomain solves its Dirichlet problem with traces from the previous composed field,
 * cores are composed, increments[it] = max-norm change; with adapt, alpha is updated after
 * each of the first n_adapt iterations and the subdomain operators follow. Subdomain solver:
 * FFB_SOLVE_CHOLESKY = the device factorisation + one refinement step (schwarz.cpp:236-247);
 * FFB_SOLVE_CG = the reference's Jacobi-PCG per subdomain warm-started from the previous
 * iteration's subdomain solution (schwarz.cpp:248-252), bitwise equal to the reference's.
 * u3: planes3 out. Resident alpha is updated in place (RegField& reg). */
int ffb_schwarz_run(ffb_ctx* ctx, const ffb_schwarz_options* opt, double* u3,
                    ffb_schwarz_stats* stats);
/* ABI-1 form of ffb_schwarz_run with the Cholesky subdomain solver (refine must be 1). */
int ffb_schwarz_solve(ffb_ctx* ctx, int n_iters, int nc, int adapt, int n_adapt, double kappa,
                      double eta_thr, double alpha_th, int refine, double* u3,
                      double* increments, double* eta_max);

/* energy (assembly.hpp:70-73, assembly.cpp:201-238): the discrete energy whose gradient is
 * A x - b, as a deterministic device reduction (u3 planes3). */
int ffb_energy(ffb_ctx* ctx, int W, int H, const double* t10, const double* alpha,
               const double* lambda, const double* u3, int nc, double* e);
/* energy of the resident solution with the resident terms and regularisation */
int ffb_energy_resident(ffb_ctx* ctx, int nc, double* e);

/* ---- multi-GPU: one rank per GPU, the exchange inside the library -----
 * Rank r of `world` owns the band of subdomain rows [r py / world, (r+1) py / world) and the
 * pixel rows of their cores; it factors and solves only those subdomains and runs the CG
 * kernels on its rows. Per CG iteration the library exchanges, with the neighbouring ranks
 * only: the residual on the rows its subdomains reach into (overlap width), the partial
 * subdomain sums of z on the rows it covers in a neighbour's band, and one row of z; the CG
 * scalars are all-reduced as per-subdomain-row values and summed in a fixed order, so the
 * iterates, iteration counts and results are BITWISE identical for every world size at equal
 * subdomain-solve cluster size (each rank sizes its clusters from its own subdomains; a
 * different size reorders the sums inside the line solves: equal to the solve tolerance). After
 * each solve every rank holds the whole solution. Set a communicator, then call
 * ffb_run_on_frames / ffb_run_on_frames_dev / ffb_pcg_solve on every rank with the same
 * inputs; the call returns when the distributed solve is done. */
typedef struct ffb_local_hub ffb_local_hub;
/* NCCL (P2P ncclSend/ncclRecv over NVLink, ncclAllReduce, ncclBroadcast): rank 0 makes the
 * 128-byte unique id, the caller shares it (torch.distributed, MPI, a file), every rank then
 * calls ffb_comm_init_nccl with its rank. libnccl.so.2 is loaded at run time. */
int ffb_comm_nccl_id(unsigned char* id128);
int ffb_comm_init_nccl(ffb_ctx* ctx, int rank, int world, const unsigned char* id128);
/* In-process communicator for N contexts driven by N host threads (on one or several
 * devices): the same protocol with host rendezvous and device copies — for tests and for a
 * single process that drives several GPUs. */
int ffb_comm_local_hub(int world, ffb_local_hub** hub);
int ffb_comm_local_hub_destroy(ffb_local_hub* hub);
int ffb_comm_init_local(ffb_ctx* ctx, ffb_local_hub* hub, int rank);
/* rank / world of the context; rows (may be NULL, needs a partition): the 12 ints
 * y0 y1 j0 j1 fa0 fa1 fb0 fb1 ra0 ra1 rb0 rb1 of ffb_comm_rows */
int ffb_comm_info(ffb_ctx* ctx, int* rank, int* world, int* rows);
/* Host-only row geometry of rank/world for build_partition(W, H, px, py, ov): owned pixel
 * rows [y0,y1), subdomain rows [j0,j1), rows its subdomains cover above [fa0,fa1) and below
 * [fb0,fb1) (its halo of r; its partial z goes there), and its rows covered by the rank
 * above [ra0,ra1) / below [rb0,rb1). */
int ffb_comm_rows(int W, int H, int px, int py, int ov, int rank, int world, int* rows12);

/* run_on_frames (pipeline.hpp:53, pipeline.cpp:38-78) under the converged-pass protocol:
 * n_passes x {solve to tol, error_indicator, update_alpha} + one final solve.
 * u3: planes3 out; alpha: per-triangle out (may be NULL); stats may be NULL. */
int ffb_run_on_frames(ffb_ctx* ctx, int W, int H, const double* f0, const double* f1,
                      const ffb_run_config* cfg, double* u3, double* alpha,
                      ffb_run_stats* stats);
/* Same with DEVICE pointers (frames and u3 resident in HBM), on the context's stream. */
int ffb_run_on_frames_dev(ffb_ctx* ctx, int W, int H, const double* d_f0, const double* d_f1,
                          const ffb_run_config* cfg, double* d_u3, ffb_run_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
