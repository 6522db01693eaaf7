/* TEST INFRASTRUCTURE (oracle) — not product code.
 *
 * Plain-C restatement of the reference hot path (arXiv 1508.02977 `flowfem`,
 * /root/reference/proj/src). It is the CPU checker for the B200 kernels and
 * the "port" CPU baseline. It mirrors the reference's floating-point operation
 * order so that, compiled the same way (-O2, no FMA), it reproduces the
 * reference bit for bit; tests pin it against the compiled reference
 * (oracle/_ref) and against the committed golden vectors in tests/golden/.
 *
 * Array conventions: see include/flowfem_b200.h (identical to the product ABI).
 */
#ifndef FLOWFEM_PORT_H
#define FLOWFEM_PORT_H

#ifdef __cplusplus
extern "C" {
#endif

const char* fp_last_error(void);
int fp_set_threads(int n);

int fp_gauss_taps(double sigma, double* taps, int cap);
int fp_gaussian_smooth(int W, int H, const double* in, double sigma, double* out);
int fp_compute_derivatives(int W, int H, const double* f0, const double* f1, double* fx,
                           double* fy, double* ft, double* f);
int fp_build_data_terms(int W, int H, const double* fx, const double* fy, const double* ft,
                        const double* f, double rho, double* out10);
int fp_frames_to_terms(int W, int H, const double* f0, const double* f1, double sigma,
                       double rho, double* out10);

int fp_choose_split(int W, int H, int n_parts, int* px, int* py, double* ratio);
long fp_build_partition(int W, int H, int px, int py, int ov, int* buf, long cap);

int fp_assemble_apply(int W, int H, const double* t10, const double* alpha,
                      const double* lambda, int nc, const double* x3, double* y3, double* b3);
int fp_cg_solve(int W, int H, const double* t10, const double* alpha, const double* lambda,
                int nc, double tol, int max_iters, const double* warm3, double* out3,
                int* iters, double* res);
int fp_csr_spmv(int n, const int* row_ptr, const int* cols, const double* vals, const double* x,
                double* y);
int fp_csr_cg_solve(int n, const int* row_ptr, const int* cols, const double* vals,
                    const double* b, double tol, int max_iters, const double* warm, double* x,
                    int* iters, double* res);
int fp_rcm_order(int n, int nc, const int* row_ptr, const int* cols, int* perm);
int fp_error_indicator(int W, int H, const double* t10, const double* alpha,
                       const double* lambda, const double* u3, int nc, double* eta,
                       double* eta_max);
int fp_update_alpha(int ntri, const double* alpha, const double* eta, double eta_max,
                    double kappa, double eta_thr, double alpha_th, double* alpha_out);
int fp_energy(int W, int H, const double* t10, const double* alpha, const double* lambda,
              const double* u3, int nc, double* e);
int fp_converged_chain(int W, int H, const double* f0, const double* f1, double sigma,
                       double rho, double alpha0, double lambda0, int nc, int n_passes,
                       double kappa, double eta_thr, double alpha_th, double tol, double* out3,
                       double* alpha_out, double* eta_max_out, int* iters_out,
                       double* seconds_out);

#ifdef __cplusplus
}
#endif
#endif
