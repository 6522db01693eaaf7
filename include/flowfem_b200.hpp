// flowfem_b200.hpp — header-only C++ host layer over the C-ABI (flowfem_b200.h) that keeps
// the reference library's hot-path API (namespace flowfem, /root/reference/proj/include/
// flowfem/*.hpp): same function names, argument meaning and std::runtime_error messages
// ("<module>.<op>: ..."). A C++ caller of the reference switches by including this header
// and linking libflowfem_b200.so; types are the reference's value types restated minimally.
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "flowfem_b200.h"

namespace flowfem_b200 {

inline void check(int rc) {
  if (rc != 0) throw std::runtime_error(ffb_last_error());
}

// imaging.hpp:10-21
struct Image {
  int width = 0, height = 0;
  std::vector<double> data;
  Image() = default;
  Image(int w, int h) : width(w), height(h), data(static_cast<size_t>(w) * h, 0.0) {}
};

// imaging.hpp:61-67 (planes a11..c back to back)
struct DataTerms {
  int width = 0, height = 0;
  std::vector<double> planes;  // 10 * W * H
};

// assembly.hpp:11-22
struct FlowState {
  int width = 0, height = 0;
  std::vector<double> u1, u2, mt;
};

// assembly.hpp:25-30
struct RegField {
  std::vector<double> alpha, lambda;
};

// schwarz.hpp:11-48
struct SplitChoice {
  int parts_x = 1, parts_y = 1;
  double ratio = 0.0;
};
struct Rect {
  int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
  int w() const { return x1 - x0; }
  int h() const { return y1 - y0; }
};
struct Subdomain {
  Rect core, ext;
  struct Neighbor {
    int part;
    Rect band;
    std::vector<int> gamma;
  };
  std::vector<Neighbor> neighbors;
  std::vector<int> boundary;
};
struct Partition {
  int width = 0, height = 0, parts_x = 1, parts_y = 1, overlap = 0;
  std::vector<Subdomain> parts;
};

// pipeline.hpp:15-33 (solver fields)
struct RunConfig {
  double sigma = 1.0, rho = 2.5, alpha0 = 1000.0, lambda0 = 1000.0;
  bool illumination = true;
  int parts = 4, overlap = 5;
  bool adapt = true;
  double kappa = 10.0, eta_threshold = 0.1, alpha_th = -1.0;  // <= 0 -> alpha0/100
  int adapt_iters = 10;
  double cg_tolerance = 1e-10;
  int max_iters = 0;
};

struct RunResult {
  FlowState flow;
  RegField reg;
  ffb_run_stats stats{};
  int width = 0, height = 0;
};

// One GPU; owns the device-resident solver state (one process per GPU).
class Context {
 public:
  explicit Context(int device = 0) { check(ffb_create(&ctx_, device)); }
  ~Context() { ffb_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ffb_ctx* get() const { return ctx_; }

 private:
  ffb_ctx* ctx_ = nullptr;
};

// ---- decomposition (host-only, bit-exact): schwarz.hpp:16-57 ---------------------------
inline std::vector<SplitChoice> enumerate_splits(int width, int height, int n_parts) {
  std::vector<int> px(n_parts > 0 ? n_parts : 1), py(px.size());
  std::vector<double> ratio(px.size());
  const int n = ffb_enumerate_splits(width, height, n_parts, px.data(), py.data(), ratio.data(),
                                     static_cast<int>(px.size()));
  if (n < 0) throw std::runtime_error(ffb_last_error());
  std::vector<SplitChoice> out(n);
  for (int i = 0; i < n; ++i) out[i] = {px[i], py[i], ratio[i]};
  return out;
}

inline SplitChoice choose_split(int width, int height, int n_parts) {
  SplitChoice s;
  check(ffb_choose_split(width, height, n_parts, &s.parts_x, &s.parts_y, &s.ratio));
  return s;
}

inline std::vector<int> assign_workers(int n_workers, int n_parts) {
  std::vector<int> a(n_workers > 0 ? n_workers : 1);
  check(ffb_assign_workers(n_workers, n_parts, a.data()));
  a.resize(n_workers > 0 ? n_workers : 0);
  return a;
}

inline Partition build_partition(int width, int height, int parts_x, int parts_y, int overlap) {
  const long need = ffb_build_partition(width, height, parts_x, parts_y, overlap, nullptr, 0);
  if (need < 0) throw std::runtime_error(ffb_last_error());
  std::vector<int> f(need);
  ffb_build_partition(width, height, parts_x, parts_y, overlap, f.data(), need);
  Partition P;
  P.width = f[0], P.height = f[1], P.parts_x = f[2], P.parts_y = f[3], P.overlap = f[4];
  const int np = f[5];
  P.parts.resize(np);
  std::vector<int> nb(np), nn(np);
  for (int p = 0; p < np; ++p) {
    const int* h = &f[6 + 10 * p];
    P.parts[p].core = {h[0], h[1], h[2], h[3]};
    P.parts[p].ext = {h[4], h[5], h[6], h[7]};
    nb[p] = h[8];
    nn[p] = h[9];
  }
  size_t pos = 6 + 10 * static_cast<size_t>(np);
  for (int p = 0; p < np; ++p) {
    P.parts[p].boundary.assign(f.begin() + pos, f.begin() + pos + nb[p]);
    pos += nb[p];
    for (int k = 0; k < nn[p]; ++k) {
      Subdomain::Neighbor n;
      n.part = f[pos];
      n.band = {f[pos + 1], f[pos + 2], f[pos + 3], f[pos + 4]};
      const int g = f[pos + 5];
      n.gamma.assign(f.begin() + pos + 6, f.begin() + pos + 6 + g);
      pos += 6 + g;
      P.parts[p].neighbors.push_back(std::move(n));
    }
  }
  return P;
}

// ---- imaging: imaging.hpp:42-69 -----------------------------------------------------------
inline Image gaussian_smooth(Context& c, const Image& img, double sigma) {
  Image out(img.width, img.height);
  check(ffb_gaussian_smooth(c.get(), img.width, img.height, img.data.data(), sigma,
                            out.data.data()));
  return out;
}

inline DataTerms frames_to_terms(Context& c, const Image& f0, const Image& f1, double sigma,
                                 double rho) {
  if (f0.width != f1.width || f0.height != f1.height)
    throw std::runtime_error("imaging.compute_derivatives: frame sizes differ");
  DataTerms t;
  t.width = f0.width;
  t.height = f0.height;
  t.planes.resize(10 * static_cast<size_t>(f0.width) * f0.height);
  check(ffb_frames_to_terms(c.get(), f0.width, f0.height, f0.data.data(), f1.data.data(), sigma,
                            rho, t.planes.data()));
  return t;
}

// ---- adaptation: adapt.hpp:20-35 ---------------------------------------------------------
inline double error_indicator(Context& c, const DataTerms& dt, const RegField& reg,
                              const FlowState& s, int components, std::vector<double>* eta) {
  const size_t n = static_cast<size_t>(dt.width) * dt.height;
  std::vector<double> u3(3 * n);
  std::copy(s.u1.begin(), s.u1.end(), u3.begin());
  std::copy(s.u2.begin(), s.u2.end(), u3.begin() + n);
  std::copy(s.mt.begin(), s.mt.end(), u3.begin() + 2 * n);
  if (eta) eta->resize(2 * static_cast<size_t>(dt.width - 1) * (dt.height - 1));
  double em = 0.0;
  check(ffb_error_indicator(c.get(), dt.width, dt.height, dt.planes.data(), reg.alpha.data(),
                            reg.lambda.data(), u3.data(), components, eta ? eta->data() : nullptr,
                            &em));
  return em;
}

// ---- linsolve: linsolve.hpp:10-62 on an explicit CSR SparseSystem -----------------------
enum class SolveMethod { DirectCholesky = FFB_SOLVE_CHOLESKY, ConjugateGradient = FFB_SOLVE_CG };
struct SolverConfig {
  SolveMethod method = SolveMethod::DirectCholesky;
  double cg_tolerance = 1e-10;
  int cg_max_iters = 0;  // 0 -> 10 n
};
struct SolveReport {
  int iterations = 0;
  double residual = 0.0;
};
// the CSR part of assembly.hpp:43-53 (free vertex major, component minor, both triangles)
struct SparseSystem {
  int n = 0;
  int components = 3;
  std::vector<int> row_ptr, cols;
  std::vector<double> vals, rhs;
};

inline std::vector<double> spmv(Context& c, const SparseSystem& s, const std::vector<double>& x) {
  std::vector<double> y(s.n);
  check(ffb_csr_spmv(c.get(), s.n, s.row_ptr.data(), s.cols.data(), s.vals.data(), x.data(),
                     y.data()));
  return y;
}

inline std::vector<int> rcm_order(const SparseSystem& s) {
  std::vector<int> perm(s.n);
  check(ffb_rcm_order(s.n, s.components, s.row_ptr.data(), s.cols.data(), perm.data()));
  return perm;
}

inline std::vector<double> cg_solve(Context& c, const SparseSystem& s, const SolverConfig& cfg,
                                    const std::vector<double>* warm_start = nullptr,
                                    SolveReport* report = nullptr) {
  std::vector<double> x(s.n);
  SolveReport r;
  const double* w = warm_start && static_cast<int>(warm_start->size()) == s.n ? warm_start->data()
                                                                            : nullptr;
  const int rc = ffb_csr_cg_solve(c.get(), s.n, s.row_ptr.data(), s.cols.data(), s.vals.data(),
                                  s.rhs.data(), cfg.cg_tolerance, cfg.cg_max_iters, w, x.data(),
                                  &r.iterations, &r.residual);
  if (report) *report = r;
  check(rc);
  return x;
}

inline std::vector<double> solve(Context& c, const SparseSystem& s, const SolverConfig& cfg,
                                 SolveReport* report = nullptr,
                                 const std::vector<double>* warm_start = nullptr) {
  std::vector<double> x(s.n);
  SolveReport r;
  const double* w = warm_start && static_cast<int>(warm_start->size()) == s.n ? warm_start->data()
                                                                            : nullptr;
  const int rc = ffb_csr_solve(c.get(), s.n, s.components, s.row_ptr.data(), s.cols.data(),
                               s.vals.data(), s.rhs.data(), static_cast<int>(cfg.method),
                               cfg.cg_tolerance, cfg.cg_max_iters, w, x.data(), &r.iterations,
                               &r.residual);
  if (report) *report = r;
  check(rc);
  return x;
}

// ---- I/O and evaluation: imaging.hpp load_image / save_pgm, metrics.hpp -----------------
inline Image load_image(const std::string& path) {
  Image img;
  check(ffb_load_image(path.c_str(), &img.width, &img.height, nullptr));
  img.data.resize(static_cast<size_t>(img.width) * img.height);
  check(ffb_load_image(path.c_str(), &img.width, &img.height, img.data.data()));
  return img;
}

inline void save_pgm(const std::string& path, const Image& img) {
  check(ffb_save_pgm(path.c_str(), img.width, img.height, img.data.data()));
}

struct FloField {
  int width = 0, height = 0;
  std::vector<float> u, v;
};

inline FloField read_flo(const std::string& path) {
  FloField f;
  check(ffb_read_flo(path.c_str(), &f.width, &f.height, nullptr, nullptr));
  f.u.resize(static_cast<size_t>(f.width) * f.height);
  f.v.resize(f.u.size());
  check(ffb_read_flo(path.c_str(), &f.width, &f.height, f.u.data(), f.v.data()));
  return f;
}

inline void write_flo(const std::string& path, const FloField& f) {
  check(ffb_write_flo(path.c_str(), f.width, f.height, f.u.data(), f.v.data()));
}

inline FloField to_flo(const FlowState& s) {
  FloField f;
  f.width = s.width;
  f.height = s.height;
  f.u.assign(s.u1.begin(), s.u1.end());
  f.v.assign(s.u2.begin(), s.u2.end());
  return f;
}

struct FlowMetrics {
  double aae_deg = 0.0, ee = 0.0;
  long valid = 0;
};

inline FlowMetrics compute_metrics(Context& c, const FlowState& flow, const FloField& truth) {
  if (flow.width != truth.width || flow.height != truth.height)
    throw std::runtime_error("metrics.compute_metrics: flow and ground truth sizes differ");
  FlowMetrics m;
  long long valid = 0;
  check(ffb_compute_metrics(c.get(), truth.width, truth.height, flow.u1.data(), flow.u2.data(),
                            truth.u.data(), truth.v.data(), &m.aae_deg, &m.ee, &valid));
  m.valid = static_cast<long>(valid);
  return m;
}

// ---- pipeline: pipeline.hpp:53 (converged-pass protocol) --------------------------------
inline RunResult run_on_frames(Context& c, const Image& f0, const Image& f1,
                               const RunConfig& cfg) {
  if (f0.width != f1.width || f0.height != f1.height)
    throw std::runtime_error("cli.run: frame sizes differ");
  const int W = f0.width, H = f0.height;
  const size_t n = static_cast<size_t>(W) * H;
  ffb_run_config rc{cfg.sigma,  cfg.rho,           cfg.alpha0,    cfg.lambda0,
                    cfg.illumination ? 1 : 0,      cfg.parts,     cfg.overlap,
                    cfg.adapt ? 1 : 0,             cfg.adapt_iters, cfg.kappa,
                    cfg.eta_threshold,             cfg.alpha_th,  cfg.cg_tolerance,
                    cfg.max_iters};
  RunResult r;
  r.width = W;
  r.height = H;
  std::vector<double> u3(3 * n);
  r.reg.alpha.resize(2 * static_cast<size_t>(W - 1) * (H - 1));
  check(ffb_run_on_frames(c.get(), W, H, f0.data.data(), f1.data.data(), &rc, u3.data(),
                          r.reg.alpha.data(), &r.stats));
  r.reg.lambda.assign(r.reg.alpha.size(), cfg.lambda0);
  r.flow.width = W;
  r.flow.height = H;
  r.flow.u1.assign(u3.begin(), u3.begin() + n);
  r.flow.u2.assign(u3.begin() + n, u3.begin() + 2 * n);
  r.flow.mt.assign(u3.begin() + 2 * n, u3.end());
  return r;
}

}  // namespace flowfem_b200
