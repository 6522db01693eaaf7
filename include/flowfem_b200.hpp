// flowfem_b200.hpp — the reference library's C++ API (namespace flowfem; the value types and
// signatures of /root/reference/proj/include/flowfem/*.hpp) implemented over the C-ABI of
// flowfem_b200.h. A C++ caller of the reference switches by putting this repository's
// include/ directory first on its include path (include/flowfem/<name>.hpp forward here) and
// linking libflowfem_b200.so instead of the reference's objects; INTEGRATION.md shows the
// patch. Every numerical function runs on the GPU; the host code below only converts between
// the reference's value types and the flat C arrays, builds the (integer) mesh and partition
// tables, and rethrows library errors as std::runtime_error with the reference's
// "<module>.<op>: ..." messages.
//
// The context is implicit, as in the reference: one process-wide device context (device
// $FFB_DEVICE, default 0), created on first use; like the reference, the API is meant to be
// called from one host thread at a time.
//
// Two deliberate extensions, both opt-in: RunConfig::protocol = "converged" runs the
// converged-pass protocol with the Schwarz-preconditioned CG (the path the
// benchmark measures) instead of the reference's literal Schwarz iteration; and
// b200::context() exposes the context for multi-GPU set-up (flowfem_b200.h ffb_comm_*).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "flowfem_b200.h"

namespace flowfem {

namespace b200 {

inline void check(int rc) {
  if (rc != 0) throw std::runtime_error(ffb_last_error());
}

class Context {
 public:
  explicit Context(int device) { check(ffb_create(&ctx_, device)); }
  ~Context() { ffb_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ffb_ctx* get() const { return ctx_; }

 private:
  ffb_ctx* ctx_ = nullptr;
};

inline Context& context() {
  static Context c(std::getenv("FFB_DEVICE") ? std::atoi(std::getenv("FFB_DEVICE")) : 0);
  return c;
}
inline ffb_ctx* ctx() { return context().get(); }

}  // namespace b200

// =================================================================== imaging.hpp
struct Image {
  int width = 0;
  int height = 0;
  std::vector<double> data;
  Image() = default;
  Image(int w, int h) : width(w), height(h), data(static_cast<size_t>(w) * h, 0.0) {}
  double& at(int x, int y) { return data[static_cast<size_t>(y) * width + x]; }
  double at(int x, int y) const { return data[static_cast<size_t>(y) * width + x]; }
  size_t size() const { return data.size(); }
};

struct RgbImage {
  int width = 0;
  int height = 0;
  std::vector<uint8_t> data;
  RgbImage() = default;
  RgbImage(int w, int h) : width(w), height(h), data(static_cast<size_t>(w) * h * 3, 0) {}
  uint8_t* px(int x, int y) { return &data[(static_cast<size_t>(y) * width + x) * 3]; }
  const uint8_t* px(int x, int y) const { return &data[(static_cast<size_t>(y) * width + x) * 3]; }
};

inline Image load_image(const std::string& path) {
  Image img;
  b200::check(ffb_load_image(path.c_str(), &img.width, &img.height, nullptr));
  img.data.resize(static_cast<size_t>(img.width) * img.height);
  b200::check(ffb_load_image(path.c_str(), &img.width, &img.height, img.data.data()));
  return img;
}

inline void save_pgm(const std::string& path, const Image& img) {
  b200::check(ffb_save_pgm(path.c_str(), img.width, img.height, img.data.data()));
}

inline void save_png_rgb(const std::string&, const RgbImage&) {
  throw std::runtime_error("imaging.save_png_rgb: visualisation output is not part of flowfem_b200");
}

inline Image gaussian_smooth(const Image& img, double sigma) {
  Image out(img.width, img.height);
  b200::check(ffb_gaussian_smooth(b200::ctx(), img.width, img.height, img.data.data(), sigma,
                                  out.data.data()));
  return out;
}

struct DerivativeField {
  int width = 0;
  int height = 0;
  std::vector<double> fx, fy, ft, f;
};

inline DerivativeField compute_derivatives(const Image& f0, const Image& f1) {
  if (f0.width != f1.width || f0.height != f1.height)
    throw std::runtime_error("imaging.compute_derivatives: frame sizes differ");
  DerivativeField d;
  d.width = f0.width;
  d.height = f0.height;
  const size_t n = f0.data.size();
  d.fx.resize(n), d.fy.resize(n), d.ft.resize(n), d.f.resize(n);
  b200::check(ffb_compute_derivatives(b200::ctx(), f0.width, f0.height, f0.data.data(),
                                      f1.data.data(), d.fx.data(), d.fy.data(), d.ft.data(),
                                      d.f.data()));
  return d;
}

struct DataTerms {
  int width = 0;
  int height = 0;
  std::vector<double> a11, a12, a13, a22, a23, a33;
  std::vector<double> f1, f2, f3;
  std::vector<double> c;
};

namespace b200 {
// the ten planes back to back (flowfem_b200.h "terms10") and back
inline std::vector<double> planes(const DataTerms& t) {
  const size_t n = static_cast<size_t>(t.width) * t.height;
  std::vector<double> out(10 * n);
  const std::vector<double>* f[10] = {&t.a11, &t.a12, &t.a13, &t.a22, &t.a23,
                                      &t.a33, &t.f1,  &t.f2,  &t.f3,  &t.c};
  for (int k = 0; k < 10; ++k) {
    if (f[k]->size() != n) throw std::runtime_error("assembly.assemble: data terms size mismatch");
    std::copy(f[k]->begin(), f[k]->end(), out.begin() + k * n);
  }
  return out;
}
inline DataTerms terms(int W, int H, const std::vector<double>& p) {
  DataTerms t;
  t.width = W;
  t.height = H;
  const size_t n = static_cast<size_t>(W) * H;
  std::vector<double>* f[10] = {&t.a11, &t.a12, &t.a13, &t.a22, &t.a23,
                                &t.a33, &t.f1,  &t.f2,  &t.f3,  &t.c};
  for (int k = 0; k < 10; ++k) f[k]->assign(p.begin() + k * n, p.begin() + (k + 1) * n);
  return t;
}
}  // namespace b200

inline DataTerms build_data_terms(const DerivativeField& d, double rho) {
  const size_t n = static_cast<size_t>(d.width) * d.height;
  std::vector<double> out(10 * n);
  b200::check(ffb_build_data_terms(b200::ctx(), d.width, d.height, d.fx.data(), d.fy.data(),
                                   d.ft.data(), d.f.data(), rho, out.data()));
  return b200::terms(d.width, d.height, out);
}

// =================================================================== mesh.hpp
struct TriMesh {
  int width = 0;
  int height = 0;
  int n_vertices = 0;
  int n_triangles = 0;
  std::vector<int> tri;
  std::vector<double> area;
  std::vector<double> hK;
  struct Edge {
    int v0, v1;
    int t0, t1;
    double length;
    double nx, ny;
  };
  std::vector<Edge> edges;
  std::vector<int> tri_edges;
  std::vector<double> lumped;
  std::vector<int> v2t_ptr, v2t;
  std::vector<int> v2v_ptr, v2v;
  int vertex(int x, int y) const { return y * width + x; }
  double vx(int v) const { return v % width; }
  double vy(int v) const { return v / width; }
};

// The half-pixel triangulation of mesh.cpp:8-170 (host integer/geometry tables; the device
// path never materialises them). Cell (x, y): lower triangle 2(y(W-1)+x) = (v00, v10, v11),
// upper +1 = (v00, v11, v01); edges in three blocks (horizontal, vertical, diagonal), t0 < t1
// with the normal pointing from t0 to t1 (outward on the boundary).
inline TriMesh build_pixel_mesh(int width, int height) {
  if (width < 2 || height < 2)
    throw std::runtime_error("mesh.build_pixel_mesh: grid must be at least 2x2");
  TriMesh m;
  m.width = width, m.height = height;
  m.n_vertices = width * height;
  const int cw = width - 1, ch = height - 1;
  m.n_triangles = 2 * cw * ch;
  m.tri.resize(3 * static_cast<size_t>(m.n_triangles));
  m.area.assign(m.n_triangles, 0.5);
  m.hK.assign(m.n_triangles, std::sqrt(2.0));
  auto cell = [cw](int x, int y) { return 2 * (y * cw + x); };  // its lower triangle
  for (int y = 0; y < ch; ++y)
    for (int x = 0; x < cw; ++x) {
      const int v = y * width + x, t = cell(x, y);
      const int lo[3] = {v, v + 1, v + width + 1}, up[3] = {v, v + width + 1, v + width};
      std::copy(lo, lo + 3, &m.tri[3 * static_cast<size_t>(t)]);
      std::copy(up, up + 3, &m.tri[3 * static_cast<size_t>(t) + 3]);
    }
  const int nh = cw * height, nvv = width * ch, nd = cw * ch;
  m.edges.resize(static_cast<size_t>(nh) + nvv + nd);
  // an edge between triangles a (on the side the unit normal (nx, ny) leaves) and b
  auto neg = [](double v) { return v == 0.0 ? 0.0 : -v; };  // no negative zeros
  auto edge = [&](int v0, int v1, double len, int a, int b, double nx, double ny) {
    TriMesh::Edge e{v0, v1, a, b, len, nx, ny};
    if (a < 0) e.t0 = b, e.t1 = -1, e.nx = neg(nx), e.ny = neg(ny);  // boundary: outward from b
    else if (b < 0) e.t1 = -1;                                      // boundary: outward from a
    else if (b < a) e.t0 = b, e.t1 = a, e.nx = neg(nx), e.ny = neg(ny);
    return e;
  };
  for (int y = 0; y < height; ++y)
    for (int x = 0; x < cw; ++x) {  // from the upper triangle below to the lower one above
      const int below = y > 0 ? cell(x, y - 1) + 1 : -1, above = y < ch ? cell(x, y) : -1;
      const int v = y * width + x;
      m.edges[y * cw + x] = edge(v, v + 1, 1.0, below, above, 0.0, 1.0);
    }
  for (int y = 0; y < ch; ++y)
    for (int x = 0; x < width; ++x) {  // from the lower triangle left to the upper one right
      const int left = x > 0 ? cell(x - 1, y) : -1, right = x < cw ? cell(x, y) + 1 : -1;
      const int v = y * width + x;
      m.edges[nh + y * width + x] = edge(v, v + width, 1.0, left, right, 1.0, 0.0);
    }
  const double s = 1.0 / std::sqrt(2.0);
  for (int y = 0; y < ch; ++y)
    for (int x = 0; x < cw; ++x) {  // from the lower triangle to the upper one
      const int v = y * width + x;
      m.edges[nh + nvv + y * cw + x] =
          TriMesh::Edge{v, v + width + 1, cell(x, y), cell(x, y) + 1, std::sqrt(2.0), -s, s};
    }
  m.tri_edges.resize(3 * static_cast<size_t>(m.n_triangles));
  for (int y = 0; y < ch; ++y)
    for (int x = 0; x < cw; ++x) {
      const int t = cell(x, y), d = nh + nvv + y * cw + x;
      const int lo[3] = {y * cw + x, nh + y * width + x + 1, d};
      const int up[3] = {d, (y + 1) * cw + x, nh + y * width + x};
      std::copy(lo, lo + 3, &m.tri_edges[3 * static_cast<size_t>(t)]);
      std::copy(up, up + 3, &m.tri_edges[3 * static_cast<size_t>(t) + 3]);
    }
  // per-vertex tables: the incident triangles and neighbours of (x, y), ascending ids
  m.lumped.assign(m.n_vertices, 0.0);
  m.v2t_ptr.assign(m.n_vertices + 1, 0);
  m.v2v_ptr.assign(m.n_vertices + 1, 0);
  m.v2t.reserve(3 * static_cast<size_t>(m.n_triangles));
  m.v2v.reserve(2 * m.edges.size());
  for (int v = 0; v < m.n_vertices; ++v) {
    const int x = v % width, y = v / width;
    const bool l = x > 0, r = x < cw, d = y > 0, u = y < ch;
    if (l && d) m.v2t.push_back(cell(x - 1, y - 1)), m.v2t.push_back(cell(x - 1, y - 1) + 1);
    if (r && d) m.v2t.push_back(cell(x, y - 1) + 1);
    if (l && u) m.v2t.push_back(cell(x - 1, y));
    if (r && u) m.v2t.push_back(cell(x, y)), m.v2t.push_back(cell(x, y) + 1);
    m.v2t_ptr[v + 1] = static_cast<int>(m.v2t.size());
    for (int k = m.v2t_ptr[v]; k < m.v2t_ptr[v + 1]; ++k) m.lumped[v] += m.area[m.v2t[k]] / 3.0;
    if (l && d) m.v2v.push_back(v - width - 1);
    if (d) m.v2v.push_back(v - width);
    if (l) m.v2v.push_back(v - 1);
    if (r) m.v2v.push_back(v + 1);
    if (u) m.v2v.push_back(v + width);
    if (r && u) m.v2v.push_back(v + width + 1);
    m.v2v_ptr[v + 1] = static_cast<int>(m.v2v.size());
  }
  return m;
}

// constant P1 hat gradients on triangle t: rot90(p_b - p_a) / (2 area) for hat k opposite
// the edge (a, b) = (k+1, k+2) (mesh.cpp:172-186)
inline void p1_gradients(const TriMesh& m, int t, double gx[3], double gy[3]) {
  const int* v = &m.tri[3 * static_cast<size_t>(t)];
  const double twoA = 2.0 * m.area[t];
  for (int k = 0; k < 3; ++k) {
    const int a = v[(k + 1) % 3], b = v[(k + 2) % 3];
    gx[k] = -(m.vy(b) - m.vy(a)) / twoA;
    gy[k] = (m.vx(b) - m.vx(a)) / twoA;
  }
}

// =================================================================== assembly.hpp
struct FlowState {
  int width = 0;
  int height = 0;
  std::vector<double> u1, u2, mt;
  FlowState() = default;
  FlowState(int w, int h)
      : width(w), height(h), u1(static_cast<size_t>(w) * h, 0.0),
        u2(static_cast<size_t>(w) * h, 0.0), mt(static_cast<size_t>(w) * h, 0.0) {}
};

struct RegField {
  std::vector<double> alpha;
  std::vector<double> lambda;
};

inline RegField uniform_reg(const TriMesh& m, double alpha0, double lambda0) {
  RegField r;
  r.alpha.assign(m.n_triangles, alpha0);
  r.lambda.assign(m.n_triangles, lambda0);
  return r;
}

struct DirichletSet {
  std::vector<int> vertices;
  std::vector<double> values;
  bool empty() const { return vertices.empty(); }
};

struct SparseSystem {
  int n = 0;
  int components = 3;
  std::vector<int> row_ptr, cols;
  std::vector<double> vals;
  std::vector<double> rhs;
  std::vector<int> vert_to_free;
  std::vector<int> free_to_vert;
  DirichletSet constraints;
};

namespace b200 {
inline std::vector<double> planes3(const FlowState& s) {
  const size_t n = s.u1.size();
  std::vector<double> p(3 * n, 0.0);
  std::copy(s.u1.begin(), s.u1.end(), p.begin());
  std::copy(s.u2.begin(), s.u2.end(), p.begin() + n);
  if (s.mt.size() == n) std::copy(s.mt.begin(), s.mt.end(), p.begin() + 2 * n);
  return p;
}
inline FlowState state(int W, int H, const std::vector<double>& p) {
  FlowState s(W, H);
  const size_t n = static_cast<size_t>(W) * H;
  std::copy(p.begin(), p.begin() + n, s.u1.begin());
  std::copy(p.begin() + n, p.begin() + 2 * n, s.u2.begin());
  std::copy(p.begin() + 2 * n, p.begin() + 3 * n, s.mt.begin());
  return s;
}
inline void check_reg(const TriMesh& m, const RegField& reg) {
  if (static_cast<int>(reg.alpha.size()) != m.n_triangles ||
      static_cast<int>(reg.lambda.size()) != m.n_triangles)
    throw std::runtime_error("assembly.assemble: regularization field size mismatch");
}
}  // namespace b200

inline SparseSystem assemble(const TriMesh& m, const DataTerms& dt, const RegField& reg,
                             int components, const DirichletSet* dirichlet = nullptr) {
  if (components != 2 && components != 3)
    throw std::runtime_error("assembly.assemble: components must be 2 or 3");
  if (dt.width != m.width || dt.height != m.height)
    throw std::runtime_error("assembly.assemble: data terms do not match the mesh");
  b200::check_reg(m, reg);
  const int nd = dirichlet ? static_cast<int>(dirichlet->vertices.size()) : 0;
  if (nd && dirichlet->values.size() != static_cast<size_t>(nd) * components)
    throw std::runtime_error("assembly.assemble: Dirichlet values size mismatch");
  const std::vector<double> t10 = b200::planes(dt);
  SparseSystem s;
  s.components = components;
  if (dirichlet) s.constraints = *dirichlet;
  long long nnz = 0;
  const int* dv = nd ? dirichlet->vertices.data() : nullptr;
  const double* dval = nd ? dirichlet->values.data() : nullptr;
  b200::check(ffb_assemble_system(b200::ctx(), m.width, m.height, t10.data(), reg.alpha.data(),
                                  reg.lambda.data(), components, nd, dv, dval, &s.n, &nnz,
                                  nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
  s.row_ptr.resize(s.n + 1);
  s.cols.resize(nnz);
  s.vals.resize(nnz);
  s.rhs.resize(s.n);
  s.vert_to_free.resize(m.n_vertices);
  s.free_to_vert.resize(s.n / components);
  b200::check(ffb_assemble_system(b200::ctx(), m.width, m.height, t10.data(), reg.alpha.data(),
                                  reg.lambda.data(), components, nd, dv, dval, &s.n, &nnz,
                                  s.row_ptr.data(), s.cols.data(), s.vals.data(), s.rhs.data(),
                                  s.vert_to_free.data(), s.free_to_vert.data()));
  return s;
}

inline FlowState expand_solution(const TriMesh& m, const SparseSystem& sys,
                                 const std::vector<double>& x) {
  if (static_cast<int>(x.size()) != sys.n)
    throw std::runtime_error("assembly.expand_solution: size mismatch");
  const int nc = sys.components;
  FlowState s(m.width, m.height);
  std::vector<double>* f[3] = {&s.u1, &s.u2, &s.mt};
  for (size_t k = 0; k < sys.free_to_vert.size(); ++k)
    for (int c = 0; c < nc; ++c) (*f[c])[sys.free_to_vert[k]] = x[k * nc + c];
  const DirichletSet& d = sys.constraints;
  for (size_t k = 0; k < d.vertices.size(); ++k)
    for (int c = 0; c < nc; ++c) (*f[c])[d.vertices[k]] = d.values[k * nc + c];
  return s;
}

inline std::vector<double> flatten_state(const SparseSystem& sys, const FlowState& state) {
  const int nc = sys.components;
  const std::vector<double>* f[3] = {&state.u1, &state.u2, &state.mt};
  std::vector<double> x(sys.n);
  for (size_t k = 0; k < sys.free_to_vert.size(); ++k)
    for (int c = 0; c < nc; ++c) x[k * nc + c] = (*f[c])[sys.free_to_vert[k]];
  return x;
}

inline double energy(const TriMesh& m, const DataTerms& dt, const RegField& reg,
                     const FlowState& state, int components = 3) {
  b200::check_reg(m, reg);
  const std::vector<double> t10 = b200::planes(dt), u3 = b200::planes3(state);
  double e = 0.0;
  b200::check(ffb_energy(b200::ctx(), m.width, m.height, t10.data(), reg.alpha.data(),
                         reg.lambda.data(), u3.data(), components, &e));
  return e;
}

inline void spmv(const SparseSystem& sys, const std::vector<double>& x, std::vector<double>& y) {
  y.resize(sys.n);
  b200::check(ffb_csr_spmv(b200::ctx(), sys.n, sys.row_ptr.data(), sys.cols.data(),
                           sys.vals.data(), x.data(), y.data()));
}

// =================================================================== linsolve.hpp
enum class SolveMethod { DirectCholesky, ConjugateGradient };

struct SolverConfig {
  SolveMethod method = SolveMethod::DirectCholesky;
  double cg_tolerance = 1e-10;
  int cg_max_iters = 0;
  int factor_workers = 1;  // accepted; the factorisation runs on the device
};

struct SolveReport {
  int iterations = 0;
  double residual = 0.0;
};

inline std::vector<int> rcm_order(const SparseSystem& sys) {
  std::vector<int> perm(sys.n);
  b200::check(ffb_rcm_order(sys.n, sys.components, sys.row_ptr.data(), sys.cols.data(),
                            perm.data()));
  return perm;
}

class SparseCholesky {
 public:
  SparseCholesky() = default;
  ~SparseCholesky() {
    if (h_) ffb_chol_destroy(h_);
  }
  SparseCholesky(SparseCholesky&& o) noexcept : h_(o.h_), n_(o.n_) { o.h_ = nullptr; }
  SparseCholesky& operator=(SparseCholesky&& o) noexcept {
    std::swap(h_, o.h_);
    std::swap(n_, o.n_);
    return *this;
  }
  void analyze(const SparseSystem& sys) {
    if (!h_) b200::check(ffb_chol_create(b200::ctx(), &h_));
    b200::check(ffb_chol_analyze(h_, sys.n, sys.components, sys.row_ptr.data(), sys.cols.data()));
    n_ = sys.n;
    analyzed_ = true;
  }
  void factorize(const SparseSystem& sys, int /*workers*/ = 1) {
    if (!analyzed_) throw std::runtime_error("linsolve.cholesky: factorize before analyze");
    b200::check(ffb_chol_factorize(h_, sys.n, sys.vals.data()));
  }
  bool analyzed() const { return analyzed_; }
  std::vector<double> solve(const std::vector<double>& b) const {
    if (!h_) throw std::runtime_error("linsolve.cholesky: solve before factorize");
    if (static_cast<int>(b.size()) != n_) throw std::runtime_error("linsolve.cholesky: rhs size mismatch");
    std::vector<double> x(n_);
    b200::check(ffb_chol_solve(h_, n_, b.data(), x.data()));
    return x;
  }
  size_t factor_nonzeros() const {
    long long nz = 0;
    if (h_) b200::check(ffb_chol_info(h_, nullptr, &nz));
    return static_cast<size_t>(nz);
  }

 private:
  ffb_chol* h_ = nullptr;
  int n_ = 0;
  bool analyzed_ = false;
};

inline std::vector<double> cg_solve(const SparseSystem& sys, const SolverConfig& cfg,
                                    const std::vector<double>* warm_start = nullptr,
                                    SolveReport* report = nullptr) {
  std::vector<double> x(sys.n);
  SolveReport r;
  const double* w = warm_start && static_cast<int>(warm_start->size()) == sys.n
                        ? warm_start->data() : nullptr;
  const int rc = ffb_csr_cg_solve(b200::ctx(), sys.n, sys.row_ptr.data(), sys.cols.data(),
                                  sys.vals.data(), sys.rhs.data(), cfg.cg_tolerance,
                                  cfg.cg_max_iters, w, x.data(), &r.iterations, &r.residual);
  if (report) *report = r;
  b200::check(rc);
  return x;
}

inline std::vector<double> solve(const SparseSystem& sys, const SolverConfig& cfg,
                                 SolveReport* report = nullptr,
                                 const std::vector<double>* warm_start = nullptr) {
  std::vector<double> x(sys.n);
  SolveReport r;
  const double* w = warm_start && static_cast<int>(warm_start->size()) == sys.n
                        ? warm_start->data() : nullptr;
  const int m = cfg.method == SolveMethod::ConjugateGradient ? FFB_SOLVE_CG : FFB_SOLVE_CHOLESKY;
  const int rc = ffb_csr_solve(b200::ctx(), sys.n, sys.components, sys.row_ptr.data(),
                               sys.cols.data(), sys.vals.data(), sys.rhs.data(), m,
                               cfg.cg_tolerance, cfg.cg_max_iters, w, x.data(), &r.iterations,
                               &r.residual);
  if (report) *report = r;
  b200::check(rc);
  return x;
}

// =================================================================== adapt.hpp
struct IndicatorField {
  std::vector<double> eta;
  double eta_max = 0.0;
};

inline IndicatorField error_indicator(const TriMesh& m, const DataTerms& dt, const RegField& reg,
                                      const FlowState& state, int components = 3) {
  b200::check_reg(m, reg);
  const std::vector<double> t10 = b200::planes(dt), u3 = b200::planes3(state);
  IndicatorField ind;
  ind.eta.resize(m.n_triangles);
  b200::check(ffb_error_indicator(b200::ctx(), m.width, m.height, t10.data(), reg.alpha.data(),
                                  reg.lambda.data(), u3.data(), components, ind.eta.data(),
                                  &ind.eta_max));
  return ind;
}

struct AdaptConfig {
  bool enabled = true;
  double kappa = 10.0;
  double eta_threshold = 0.1;
  double alpha_th = 10.0;
  int n_adapt = 10;
};

inline RegField update_alpha(const RegField& reg, const IndicatorField& ind,
                             const AdaptConfig& cfg) {
  RegField out = reg;
  b200::check(ffb_update_alpha(b200::ctx(), static_cast<int>(reg.alpha.size()), reg.alpha.data(),
                               ind.eta.data(), ind.eta_max, cfg.kappa, cfg.eta_threshold,
                               cfg.alpha_th, out.alpha.data()));
  return out;
}

// =================================================================== schwarz.hpp
struct SplitChoice {
  int parts_x = 1;
  int parts_y = 1;
  double ratio = 0.0;
};

inline std::vector<SplitChoice> enumerate_splits(int width, int height, int n_parts) {
  const int cap = std::max(n_parts, 1);
  std::vector<int> px(cap), py(cap);
  std::vector<double> ratio(cap);
  const int n = ffb_enumerate_splits(width, height, n_parts, px.data(), py.data(), ratio.data(), cap);
  if (n < 0) throw std::runtime_error(ffb_last_error());
  std::vector<SplitChoice> out(n);
  for (int i = 0; i < n; ++i) out[i] = {px[i], py[i], ratio[i]};
  return out;
}

inline SplitChoice choose_split(int width, int height, int n_parts) {
  SplitChoice s;
  b200::check(ffb_choose_split(width, height, n_parts, &s.parts_x, &s.parts_y, &s.ratio));
  return s;
}

struct Rect {
  int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
  int w() const { return x1 - x0; }
  int h() const { return y1 - y0; }
  bool contains(int x, int y) const { return x >= x0 && x < x1 && y >= y0 && y < y1; }
};

struct Subdomain {
  Rect core;
  Rect ext;
  struct Neighbor {
    int part;
    Rect band;
    std::vector<int> gamma;
  };
  std::vector<Neighbor> neighbors;
  std::vector<int> boundary;
};

struct Partition {
  int width = 0, height = 0;
  int parts_x = 1, parts_y = 1;
  int overlap = 0;
  std::vector<Subdomain> parts;
};

namespace b200 {
// Partition <-> the flat format of flowfem_b200.h
inline Partition unflatten(const std::vector<int>& f) {
  Partition P;
  P.width = f[0], P.height = f[1], P.parts_x = f[2], P.parts_y = f[3], P.overlap = f[4];
  const int np = f[5];
  P.parts.resize(np);
  std::vector<int> nb(np), nn(np);
  for (int p = 0; p < np; ++p) {
    const int* h = &f[6 + 10 * p];
    P.parts[p].core = {h[0], h[1], h[2], h[3]};
    P.parts[p].ext = {h[4], h[5], h[6], h[7]};
    nb[p] = h[8], nn[p] = h[9];
  }
  size_t pos = 6 + 10 * static_cast<size_t>(np);
  for (int p = 0; p < np; ++p) {
    P.parts[p].boundary.assign(f.begin() + pos, f.begin() + pos + nb[p]);
    pos += nb[p];
    for (int k = 0; k < nn[p]; ++k) {
      Subdomain::Neighbor n;
      n.part = f[pos];
      n.band = {f[pos + 1], f[pos + 2], f[pos + 3], f[pos + 4]};
      n.gamma.assign(f.begin() + pos + 6, f.begin() + pos + 6 + f[pos + 5]);
      pos += 6 + f[pos + 5];
      P.parts[p].neighbors.push_back(std::move(n));
    }
  }
  return P;
}
inline std::vector<int> flatten(const Partition& P) {
  std::vector<int> f = {P.width, P.height, P.parts_x, P.parts_y, P.overlap,
                        static_cast<int>(P.parts.size())};
  for (const Subdomain& s : P.parts) {
    const int h[10] = {s.core.x0, s.core.y0, s.core.x1, s.core.y1, s.ext.x0, s.ext.y0,
                       s.ext.x1,  s.ext.y1,  static_cast<int>(s.boundary.size()),
                       static_cast<int>(s.neighbors.size())};
    f.insert(f.end(), h, h + 10);
  }
  for (const Subdomain& s : P.parts) {
    f.insert(f.end(), s.boundary.begin(), s.boundary.end());
    for (const auto& n : s.neighbors) {
      const int h[6] = {n.part, n.band.x0, n.band.y0, n.band.x1, n.band.y1,
                        static_cast<int>(n.gamma.size())};
      f.insert(f.end(), h, h + 6);
      f.insert(f.end(), n.gamma.begin(), n.gamma.end());
    }
  }
  return f;
}
}  // namespace b200

inline Partition build_partition(int width, int height, int parts_x, int parts_y, int overlap) {
  const long need = ffb_build_partition(width, height, parts_x, parts_y, overlap, nullptr, 0);
  if (need < 0) throw std::runtime_error(ffb_last_error());
  std::vector<int> f(need);
  ffb_build_partition(width, height, parts_x, parts_y, overlap, f.data(), need);
  return b200::unflatten(f);
}

inline std::vector<int> assign_workers(int n_workers, int n_parts) {
  std::vector<int> a(std::max(n_workers, 1));
  b200::check(ffb_assign_workers(n_workers, n_parts, a.data()));
  a.resize(std::max(n_workers, 0));
  return a;
}

struct SchwarzOptions {
  int n_iters = 10;
  int workers = 1;
  int components = 3;
  AdaptConfig adapt;
  SolverConfig solver;
  bool record_alpha_history = false;
};

struct SchwarzStats {
  std::vector<double> increments;
  std::vector<double> seconds;
  std::vector<double> eta_max;
  std::vector<std::vector<double>> alpha_history;
};

// the reference's synchronous restricted-additive-Schwarz loop (schwarz.cpp:162-319) on the
// device: Cholesky subdomain solves (+ one refinement step) or the reference's CG per
// subdomain, bitwise; reg is updated in place when adapting
inline FlowState schwarz_solve(const TriMesh& m, const DataTerms& dt, RegField& reg,
                               const Partition& part, const SchwarzOptions& opt,
                               SchwarzStats* stats = nullptr) {
  if (part.width != m.width || part.height != m.height)
    throw std::runtime_error("schwarz.schwarz_solve: partition does not match the mesh");
  b200::check_reg(m, reg);
  ffb_ctx* c = b200::ctx();
  const std::vector<double> t10 = b200::planes(dt);
  b200::check(ffb_set_terms(c, m.width, m.height, t10.data()));
  b200::check(ffb_set_reg(c, reg.alpha.data(), reg.lambda.data()));
  const std::vector<int> flat = b200::flatten(part);
  b200::check(ffb_set_partition_flat(c, flat.data(), static_cast<long>(flat.size())));
  ffb_schwarz_options o{};
  o.n_iters = opt.n_iters, o.workers = opt.workers, o.components = opt.components;
  o.adapt = opt.adapt.enabled ? 1 : 0, o.n_adapt = opt.adapt.n_adapt;
  o.kappa = opt.adapt.kappa, o.eta_threshold = opt.adapt.eta_threshold;
  o.alpha_th = opt.adapt.alpha_th;
  o.method = opt.solver.method == SolveMethod::ConjugateGradient ? FFB_SOLVE_CG : FFB_SOLVE_CHOLESKY;
  o.cg_max_iters = opt.solver.cg_max_iters, o.cg_tolerance = opt.solver.cg_tolerance;
  o.record_alpha_history = opt.record_alpha_history ? 1 : 0;
  const int n_it = std::max(opt.n_iters, 0);
  const int n_upd = opt.adapt.enabled ? std::min(std::max(opt.adapt.n_adapt, 0), n_it) : 0;
  std::vector<double> u3(3 * static_cast<size_t>(m.n_vertices)), inc(std::max(n_it, 1)),
      sec(std::max(n_it, 1)), em(std::max(n_upd, 1));
  std::vector<double> hist(opt.record_alpha_history ? static_cast<size_t>(std::max(n_upd, 1)) * m.n_triangles : 0);
  ffb_schwarz_stats st{inc.data(), stats ? sec.data() : nullptr, em.data(),
                       hist.empty() ? nullptr : hist.data(), 0};
  b200::check(ffb_schwarz_run(c, &o, u3.data(), &st));
  if (opt.adapt.enabled) b200::check(ffb_get_reg(c, reg.alpha.data(), nullptr));
  if (stats) {
    stats->increments.insert(stats->increments.end(), inc.begin(), inc.begin() + n_it);
    stats->seconds.insert(stats->seconds.end(), sec.begin(), sec.begin() + n_it);
    stats->eta_max.insert(stats->eta_max.end(), em.begin(), em.begin() + st.n_updates);
    for (int k = 0; k < st.n_updates && !hist.empty(); ++k)
      stats->alpha_history.emplace_back(hist.begin() + static_cast<size_t>(k) * m.n_triangles,
                                        hist.begin() + static_cast<size_t>(k + 1) * m.n_triangles);
  }
  FlowState s = b200::state(m.width, m.height, u3);
  if (opt.components == 2) std::fill(s.mt.begin(), s.mt.end(), 0.0);
  return s;
}

// =================================================================== metrics.hpp
struct FloField {
  int width = 0;
  int height = 0;
  std::vector<float> u, v;
  FloField() = default;
  FloField(int w, int h)
      : width(w), height(h), u(static_cast<size_t>(w) * h, 0.0f), v(static_cast<size_t>(w) * h, 0.0f) {}
};

constexpr float kFloMagic = 202021.25f;
constexpr double kFloValidLimit = 1e9;

inline FloField read_flo(const std::string& path) {
  FloField f;
  b200::check(ffb_read_flo(path.c_str(), &f.width, &f.height, nullptr, nullptr));
  f.u.resize(static_cast<size_t>(f.width) * f.height);
  f.v.resize(f.u.size());
  b200::check(ffb_read_flo(path.c_str(), &f.width, &f.height, f.u.data(), f.v.data()));
  return f;
}

inline void write_flo(const std::string& path, const FloField& f) {
  b200::check(ffb_write_flo(path.c_str(), f.width, f.height, f.u.data(), f.v.data()));
}

inline FloField to_flo(const FlowState& s) {
  FloField f(s.width, s.height);
  for (size_t i = 0; i < f.u.size(); ++i) {
    f.u[i] = static_cast<float>(s.u1[i]);
    f.v[i] = static_cast<float>(s.u2[i]);
  }
  return f;
}

struct FlowMetrics {
  double aae_deg = 0.0;
  double ee = 0.0;
  long valid = 0;
};

inline FlowMetrics compute_metrics(const FlowState& flow, const FloField& truth) {
  if (flow.width != truth.width || flow.height != truth.height)
    throw std::runtime_error("metrics.compute_metrics: flow and ground truth sizes differ");
  FlowMetrics m;
  long long valid = 0;
  b200::check(ffb_compute_metrics(b200::ctx(), truth.width, truth.height, flow.u1.data(),
                                  flow.u2.data(), truth.u.data(), truth.v.data(), &m.aae_deg,
                                  &m.ee, &valid));
  m.valid = static_cast<long>(valid);
  return m;
}

inline RgbImage colorize_flow(const FlowState&, double = 0.0) {
  throw std::runtime_error("metrics.colorize_flow: visualisation is not part of flowfem_b200");
}
inline RgbImage colorize_signed(const std::vector<double>&, int, int) {
  throw std::runtime_error("metrics.colorize_signed: visualisation is not part of flowfem_b200");
}
inline Image rasterize_triangle_field(const TriMesh&, const std::vector<double>&) {
  throw std::runtime_error("metrics.rasterize_triangle_field: visualisation is not part of flowfem_b200");
}

// =================================================================== pipeline.hpp
struct RunConfig {
  std::string frame0, frame1;
  double sigma = 1.0;
  double rho = 2.5;
  double alpha0 = 1000.0;
  double lambda0 = 1000.0;
  bool illumination = true;
  int parts = 4;
  int overlap = 5;
  int schwarz_iters = 10;
  int workers = 4;
  bool adapt = true;
  double kappa = 10.0;
  double eta_threshold = 0.1;
  std::optional<double> alpha_th;
  int adapt_iters = 10;
  std::string solver = "auto";
  double cg_tolerance = 1e-10;
  std::string ground_truth;
  std::string out_flo, out_png, out_metrics, out_increments;
  std::string dump_alpha, dump_mt;
  // flowfem_b200 extension: "schwarz" (default) = the reference's literal Schwarz iteration
  // (schwarz_iters iterations, solver per pick_method); "converged" = the converged-pass
  // protocol, adapt_iters x {Schwarz-PCG solve to cg_tolerance, indicator, alpha update} +
  // a final solve
  std::string protocol = "schwarz";
};

struct RunResult {
  FlowState flow;
  RegField reg;
  SchwarzStats stats;
  std::optional<FlowMetrics> metrics;
  int width = 0, height = 0;
};

inline Image scale_brightness(const Image& img, double gain) {
  Image out = img;
  for (double& v : out.data) v = std::clamp(v * gain, 0.0, 1.0);
  return out;
}

inline RunResult run_on_frames(const Image& f0, const Image& f1, const RunConfig& cfg) {
  if (f0.width != f1.width || f0.height != f1.height)
    throw std::runtime_error("cli.run: frame sizes differ");
  if (f0.width < 2 || f0.height < 2) throw std::runtime_error("cli.run: frames must be at least 2x2");
  if (cfg.solver != "auto" && cfg.solver != "cholesky" && cfg.solver != "cg")
    throw std::runtime_error("cli.solver: unknown solver '" + cfg.solver +
                             "' (want auto, cholesky or cg)");
  const int W = f0.width, H = f0.height, nc = cfg.illumination ? 3 : 2;
  RunResult res;
  res.width = W, res.height = H;
  if (cfg.protocol == "converged") {
    ffb_run_config rc{cfg.sigma, cfg.rho, cfg.alpha0, cfg.lambda0, cfg.illumination ? 1 : 0,
                      cfg.parts, cfg.overlap, cfg.adapt ? 1 : 0, cfg.adapt_iters, cfg.kappa,
                      cfg.eta_threshold,
                      cfg.alpha_th ? *cfg.alpha_th : std::numeric_limits<double>::quiet_NaN(),
                      cfg.cg_tolerance, 0};
    std::vector<double> u3(3 * static_cast<size_t>(W) * H);
    res.reg.alpha.resize(2 * static_cast<size_t>(W - 1) * (H - 1));
    ffb_run_stats st{};
    b200::check(ffb_run_on_frames(b200::ctx(), W, H, f0.data.data(), f1.data.data(), &rc,
                                  u3.data(), res.reg.alpha.data(), &st));
    res.reg.lambda.assign(res.reg.alpha.size(), cfg.lambda0);
    res.flow = b200::state(W, H, u3);
    res.stats.eta_max.assign(st.eta_max, st.eta_max + std::max(st.n_solves - 1, 0));
    return res;
  }
  if (cfg.protocol != "schwarz")
    throw std::runtime_error("cli.run: unknown protocol '" + cfg.protocol +
                             "' (want schwarz or converged)");
  // pipeline.cpp:49-78 with every stage on the device
  std::vector<double> t10(10 * static_cast<size_t>(W) * H);
  b200::check(ffb_frames_to_terms(b200::ctx(), W, H, f0.data.data(), f1.data.data(), cfg.sigma,
                                  cfg.rho, t10.data()));
  const DataTerms dt = b200::terms(W, H, t10);
  const TriMesh mesh = build_pixel_mesh(W, H);
  RegField reg = uniform_reg(mesh, cfg.alpha0, cfg.lambda0);
  const SplitChoice split = choose_split(W, H, cfg.parts);
  const Partition part = build_partition(W, H, split.parts_x, split.parts_y, cfg.overlap);
  SchwarzOptions opt;
  opt.n_iters = cfg.schwarz_iters;
  opt.workers = cfg.workers;
  opt.components = nc;
  opt.adapt.enabled = cfg.adapt;
  opt.adapt.kappa = cfg.kappa;
  opt.adapt.eta_threshold = cfg.eta_threshold;
  opt.adapt.alpha_th = cfg.alpha_th.value_or(cfg.alpha0 / 100.0);
  opt.adapt.n_adapt = cfg.adapt_iters;
  // pick_method (pipeline.cpp:16-28): direct up to 20000 unknowns per extended rectangle
  size_t most = 0;
  for (const Subdomain& p : part.parts) most = std::max(most, static_cast<size_t>(p.ext.w()) * p.ext.h() * nc);
  opt.solver.method = cfg.solver == "cholesky" ? SolveMethod::DirectCholesky
                      : cfg.solver == "cg"     ? SolveMethod::ConjugateGradient
                      : most <= 20000          ? SolveMethod::DirectCholesky
                                               : SolveMethod::ConjugateGradient;
  opt.solver.cg_tolerance = cfg.cg_tolerance;
  res.flow = schwarz_solve(mesh, dt, reg, part, opt, &res.stats);
  res.reg = std::move(reg);
  return res;
}

inline RunResult run_pipeline(const RunConfig& cfg) {
  if (cfg.frame0.empty() || cfg.frame1.empty())
    throw std::runtime_error("cli.run: both frames are required");
  RunResult res = run_on_frames(load_image(cfg.frame0), load_image(cfg.frame1), cfg);
  if (!cfg.ground_truth.empty()) res.metrics = compute_metrics(res.flow, read_flo(cfg.ground_truth));
  if (!cfg.out_flo.empty()) write_flo(cfg.out_flo, to_flo(res.flow));
  if (!cfg.out_png.empty()) save_png_rgb(cfg.out_png, colorize_flow(res.flow));
  if (!cfg.out_increments.empty()) {
    std::ofstream out(cfg.out_increments);
    if (!out) throw std::runtime_error("cli.out_increments: cannot open " + cfg.out_increments);
    out << "iteration,increment,seconds\n";
    for (size_t i = 0; i < res.stats.increments.size(); ++i)
      out << i + 1 << "," << res.stats.increments[i] << ","
          << (i < res.stats.seconds.size() ? res.stats.seconds[i] : 0.0) << "\n";
  }
  if (!cfg.out_metrics.empty()) {
    std::ofstream out(cfg.out_metrics);
    if (!out) throw std::runtime_error("cli.out_metrics: cannot open " + cfg.out_metrics);
    out << "mode,aae_deg,ee,valid_pixels\n";
    if (res.metrics)
      out << (cfg.illumination ? "illum_on" : "illum_off") << "," << res.metrics->aae_deg << ","
          << res.metrics->ee << "," << res.metrics->valid << "\n";
  }
  if (!cfg.dump_alpha.empty() || !cfg.dump_mt.empty())
    throw std::runtime_error("cli.dump: visualisation is not part of flowfem_b200");
  return res;
}

}  // namespace flowfem
