/* TEST INFRASTRUCTURE (oracle) — not product code.
 *
 * Plain-C restatement of the reference hot path; see flowfem_port.h. Each
 * function names the reference file:line it restates (paths relative to
 * /root/reference/proj). The structure is ours: no mesh arrays, CSR or
 * symbolic factorisation — the pixel triangulation is implicit in (x, y) and
 * the operator is applied matrix-free — but every floating-point expression is
 * evaluated in the reference's order so results are bitwise comparable.
 */
#define _POSIX_C_SOURCE 200809L
#include "flowfem_port.h"

#include <math.h>
#include <omp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[512];

static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return -1;
}

/* std::max(a, b) == (a < b) ? b : a — keep the reference's signed-zero behaviour */
#define MAXD(a, b) ((a) < (b) ? (b) : (a))

const char* fp_last_error(void) { return g_err; }

int fp_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
}

/* ------------------------------------------------------------------ imaging */

/* symmetric reflection, imaging.cpp:11-17 */
static inline int fold(int i, int n) {
  while (i < 0 || i >= n) {
    if (i < 0) i = -1 - i;
    if (i >= n) i = 2 * n - 1 - i;
  }
  return i;
}

/* truncated renormalised Gaussian, imaging.cpp:19-29; returns the radius */
int fp_gauss_taps(double sigma, double* taps, int cap) {
  const int r = (int)ceil(3.0 * sigma);
  if (2 * r + 1 > cap) return fail("imaging.gauss_kernel: radius %d too large", r);
  double sum = 0.0;
  for (int k = -r; k <= r; ++k) {
    taps[k + r] = exp(-0.5 * (double)(k * k) / (sigma * sigma));
    sum += taps[k + r];
  }
  for (int k = 0; k < 2 * r + 1; ++k) taps[k] /= sum;
  return r;
}

/* separable smoothing, horizontal then vertical, imaging.cpp:33-63 */
int fp_gaussian_smooth(int W, int H, const double* in, double sigma, double* out) {
  const size_t n = (size_t)W * H;
  if (!(sigma > 0.0)) {
    memcpy(out, in, n * sizeof(double));
    return 0;
  }
  double w[1024];
  const int r = fp_gauss_taps(sigma, w, 1024);
  if (r < 0) return -1;
  double* tmp = (double*)malloc(n * sizeof(double));
  if (!tmp) return fail("imaging.gaussian_smooth: out of memory");
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y) {
    const double* row = in + (size_t)y * W;
    for (int x = 0; x < W; ++x) {
      double s = 0.0;
      for (int k = -r; k <= r; ++k) s += w[k + r] * row[fold(x + k, W)];
      tmp[(size_t)y * W + x] = s;
    }
  }
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y) {
    for (int x = 0; x < W; ++x) {
      double s = 0.0;
      for (int k = -r; k <= r; ++k) s += w[k + r] * tmp[(size_t)fold(y + k, H) * W + x];
      out[(size_t)y * W + x] = s;
    }
  }
  free(tmp);
  return 0;
}

/* frame-average central differences, one-sided at the border, imaging.cpp:65-106 */
int fp_compute_derivatives(int W, int H, const double* f0, const double* f1, double* fx,
                           double* fy, double* ft, double* f) {
  if (W < 2 || H < 2) return fail("imaging.compute_derivatives: frames must be at least 2x2");
#define FAVG(xx, yy) (0.5 * (f0[(size_t)(yy) * W + (xx)] + f1[(size_t)(yy) * W + (xx)]))
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y) {
    for (int x = 0; x < W; ++x) {
      const size_t i = (size_t)y * W + x;
      if (x == 0)
        fx[i] = FAVG(1, y) - FAVG(0, y);
      else if (x == W - 1)
        fx[i] = FAVG(W - 1, y) - FAVG(W - 2, y);
      else
        fx[i] = 0.5 * (FAVG(x + 1, y) - FAVG(x - 1, y));
      if (y == 0)
        fy[i] = FAVG(x, 1) - FAVG(x, 0);
      else if (y == H - 1)
        fy[i] = FAVG(x, H - 1) - FAVG(x, H - 2);
      else
        fy[i] = 0.5 * (FAVG(x, y + 1) - FAVG(x, y - 1));
      ft[i] = f1[i] - f0[i];
      f[i] = f0[i];
    }
  }
#undef FAVG
  return 0;
}

/* ten rho-smoothed products, imaging.cpp:108-138 (signs :126-135) */
int fp_build_data_terms(int W, int H, const double* fx, const double* fy, const double* ft,
                        const double* f, double rho, double* out10) {
  const size_t n = (size_t)W * H;
  double* p = (double*)malloc(n * sizeof(double));
  if (!p) return fail("imaging.build_data_terms: out of memory");
  for (int k = 0; k < 10; ++k) {
#pragma omp parallel for schedule(static)
    for (long i = 0; i < (long)n; ++i) {
      double v;
      switch (k) {
        case 0: v = fx[i] * fx[i]; break;
        case 1: v = fx[i] * fy[i]; break;
        case 2: v = -fx[i] * f[i]; break;
        case 3: v = fy[i] * fy[i]; break;
        case 4: v = -fy[i] * f[i]; break;
        case 5: v = f[i] * f[i]; break;
        case 6: v = -fx[i] * ft[i]; break;
        case 7: v = -fy[i] * ft[i]; break;
        case 8: v = f[i] * ft[i]; break;
        default: v = ft[i] * ft[i]; break;
      }
      p[i] = v;
    }
    if (fp_gaussian_smooth(W, H, p, rho, out10 + k * n)) {
      free(p);
      return -1;
    }
  }
  free(p);
  return 0;
}

/* run_on_frames' imaging prefix, pipeline.cpp:49-52 */
int fp_frames_to_terms(int W, int H, const double* f0, const double* f1, double sigma,
                       double rho, double* out10) {
  const size_t n = (size_t)W * H;
  double* buf = (double*)malloc(6 * n * sizeof(double));
  if (!buf) return fail("imaging: out of memory");
  int rc = fp_gaussian_smooth(W, H, f0, sigma, buf);
  if (!rc) rc = fp_gaussian_smooth(W, H, f1, sigma, buf + n);
  if (!rc) rc = fp_compute_derivatives(W, H, buf, buf + n, buf + 2 * n, buf + 3 * n, buf + 4 * n,
                                       buf + 5 * n);
  if (!rc) rc = fp_build_data_terms(W, H, buf + 2 * n, buf + 3 * n, buf + 4 * n, buf + 5 * n, rho,
                                    out10);
  free(buf);
  return rc;
}

/* ---------------------------------------------------------------- partition */

/* enumerate_splits / choose_split, schwarz.cpp:16-44 */
int fp_choose_split(int W, int H, int n_parts, int* px_out, int* py_out, double* ratio_out) {
  if (n_parts < 1) return fail("schwarz.enumerate_splits: n_parts must be >= 1");
  int bpx = 0, bpy = 0;
  double bratio = 0.0;
  int have = 0;
  for (int px = 1; px <= n_parts; ++px) {
    if (n_parts % px) continue;
    const int py = n_parts / px;
    const double cw = (double)W / px, ch = (double)H / py;
    const double ratio = (cw * ch) / (2.0 * (cw + ch));
    if (!have) {
      bpx = px, bpy = py, bratio = ratio, have = 1;
      continue;
    }
    const double tol = 1e-9 * MAXD(1.0, bratio);
    if (ratio > bratio + tol)
      bpx = px, bpy = py, bratio = ratio;
    else if (fabs(ratio - bratio) <= tol && px >= py && bpx < bpy)
      bpx = px, bpy = py, bratio = ratio;
  }
  *px_out = bpx;
  *py_out = bpy;
  *ratio_out = bratio;
  return 0;
}

typedef struct {
  int x0, y0, x1, y1;
} rect_t;

/* build_partition, schwarz.cpp:54-128, emitted in the flat format of
 * include/flowfem_b200.h */
long fp_build_partition(int W, int H, int px, int py, int ov, int* buf, long cap) {
  if (px < 1 || py < 1) return fail("schwarz.build_partition: part counts must be >= 1");
  const int np = px * py;
  if (ov < 1 && np > 1) return fail("schwarz.build_partition: overlap must be >= 1");
  int* xs = (int*)malloc((px + 1) * sizeof(int));
  int* ys = (int*)malloc((py + 1) * sizeof(int));
  rect_t* core = (rect_t*)malloc(np * sizeof(rect_t));
  rect_t* ext = (rect_t*)malloc(np * sizeof(rect_t));
  for (int i = 0; i <= px; ++i) xs[i] = (int)((long long)i * W / px);
  for (int j = 0; j <= py; ++j) ys[j] = (int)((long long)j * H / py);
  long err = 0;
  for (int j = 0; j < py && !err; ++j)
    for (int i = 0; i < px; ++i) {
      rect_t c = {xs[i], ys[j], xs[i + 1], ys[j + 1]};
      if (np > 1 && (c.x1 - c.x0 <= 2 * ov || c.y1 - c.y0 <= 2 * ov)) {
        err = fail("schwarz.build_partition: core %dx%d not larger than twice the overlap %d",
                   c.x1 - c.x0, c.y1 - c.y0, ov);
        break;
      }
      core[j * px + i] = c;
      rect_t e = {c.x0 - ov < 0 ? 0 : c.x0 - ov, c.y0 - ov < 0 ? 0 : c.y0 - ov,
                  c.x1 + ov > W ? W : c.x1 + ov, c.y1 + ov > H ? H : c.y1 + ov};
      ext[j * px + i] = e;
    }
  if (err) {
    free(xs), free(ys), free(core), free(ext);
    return -1;
  }
  /* pass 1: sizes; pass 2: write */
  long need = 6 + 10L * np;
  long pos_tail = need;
  int* owner_list = NULL;
  int* vert_list = NULL;
  long list_cap = 0;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      if (!buf || cap < need) break;
      buf[0] = W, buf[1] = H, buf[2] = px, buf[3] = py, buf[4] = ov, buf[5] = np;
      pos_tail = 6 + 10L * np;
    }
    for (int p = 0; p < np; ++p) {
      const rect_t e = ext[p];
      /* ring vertices in row-major order, keeping the artificial ones */
      long cnt = 0;
      const long ring = 2L * (e.x1 - e.x0) + 2L * (e.y1 - e.y0);
      if (ring > list_cap) {
        list_cap = ring;
        owner_list = (int*)realloc(owner_list, list_cap * sizeof(int));
        vert_list = (int*)realloc(vert_list, list_cap * sizeof(int));
      }
      for (int y = e.y0; y < e.y1; ++y) {
        const int edge_row = (y == e.y0 || y == e.y1 - 1);
        for (int x = e.x0; x < e.x1; ++x) {
          if (!edge_row && x != e.x0 && x != e.x1 - 1) continue;
          const int art = (x == e.x0 && e.x0 > 0) || (x == e.x1 - 1 && e.x1 < W) ||
                          (y == e.y0 && e.y0 > 0) || (y == e.y1 - 1 && e.y1 < H);
          if (!art) continue;
          int oi = 0, oj = 0;
          while (oi + 1 <= px && xs[oi + 1] <= x) ++oi; /* upper_bound - 1 */
          while (oj + 1 <= py && ys[oj + 1] <= y) ++oj;
          owner_list[cnt] = oj * px + oi;
          vert_list[cnt] = y * W + x;
          ++cnt;
        }
      }
      int n_nb = 0;
      long nb_words = 0;
      for (int q = 0; q < np; ++q) {
        if (q == p) continue;
        long g = 0;
        for (long k = 0; k < cnt; ++k) g += owner_list[k] == q;
        if (!g) continue;
        ++n_nb;
        nb_words += 6 + g;
        if (pass == 1) {
          const rect_t f = ext[q];
          int* o = buf + pos_tail + cnt + (nb_words - 6 - g);
          o[0] = q;
          o[1] = e.x0 > f.x0 ? e.x0 : f.x0;
          o[2] = e.y0 > f.y0 ? e.y0 : f.y0;
          o[3] = e.x1 < f.x1 ? e.x1 : f.x1;
          o[4] = e.y1 < f.y1 ? e.y1 : f.y1;
          o[5] = (int)g;
          long w = 6;
          for (long k = 0; k < cnt; ++k)
            if (owner_list[k] == q) o[w++] = vert_list[k];
        }
      }
      if (pass == 0) {
        need += cnt + nb_words;
      } else {
        int* h = buf + 6 + 10L * p;
        const rect_t c = core[p];
        h[0] = c.x0, h[1] = c.y0, h[2] = c.x1, h[3] = c.y1;
        h[4] = e.x0, h[5] = e.y0, h[6] = e.x1, h[7] = e.y1;
        h[8] = (int)cnt, h[9] = n_nb;
        memcpy(buf + pos_tail, vert_list, cnt * sizeof(int));
        pos_tail += cnt + nb_words;
      }
    }
  }
  free(owner_list), free(vert_list);
  free(xs), free(ys), free(core), free(ext);
  return need;
}

/* ----------------------------------------------------------------- operator */

/* Lumped vertex weight: sum over incident triangles of area/3 (mesh.cpp:122-126).
 * All terms are the same constant, so only their count matters. */
static inline double lumped_weight(int x, int y, int W, int H) {
  int cnt = 0;
  if (x > 0 && y > 0) cnt += 2;         /* cell (x-1,y-1): lower and upper */
  if (x < W - 1 && y > 0) cnt += 1;     /* cell (x,y-1): upper */
  if (x > 0 && y < H - 1) cnt += 1;     /* cell (x-1,y): lower */
  if (x < W - 1 && y < H - 1) cnt += 2; /* cell (x,y): lower and upper */
  double s = 0.0;
  for (int k = 0; k < cnt; ++k) s += 0.5 / 3.0;
  return s;
}

#define TRI_LO(x, y) (2 * ((long)(y) * (W - 1) + (x)))
#define TRI_UP(x, y) (2 * ((long)(y) * (W - 1) + (x)) + 1)

/* Stiffness row of vertex (x,y) for one coefficient field, accumulated over the
 * incident triangles in ascending id as assemble() does (assembly.cpp:114-129).
 * P1 gradients on the half-pixel triangles make the diagonal-edge couplings
 * exactly zero; the h/v couplings are -area*|grad|^2 sums of two triangles. */
typedef struct {
  double diag, left, right, down, up;
} stencil_t;

static inline stencil_t stiffness(const double* coef, int x, int y, int W, int H) {
  stencil_t s = {0.0, 0.0, 0.0, 0.0, 0.0};
  /* ascending triangle ids: cell(x-1,y-1) lo,up; cell(x,y-1) up; cell(x-1,y) lo; cell(x,y) lo,up */
  if (x > 0 && y > 0) {
    const double a = coef[TRI_LO(x - 1, y - 1)], b = coef[TRI_UP(x - 1, y - 1)];
    /* lower (v00,v10,v11): v = v11, |grad|^2 = 1; couples v10 = (x,y-1) by -1 */
    s.diag += a * 0.5;
    s.down += a * -0.5;
    /* upper (v00,v11,v01): v = v11, |grad|^2 = 1; couples v01 = (x-1,y) by -1 */
    s.diag += b * 0.5;
    s.left += b * -0.5;
  }
  if (x < W - 1 && y > 0) {
    const double b = coef[TRI_UP(x, y - 1)];
    /* upper of cell (x,y-1): v = v01, |grad|^2 = 2; couples v00 = (x,y-1), v11 = (x+1,y) */
    s.diag += b * 1.0;
    s.down += b * -0.5;
    s.right += b * -0.5;
  }
  if (x > 0 && y < H - 1) {
    const double a = coef[TRI_LO(x - 1, y)];
    /* lower of cell (x-1,y): v = v10, |grad|^2 = 2; couples v00 = (x-1,y), v11 = (x,y+1) */
    s.diag += a * 1.0;
    s.left += a * -0.5;
    s.up += a * -0.5;
  }
  if (x < W - 1 && y < H - 1) {
    const double a = coef[TRI_LO(x, y)], b = coef[TRI_UP(x, y)];
    /* lower: v = v00, couples v10 = (x+1,y); upper: v = v00, couples v01 = (x,y+1) */
    s.diag += a * 0.5;
    s.right += a * -0.5;
    s.diag += b * 0.5;
    s.up += b * -0.5;
  }
  return s;
}

/* Row-major traversal of one scalar row of the assembled system in the CSR
 * column order of assemble() (ascending vertex ids, the vertex's own nc-block
 * in place of itself), giving bitwise the reference's spmv (assembly.cpp:240-249). */
typedef struct {
  int W, H, nc;
  const double* t10;
  const double* alpha;
  const double* lambda;
} op_t;

static inline double row_apply(const op_t* op, int x, int y, int c, const double* xs,
                               double* diag_out) {
  const int W = op->W, H = op->H, nc = op->nc;
  const size_t n = (size_t)W * H;
  const long v = (long)y * W + x;
  const stencil_t st = stiffness(c < 2 ? op->alpha : op->lambda, x, y, W, H);
  const double wv = lumped_weight(x, y, W, H);
  const double* t = op->t10;
  double A[9] = {0};
  A[0] = t[0 * n + v], A[1] = t[1 * n + v], A[3] = t[1 * n + v], A[4] = t[3 * n + v];
  if (nc == 3) {
    A[2] = t[2 * n + v], A[5] = t[4 * n + v];
    A[6] = t[2 * n + v], A[7] = t[4 * n + v], A[8] = t[5 * n + v];
  }
  double s = 0.0;
  if (y > 0 && x > 0) s += 0.0 * xs[(v - W - 1) * nc + c]; /* diagonal edge: stored zero */
  if (y > 0) s += st.down * xs[(v - W) * nc + c];
  if (x > 0) s += st.left * xs[(v - 1) * nc + c];
  for (int c2 = 0; c2 < nc; ++c2) {
    double val = wv * A[c * 3 + c2];
    if (c2 == c) {
      val += st.diag;
      if (diag_out) *diag_out = val;
    }
    s += val * xs[v * nc + c2];
  }
  if (x < W - 1) s += st.right * xs[(v + 1) * nc + c];
  if (y < H - 1) s += st.up * xs[(v + W) * nc + c];
  if (y < H - 1 && x < W - 1) s += 0.0 * xs[(v + W + 1) * nc + c];
  return s;
}

static void apply_interleaved(const op_t* op, const double* xs, double* ys) {
  const int W = op->W, H = op->H, nc = op->nc;
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x)
      for (int c = 0; c < nc; ++c)
        ys[((size_t)y * W + x) * nc + c] = row_apply(op, x, y, c, xs, NULL);
}

static void rhs_interleaved(const op_t* op, double* b) {
  const int W = op->W, H = op->H, nc = op->nc;
  const size_t n = (size_t)W * H;
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const size_t v = (size_t)y * W + x;
      const double wv = lumped_weight(x, y, W, H);
      for (int c = 0; c < nc; ++c) b[v * nc + c] = wv * op->t10[(6 + c) * n + v];
    }
}

static void planes_to_interleaved(size_t n, int nc, const double* p3, double* xs) {
  for (size_t v = 0; v < n; ++v)
    for (int c = 0; c < nc; ++c) xs[v * nc + c] = p3[c * n + v];
}

static void interleaved_to_planes(size_t n, int nc, const double* xs, double* p3) {
  for (size_t v = 0; v < n; ++v) {
    for (int c = 0; c < nc; ++c) p3[c * n + v] = xs[v * nc + c];
    if (nc == 2) p3[2 * n + v] = 0.0;
  }
}

int fp_assemble_apply(int W, int H, const double* t10, const double* alpha,
                      const double* lambda, int nc, const double* x3, double* y3, double* b3) {
  if (nc != 2 && nc != 3) return fail("assembly.assemble: components must be 2 or 3");
  const size_t n = (size_t)W * H;
  op_t op = {W, H, nc, t10, alpha, lambda};
  double* xs = (double*)malloc(3 * n * nc * sizeof(double));
  if (!xs) return fail("assembly: out of memory");
  double *ys = xs + n * nc, *bs = xs + 2 * n * nc;
  planes_to_interleaved(n, nc, x3, xs);
  apply_interleaved(&op, xs, ys);
  rhs_interleaved(&op, bs);
  interleaved_to_planes(n, nc, ys, y3);
  interleaved_to_planes(n, nc, bs, b3);
  free(xs);
  return 0;
}

/* --------------------------------------------------------------------- CG */

/* fixed-chunk deterministic dot, linsolve.cpp:279-294 */
static double det_dot(const double* a, const double* b, long n) {
  const long chunk = 8192;
  const long nchunks = (n + chunk - 1) / chunk;
  double* partial = (double*)malloc((nchunks ? nchunks : 1) * sizeof(double));
#pragma omp parallel for schedule(static)
  for (long c = 0; c < nchunks; ++c) {
    const long lo = c * chunk, hi = lo + chunk < n ? lo + chunk : n;
    double s = 0.0;
    for (long i = lo; i < hi; ++i) s += a[i] * b[i];
    partial[c] = s;
  }
  double s = 0.0;
  for (long c = 0; c < nchunks; ++c) s += partial[c];
  free(partial);
  return s;
}

/* Jacobi PCG with the reference's stopping rule, linsolve.cpp:298-361 */
static int cg_interleaved(const op_t* op, double tol, int max_iters_cfg, const double* warm,
                          double* x, int* iters_out, double* res_out) {
  const int W = op->W, H = op->H, nc = op->nc;
  const long n = (long)W * H * nc;
  double* diag = (double*)malloc(n * sizeof(double));
  double* b = (double*)malloc(n * sizeof(double));
  double* r = (double*)malloc(n * sizeof(double));
  double* z = (double*)malloc(n * sizeof(double));
  double* p = (double*)malloc(n * sizeof(double));
  double* Ap = (double*)malloc(n * sizeof(double));
  int rc = 0;
  /* diagonal of the assembled matrix (values of a zero vector are never used) */
  memset(Ap, 0, n * sizeof(double));
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int xx = 0; xx < W; ++xx)
      for (int c = 0; c < nc; ++c) {
        double d = 0.0;
        row_apply(op, xx, y, c, Ap, &d);
        diag[((long)y * W + xx) * nc + c] = d;
      }
  for (long i = 0; i < n; ++i)
    if (!(diag[i] > 0.0)) {
      rc = fail("linsolve.cg: non-positive diagonal at row %ld", i);
      goto out;
    }
  rhs_interleaved(op, b);
  {
    const double normb = sqrt(det_dot(b, b, n));
    if (warm)
      memcpy(x, warm, n * sizeof(double));
    else
      memset(x, 0, n * sizeof(double));
    if (normb == 0.0) {
      memset(x, 0, n * sizeof(double));
      if (iters_out) *iters_out = 0;
      if (res_out) *res_out = 0.0;
      goto out;
    }
    apply_interleaved(op, x, Ap);
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) {
      r[i] = b[i] - Ap[i];
      z[i] = r[i] / diag[i];
      p[i] = z[i];
    }
    double rz = det_dot(r, z, n);
    double res = sqrt(det_dot(r, r, n)) / normb;
    const long max_iters = max_iters_cfg > 0 ? max_iters_cfg : 10 * n;
    long it = 0;
    while (res > tol && it < max_iters) {
      ++it;
      apply_interleaved(op, p, Ap);
      const double pAp = det_dot(p, Ap, n);
      if (pAp <= 0.0) {
        rc = fail("linsolve.cg: indefinite matrix detected at iteration %ld", it);
        goto out;
      }
      const double alpha = rz / pAp;
#pragma omp parallel for schedule(static)
      for (long i = 0; i < n; ++i) {
        x[i] += alpha * p[i];
        r[i] -= alpha * Ap[i];
      }
      res = sqrt(det_dot(r, r, n)) / normb;
      if (res <= tol) break;
#pragma omp parallel for schedule(static)
      for (long i = 0; i < n; ++i) z[i] = r[i] / diag[i];
      const double rz_new = det_dot(r, z, n);
      const double beta = rz_new / rz;
      rz = rz_new;
#pragma omp parallel for schedule(static)
      for (long i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
    if (iters_out) *iters_out = (int)it;
    if (res_out) *res_out = res;
    if (res > tol)
      rc = fail("linsolve.cg: no convergence after %ld iterations, relative residual %f", it, res);
  }
out:
  free(diag), free(b), free(r), free(z), free(p), free(Ap);
  return rc;
}

int fp_cg_solve(int W, int H, const double* t10, const double* alpha, const double* lambda,
                int nc, double tol, int max_iters, const double* warm3, double* out3,
                int* iters, double* res) {
  if (nc != 2 && nc != 3) return fail("assembly.assemble: components must be 2 or 3");
  const size_t n = (size_t)W * H;
  op_t op = {W, H, nc, t10, alpha, lambda};
  double* x = (double*)malloc(2 * n * nc * sizeof(double));
  double* warm = NULL;
  if (warm3) {
    warm = x + n * nc;
    planes_to_interleaved(n, nc, warm3, warm);
  }
  const int rc = cg_interleaved(&op, tol, max_iters, warm, x, iters, res);
  if (!rc) interleaved_to_planes(n, nc, x, out3);
  free(x);
  return rc;
}

/* ------------------------------------------------------------- CSR path */

/* y = A x, row-sequential sums in CSR order (spmv, assembly.cpp:240-249) */
int fp_csr_spmv(int n, const int* row_ptr, const int* cols, const double* vals, const double* x,
                double* y) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < n; ++r) {
    double s = 0.0;
    for (int q = row_ptr[r]; q < row_ptr[r + 1]; ++q) s += vals[q] * x[cols[q]];
    y[r] = s;
  }
  return 0;
}

/* Jacobi PCG on an explicit CSR system (cg_solve, linsolve.cpp:298-361): diagonal = last
 * stored entry of column r in row r, det_dot chunks, true-residual stop, warm start */
int fp_csr_cg_solve(int n, const int* row_ptr, const int* cols, const double* vals,
                    const double* b, double tol, int max_iters_cfg, const double* warm,
                    double* x, int* iters_out, double* res_out) {
  double* diag = (double*)malloc((n ? n : 1) * sizeof(double));
  double* r = (double*)malloc((n ? n : 1) * sizeof(double));
  double* z = (double*)malloc((n ? n : 1) * sizeof(double));
  double* p = (double*)malloc((n ? n : 1) * sizeof(double));
  double* Ap = (double*)malloc((n ? n : 1) * sizeof(double));
  int rc = 0;
  for (int i = 0; i < n; ++i) {
    double d = 0.0;
    for (int q = row_ptr[i]; q < row_ptr[i + 1]; ++q)
      if (cols[q] == i) d = vals[q];
    diag[i] = d;
  }
  for (int i = 0; i < n; ++i)
    if (!(diag[i] > 0.0)) {
      rc = fail("linsolve.cg: non-positive diagonal at row %d", i);
      goto out;
    }
  {
    const double normb = sqrt(det_dot(b, b, n));
    if (warm)
      memcpy(x, warm, n * sizeof(double));
    else
      memset(x, 0, n * sizeof(double));
    if (normb == 0.0) {
      memset(x, 0, n * sizeof(double));
      if (iters_out) *iters_out = 0;
      if (res_out) *res_out = 0.0;
      goto out;
    }
    fp_csr_spmv(n, row_ptr, cols, vals, x, Ap);
    for (int i = 0; i < n; ++i) {
      r[i] = b[i] - Ap[i];
      z[i] = r[i] / diag[i];
      p[i] = z[i];
    }
    double rz = det_dot(r, z, n);
    double res = sqrt(det_dot(r, r, n)) / normb;
    const long max_iters = max_iters_cfg > 0 ? max_iters_cfg : 10L * n;
    long it = 0;
    while (res > tol && it < max_iters) {
      ++it;
      fp_csr_spmv(n, row_ptr, cols, vals, p, Ap);
      const double pAp = det_dot(p, Ap, n);
      if (pAp <= 0.0) {
        rc = fail("linsolve.cg: indefinite matrix detected at iteration %ld", it);
        goto out;
      }
      const double alpha = rz / pAp;
      for (int i = 0; i < n; ++i) {
        x[i] += alpha * p[i];
        r[i] -= alpha * Ap[i];
      }
      res = sqrt(det_dot(r, r, n)) / normb;
      if (res <= tol) break;
      for (int i = 0; i < n; ++i) z[i] = r[i] / diag[i];
      const double rz_new = det_dot(r, z, n);
      const double beta = rz_new / rz;
      rz = rz_new;
      for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
    if (iters_out) *iters_out = (int)it;
    if (res_out) *res_out = res;
    if (res > tol)
      rc = fail("linsolve.cg: no convergence after %ld iterations, relative residual %f", it, res);
  }
out:
  free(diag), free(r), free(z), free(p), free(Ap);
  return rc;
}

/* RCM of the free-vertex graph expanded to scalar unknowns (rcm_order, linsolve.cpp:37-83):
 * block adjacency from each vertex's first-component row (:20-33), start = unvisited vertex
 * of minimum degree (smallest id on ties), BFS with neighbours by (degree, id), reversed */
static const int* g_rcm_degree;
static int rcm_cmp(const void* pa, const void* pb) {
  const int a = *(const int*)pa, b = *(const int*)pb;
  if (g_rcm_degree[a] != g_rcm_degree[b]) return g_rcm_degree[a] < g_rcm_degree[b] ? -1 : 1;
  return a < b ? -1 : (a > b ? 1 : 0);
}

int fp_rcm_order(int n, int nc, const int* row_ptr, const int* cols, int* perm) {
  if (nc <= 0 || n % nc != 0) return fail("linsolve.rcm_order: system size not a multiple of components");
  const int nb = n / nc;
  int* adj_ptr = (int*)calloc(nb + 1, sizeof(int));
  int* adj = (int*)malloc(((size_t)row_ptr[n] + 1) * sizeof(int));
  for (int b = 0; b < nb; ++b) {
    const int row = b * nc;
    int last = -1, cnt = 0;
    adj_ptr[b + 1] = adj_ptr[b];
    for (int q = row_ptr[row]; q < row_ptr[row + 1]; ++q) {
      const int k = cols[q] / nc;
      if (k != b && k != last) adj[adj_ptr[b] + cnt++] = k;
      last = k;
    }
    adj_ptr[b + 1] = adj_ptr[b] + cnt;
  }
  int* degree = (int*)malloc((nb ? nb : 1) * sizeof(int));
  for (int b = 0; b < nb; ++b) degree[b] = adj_ptr[b + 1] - adj_ptr[b];
  char* visited = (char*)calloc(nb ? nb : 1, 1);
  int* order = (int*)malloc((nb ? nb : 1) * sizeof(int));
  int* nbrs = (int*)malloc((nb ? nb : 1) * sizeof(int));
  int norder = 0, scanned = 0;
  g_rcm_degree = degree;
  while (norder < nb) {
    int start = -1;
    for (int b = scanned; b < nb; ++b)
      if (!visited[b] && (start < 0 || degree[b] < degree[start])) start = b;
    while (scanned < nb && visited[scanned]) ++scanned;
    visited[start] = 1;
    int head = norder;
    order[norder++] = start;
    while (head < norder) {
      const int v = order[head++];
      int m = 0;
      for (int q = adj_ptr[v]; q < adj_ptr[v + 1]; ++q)
        if (!visited[adj[q]]) nbrs[m++] = adj[q];
      qsort(nbrs, m, sizeof(int), rcm_cmp);
      for (int i = 0; i < m; ++i) {
        visited[nbrs[i]] = 1;
        order[norder++] = nbrs[i];
      }
    }
  }
  for (int i = 0; i < nb; ++i)
    for (int c = 0; c < nc; ++c) perm[i * nc + c] = order[nb - 1 - i] * nc + c;
  free(adj_ptr), free(adj), free(degree), free(visited), free(order), free(nbrs);
  return 0;
}

/* ---------------------------------------------------------------- adapt */

/* constant P1 gradients (p1_gradients, mesh.cpp:172-186) for the two triangle
 * shapes of the pixel mesh, local vertex order of mesh.cpp:30-35 */
static const double GX_LO[3] = {-1.0, 1.0, -0.0}, GY_LO[3] = {0.0, -1.0, 1.0};
static const double GX_UP[3] = {-0.0, 1.0, -1.0}, GY_UP[3] = {-1.0, 0.0, 1.0};

static inline void tri_vertices(int W, long t, long v[3]) {
  const long cell = t >> 1;
  const long x = cell % (W - 1), y = cell / (W - 1);
  const long v00 = y * W + x;
  if ((t & 1) == 0) {
    v[0] = v00, v[1] = v00 + 1, v[2] = v00 + W + 1;
  } else {
    v[0] = v00, v[1] = v00 + W + 1, v[2] = v00 + W;
  }
}

/* error_indicator, adapt.cpp:9-99 */
int fp_error_indicator(int W, int H, const double* t10, const double* alpha,
                       const double* lambda, const double* u3, int nc, double* eta_out,
                       double* eta_max_out) {
  const size_t n = (size_t)W * H;
  const long ntri = 2L * (W - 1) * (H - 1);
  const double* u1 = u3;
  const double* u2 = u3 + n;
  const double* mt = u3 + 2 * n;
  double* grad = (double*)calloc(ntri * 6, sizeof(double));
  double* eta = eta_out ? eta_out : (double*)malloc(ntri * sizeof(double));
  /* per-triangle gradients, adapt.cpp:17-36 */
#pragma omp parallel for schedule(static)
  for (long t = 0; t < ntri; ++t) {
    long v[3];
    tri_vertices(W, t, v);
    const double* gx = (t & 1) ? GX_UP : GX_LO;
    const double* gy = (t & 1) ? GY_UP : GY_LO;
    double* g = grad + t * 6;
    for (int k = 0; k < 3; ++k) {
      const double a = u1[v[k]], b = u2[v[k]];
      g[0] += gx[k] * a;
      g[1] += gy[k] * a;
      g[2] += gx[k] * b;
      g[3] += gy[k] * b;
      if (nc == 3) {
        const double m = mt[v[k]];
        g[4] += gx[k] * m;
        g[5] += gy[k] * m;
      }
    }
  }
  /* edge terms, adapt.cpp:38-64; edge geometry of mesh.cpp:38-104 */
  const long cw = W - 1, ch = H - 1;
  const long nh = cw * H, nv = (long)W * ch, nd = cw * ch;
  double* edge = (double*)malloc((nh + nv + nd) * sizeof(double));
  const double inv_sqrt2 = 1.0 / sqrt(2.0);
#pragma omp parallel for schedule(static)
  for (long e = 0; e < nh + nv + nd; ++e) {
    long t0, t1;
    double nxv, nyv, len;
    if (e < nh) { /* horizontal (x,y)-(x+1,y) */
      const long y = e / cw, x = e % cw;
      const long below = y > 0 ? TRI_UP(x, y - 1) : -1;
      const long above = y < ch ? TRI_LO(x, y) : -1;
      len = 1.0, nxv = 0.0;
      if (below >= 0 && above >= 0) {
        t0 = below < above ? below : above;
        t1 = below < above ? above : below;
        nyv = (t0 == below) ? 1.0 : -1.0;
      } else {
        t0 = below >= 0 ? below : above;
        t1 = -1;
        nyv = below >= 0 ? 1.0 : -1.0;
      }
    } else if (e < nh + nv) { /* vertical (x,y)-(x,y+1) */
      const long k = e - nh, y = k / W, x = k % W;
      const long left = x > 0 ? TRI_LO(x - 1, y) : -1;
      const long right = x < cw ? TRI_UP(x, y) : -1;
      len = 1.0, nyv = 0.0;
      if (left >= 0 && right >= 0) {
        t0 = left < right ? left : right;
        t1 = left < right ? right : left;
        nxv = (t0 == left) ? 1.0 : -1.0;
      } else {
        t0 = left >= 0 ? left : right;
        t1 = -1;
        nxv = left >= 0 ? 1.0 : -1.0;
      }
    } else { /* diagonal of cell (x,y) */
      const long k = e - nh - nv, y = k / cw, x = k % cw;
      t0 = TRI_LO(x, y), t1 = t0 + 1;
      len = sqrt(2.0), nxv = -inv_sqrt2, nyv = inv_sqrt2;
    }
    double sum = 0.0;
    for (int c = 0; c < nc; ++c) {
      const double* coef = c < 2 ? alpha : lambda;
      const double* g0 = grad + t0 * 6 + c * 2;
      const double flux0 = coef[t0] * (g0[0] * nxv + g0[1] * nyv);
      double jump, coef_e;
      if (t1 >= 0) {
        const double* g1 = grad + t1 * 6 + c * 2;
        const double flux1 = coef[t1] * (g1[0] * nxv + g1[1] * nyv);
        jump = flux0 - flux1;
        coef_e = MAXD(coef[t0], coef[t1]);
      } else {
        jump = flux0;
        coef_e = coef[t0];
      }
      sum += jump * jump / coef_e;
    }
    edge[e] = len * sqrt(sum);
  }
  /* element residual + assembly of eta, adapt.cpp:66-98 */
  double eta_max = 0.0;
  const double hK = sqrt(2.0), area = 0.5;
#pragma omp parallel for schedule(static) reduction(max : eta_max)
  for (long t = 0; t < ntri; ++t) {
    long v[3];
    tri_vertices(W, t, v);
    double R[3][3];
    for (int k = 0; k < 3; ++k) {
      const long q = v[k];
      const double U0 = u1[q], U1 = u2[q], U2 = nc == 3 ? mt[q] : 0.0;
      const double a13 = nc == 3 ? t10[2 * n + q] : 0.0;
      const double a23 = nc == 3 ? t10[4 * n + q] : 0.0;
      R[0][k] = t10[6 * n + q] - (t10[0 * n + q] * U0 + t10[1 * n + q] * U1 + a13 * U2);
      R[1][k] = t10[7 * n + q] - (t10[1 * n + q] * U0 + t10[3 * n + q] * U1 + a23 * U2);
      if (nc == 3)
        R[2][k] = t10[8 * n + q] - (t10[2 * n + q] * U0 + t10[4 * n + q] * U1 +
                                    t10[5 * n + q] * U2);
    }
    double elem = 0.0;
    for (int c = 0; c < nc; ++c) {
      const double s = R[c][0] + R[c][1] + R[c][2];
      const double sq = R[c][0] * R[c][0] + R[c][1] * R[c][1] + R[c][2] * R[c][2];
      const double l2 = area / 12.0 * (s * s + sq);
      elem += l2 / (c < 2 ? alpha[t] : lambda[t]);
    }
    double et = hK * sqrt(elem);
    const long cell = t >> 1, x = cell % cw, y = cell / cw;
    long te[3];
    if ((t & 1) == 0) { /* lower: bottom h, right v, diagonal (mesh.cpp:106-120) */
      te[0] = y * cw + x, te[1] = nh + y * W + x + 1, te[2] = nh + nv + y * cw + x;
    } else { /* upper: diagonal, top h, left v */
      te[0] = nh + nv + y * cw + x, te[1] = (y + 1) * cw + x, te[2] = nh + y * W + x;
    }
    for (int k = 0; k < 3; ++k) et += 0.5 * edge[te[k]];
    eta[t] = et;
    eta_max = MAXD(eta_max, et);
  }
  *eta_max_out = eta_max;
  free(grad), free(edge);
  if (!eta_out) free(eta);
  return 0;
}

/* update_alpha, adapt.cpp:101-112 */
int fp_update_alpha(int ntri, const double* alpha, const double* eta, double eta_max,
                    double kappa, double eta_thr, double alpha_th, double* alpha_out) {
  if (eta_max <= 0.0) {
    if (alpha_out != alpha) memcpy(alpha_out, alpha, ntri * sizeof(double));
    return 0;
  }
#pragma omp parallel for schedule(static)
  for (int t = 0; t < ntri; ++t) {
    const double excess = MAXD(eta[t] / eta_max - eta_thr, 0.0);
    alpha_out[t] = MAXD(alpha[t] / (1.0 + kappa * excess), alpha_th);
  }
  return 0;
}

/* ------------------------------------------------------------------ chain */

/* converged-pass protocol, same composition as
 * oracle/ref_capi.cpp:ref_converged_chain */
int fp_converged_chain(int W, int H, const double* f0, const double* f1, double sigma,
                       double rho, double alpha0, double lambda0, int nc, int n_passes,
                       double kappa, double eta_thr, double alpha_th, double tol, double* out3,
                       double* alpha_out, double* eta_max_out, int* iters_out,
                       double* seconds_out) {
  struct timespec ts0, ts1;
  clock_gettime(CLOCK_MONOTONIC, &ts0);
  const size_t n = (size_t)W * H;
  const long ntri = 2L * (W - 1) * (H - 1);
  double* t10 = (double*)malloc(10 * n * sizeof(double));
  double* alpha = (double*)malloc(ntri * sizeof(double));
  double* lambda = (double*)malloc(ntri * sizeof(double));
  double* eta = (double*)malloc(ntri * sizeof(double));
  double* x = (double*)malloc(2 * n * nc * sizeof(double));
  double* warm = x + n * nc;
  int rc = fp_frames_to_terms(W, H, f0, f1, sigma, rho, t10);
  for (long t = 0; t < ntri; ++t) alpha[t] = alpha0, lambda[t] = lambda0;
  op_t op = {W, H, nc, t10, alpha, lambda};
  for (int pass = 0; !rc && pass <= n_passes; ++pass) {
    int it = 0;
    double res = 0.0;
    rc = cg_interleaved(&op, tol, 0, pass ? warm : NULL, x, &it, &res);
    if (rc) break;
    if (iters_out) iters_out[pass] = it;
    memcpy(warm, x, n * nc * sizeof(double));
    interleaved_to_planes(n, nc, x, out3);
    if (pass == n_passes) break;
    double em = 0.0;
    fp_error_indicator(W, H, t10, alpha, lambda, out3, nc, eta, &em);
    if (eta_max_out) eta_max_out[pass] = em;
    fp_update_alpha((int)ntri, alpha, eta, em, kappa, eta_thr, alpha_th, alpha);
  }
  if (!rc && alpha_out) memcpy(alpha_out, alpha, ntri * sizeof(double));
  free(t10), free(alpha), free(lambda), free(eta), free(x);
  clock_gettime(CLOCK_MONOTONIC, &ts1);
  if (seconds_out) *seconds_out = (ts1.tv_sec - ts0.tv_sec) + 1e-9 * (ts1.tv_nsec - ts0.tv_nsec);
  return rc;
}

/* ---------------------------------------------------------------- energy */

/* Discrete energy (assembly.cpp:201-238): 1/2 (sum_t area (alpha |grad u1|^2 + alpha
 * |grad u2|^2 + lambda |grad mt|^2) + sum_v lumped_v (U^T A_v U - 2 F_v^T U + c_v)).
 * Both sums run serially in the reference's order, so the result is bitwise equal. */
int fp_energy(int W, int H, const double* t10, const double* alpha, const double* lambda,
              const double* u3, int nc, double* e_out) {
  if (nc != 2 && nc != 3) return fail("assembly.energy: components must be 2 or 3");
  const size_t n = (size_t)W * H;
  const long ntri = 2L * (W - 1) * (H - 1);
  const double* u1 = u3;
  const double* u2 = u3 + n;
  const double* mt = u3 + 2 * n;
  double e_grad = 0.0;
  for (long t = 0; t < ntri; ++t) {
    long v[3];
    tri_vertices(W, t, v);
    const double* gx = (t & 1) ? GX_UP : GX_LO;
    const double* gy = (t & 1) ? GY_UP : GY_LO;
    double du1x = 0, du1y = 0, du2x = 0, du2y = 0, dmx = 0, dmy = 0;
    for (int k = 0; k < 3; ++k) {
      du1x += gx[k] * u1[v[k]];
      du1y += gy[k] * u1[v[k]];
      du2x += gx[k] * u2[v[k]];
      du2y += gy[k] * u2[v[k]];
      if (nc == 3) {
        dmx += gx[k] * mt[v[k]];
        dmy += gy[k] * mt[v[k]];
      }
    }
    double s = alpha[t] * (du1x * du1x + du1y * du1y + du2x * du2x + du2y * du2y);
    if (nc == 3) s += lambda[t] * (dmx * dmx + dmy * dmy);
    e_grad += 0.5 * s;
  }
  double e_data = 0.0;
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const size_t v = (size_t)y * W + x;
      double A[9] = {0}, F[3] = {0};
      A[0] = t10[0 * n + v], A[1] = t10[1 * n + v], A[3] = t10[1 * n + v], A[4] = t10[3 * n + v];
      F[0] = t10[6 * n + v], F[1] = t10[7 * n + v];
      if (nc == 3) {
        A[2] = t10[2 * n + v], A[5] = t10[4 * n + v];
        A[6] = t10[2 * n + v], A[7] = t10[4 * n + v], A[8] = t10[5 * n + v];
        F[2] = t10[8 * n + v];
      }
      const double U[3] = {u1[v], u2[v], nc == 3 ? mt[v] : 0.0};
      double quad = 0.0, lin = 0.0;
      for (int c = 0; c < nc; ++c) {
        for (int c2 = 0; c2 < nc; ++c2) quad += U[c] * A[c * 3 + c2] * U[c2];
        lin += F[c] * U[c];
      }
      e_data += lumped_weight(x, y, W, H) * (quad - 2.0 * lin + t10[9 * n + v]);
    }
  *e_out = 0.5 * (e_grad + e_data);
  return 0;
}
