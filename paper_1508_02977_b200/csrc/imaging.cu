// K1/K2: Gaussian pre-smoothing, frame-average derivatives and the ten rho-smoothed
// data-term products (src/imaging.cpp:11-138).
//
// Compiled with --fmad=false and evaluated in the reference's tap order, so every plane is
// bitwise equal to the reference's x86-64 (-O2, no FMA) result. All kernels are
// HBM-bound (taps are re-read from L1); a plane pass moves 16 B/px.
#include "ffb_internal.cuh"

#include <cmath>

namespace ffb {

Taps make_taps(double sigma) {
  // gauss_kernel, imaging.cpp:19-29
  Taps t{};
  const int r = static_cast<int>(std::ceil(3.0 * sigma));
  if (2 * r + 1 > kMaxTaps) fail("imaging.gaussian_smooth: sigma too large for the device taps");
  t.r = r;
  double sum = 0.0;
  for (int k = -r; k <= r; ++k) {
    t.w[k + r] = std::exp(-0.5 * (k * k) / (sigma * sigma));
    sum += t.w[k + r];
  }
  for (int k = 0; k < 2 * r + 1; ++k) t.w[k] /= sum;
  return t;
}

namespace {

// symmetric reflection, imaging.cpp:11-17
__device__ __forceinline__ int fold(int i, int n) {
  while (i < 0 || i >= n) {
    if (i < 0) i = -1 - i;
    if (i >= n) i = 2 * n - 1 - i;
  }
  return i;
}

// horizontal pass (imaging.cpp:40-49); blockIdx.z = plane
__global__ void k_smooth_h(const double* __restrict__ in, double* __restrict__ out, int W,
                           int H, Taps t) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= W) return;
  const size_t plane = static_cast<size_t>(W) * H * blockIdx.z;
  const double* row = in + plane + static_cast<size_t>(y) * W;
  double s = 0.0;
  if (x >= t.r && x + t.r < W) {
    for (int k = -t.r; k <= t.r; ++k) s += t.w[k + t.r] * __ldg(row + x + k);
  } else {
    for (int k = -t.r; k <= t.r; ++k) s += t.w[k + t.r] * __ldg(row + fold(x + k, W));
  }
  out[plane + static_cast<size_t>(y) * W + x] = s;
}

// vertical pass (imaging.cpp:52-61)
__global__ void k_smooth_v(const double* __restrict__ in, double* __restrict__ out, int W,
                           int H, Taps t) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= W) return;
  const size_t plane = static_cast<size_t>(W) * H * blockIdx.z;
  const double* col = in + plane + x;
  double s = 0.0;
  for (int k = -t.r; k <= t.r; ++k)
    s += t.w[k + t.r] * __ldg(col + static_cast<size_t>(fold(y + k, H)) * W);
  out[plane + static_cast<size_t>(y) * W + x] = s;
}

__device__ __forceinline__ double favg(const double* f0, const double* f1, size_t j) {
  return 0.5 * (f0[j] + f1[j]);
}

// compute_derivatives (imaging.cpp:78-103) at one pixel
__device__ __forceinline__ void deriv_at(const double* __restrict__ f0,
                                         const double* __restrict__ f1, int W, int H, int x,
                                         int y, double& fx, double& fy, double& ft, double& f) {
  const size_t i = static_cast<size_t>(y) * W + x;
  const size_t row = static_cast<size_t>(y) * W;
  if (x == 0)
    fx = favg(f0, f1, row + 1) - favg(f0, f1, row + 0);
  else if (x == W - 1)
    fx = favg(f0, f1, row + W - 1) - favg(f0, f1, row + W - 2);
  else
    fx = 0.5 * (favg(f0, f1, row + x + 1) - favg(f0, f1, row + x - 1));
  if (y == 0)
    fy = favg(f0, f1, static_cast<size_t>(1) * W + x) - favg(f0, f1, x);
  else if (y == H - 1)
    fy = favg(f0, f1, static_cast<size_t>(H - 1) * W + x) -
         favg(f0, f1, static_cast<size_t>(H - 2) * W + x);
  else
    fy = 0.5 * (favg(f0, f1, static_cast<size_t>(y + 1) * W + x) -
                favg(f0, f1, static_cast<size_t>(y - 1) * W + x));
  ft = f1[i] - f0[i];
  f = f0[i];
}

// the ten products with the reference's signs (imaging.cpp:126-135)
__device__ __forceinline__ void products(double fx, double fy, double ft, double f, double* p,
                                         size_t i, size_t n) {
  p[0 * n + i] = fx * fx;
  p[1 * n + i] = fx * fy;
  p[2 * n + i] = -fx * f;
  p[3 * n + i] = fy * fy;
  p[4 * n + i] = -fy * f;
  p[5 * n + i] = f * f;
  p[6 * n + i] = -fx * ft;
  p[7 * n + i] = -fy * ft;
  p[8 * n + i] = f * ft;
  p[9 * n + i] = ft * ft;
}

__global__ void k_deriv_products(const double* __restrict__ s0, const double* __restrict__ s1,
                                 double* __restrict__ p, int W, int H) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= W) return;
  double fx, fy, ft, f;
  deriv_at(s0, s1, W, H, x, y, fx, fy, ft, f);
  products(fx, fy, ft, f, p, static_cast<size_t>(y) * W + x, static_cast<size_t>(W) * H);
}

__global__ void k_deriv4(const double* __restrict__ s0, const double* __restrict__ s1,
                         double* fx_o, double* fy_o, double* ft_o, double* f_o, int W, int H) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= W) return;
  double fx, fy, ft, f;
  deriv_at(s0, s1, W, H, x, y, fx, fy, ft, f);
  const size_t i = static_cast<size_t>(y) * W + x;
  fx_o[i] = fx;
  fy_o[i] = fy;
  ft_o[i] = ft;
  f_o[i] = f;
}

__global__ void k_products4(const double* __restrict__ fx, const double* __restrict__ fy,
                            const double* __restrict__ ft, const double* __restrict__ f,
                            double* __restrict__ p, size_t n) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  products(fx[i], fy[i], ft[i], f[i], p, i, n);
}

constexpr int kRowThreads = 128;

// ---- shared-memory tiled kernels (radius <= kTileMaxR; the row kernels above take the rest)
//
// One CTA owns a kTX x kTY output tile. It stages the folded (TX+2R) x (TY+2R) neighbourhood
// once in shared memory with coalesced row loads (16-byte pairs where the row segment is
// inside the image and aligned), runs the horizontal pass over all TY+2R rows into a
// TX-wide buffer and the vertical pass from there, and stores 16-byte output pairs. The
// arithmetic per output is the reference's: the horizontal sum over fold(x+k) of row
// fold(y+k) in tap order, then the vertical sum in tap order — the same operations in the
// same order as the two-pass reference, so results are bitwise equal (--fmad=false).
constexpr int kTX = 32, kTY = 32, kTileThreads = 256, kTileMaxR = 16;

__host__ __device__ constexpr int ext_of(int r) { return kTX + 2 * r; }  // kTX == kTY

// stage the folded (EW x EH) neighbourhood of the tile at (x0, y0) of one plane
__device__ __forceinline__ void stage_ext(const double* __restrict__ in, double* ext, int W,
                                          int H, int x0, int y0, int r) {
  const int E = ext_of(r);
  const int xs = x0 - r;
  // pairs: E is even; a pair is one 16-byte load when both columns are in the image, the
  // row offset is even and W is even (then the address is 16-byte aligned)
  const bool vec = xs >= 0 && xs + E <= W && !(xs & 1) && !(W & 1);
  for (int idx = threadIdx.x; idx < E * (E / 2); idx += kTileThreads) {
    const int j = idx / (E / 2), i = 2 * (idx % (E / 2));
    const double* row = in + static_cast<size_t>(fold(y0 - r + j, H)) * W;
    double2 v;
    if (vec) {
      v = __ldg(reinterpret_cast<const double2*>(row + xs + i));
    } else {
      v.x = __ldg(row + fold(xs + i, W));
      v.y = __ldg(row + fold(xs + i + 1, W));
    }
    *reinterpret_cast<double2*>(ext + j * E + i) = v;
  }
}

// vertical pass of a TX x (TY+2R) horizontal buffer; two outputs per thread, 16-byte stores
__device__ __forceinline__ void vpass_store(const double* htmp, double* __restrict__ out,
                                            int W, int H, int x0, int y0, const Taps& t) {
  const int r = t.r;
  for (int idx = threadIdx.x; idx < kTY * (kTX / 2); idx += kTileThreads) {
    const int j = idx / (kTX / 2), i = 2 * (idx % (kTX / 2));
    const int y = y0 + j, x = x0 + i;
    if (y >= H || x >= W) continue;
    double sx = 0.0, sy = 0.0;
    for (int k = 0; k <= 2 * r; ++k) {
      const double2 h = *reinterpret_cast<const double2*>(htmp + (j + k) * kTX + i);
      sx += t.w[k] * h.x;
      sy += t.w[k] * h.y;
    }
    double* o = out + static_cast<size_t>(y) * W + x;
    if (x + 1 < W) {
      if (!(W & 1)) {
        *reinterpret_cast<double2*>(o) = make_double2(sx, sy);
      } else {
        o[0] = sx;
        o[1] = sy;
      }
    } else {
      o[0] = sx;
    }
  }
}

// gaussian_smooth (imaging.cpp:33-63) of `planes` contiguous planes; blockIdx.z = plane
__global__ void __launch_bounds__(kTileThreads) k_smooth_tile(const double* __restrict__ in,
                                                              double* __restrict__ out, int W,
                                                              int H, Taps t) {
  extern __shared__ __align__(16) double sm[];
  const int r = t.r, E = ext_of(r);
  double* ext = sm;
  double* htmp = sm + E * E;
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  const size_t plane = static_cast<size_t>(W) * H * blockIdx.z;
  stage_ext(in + plane, ext, W, H, x0, y0, r);
  __syncthreads();
  for (int idx = threadIdx.x; idx < E * kTX; idx += kTileThreads) {
    const int j = idx / kTX, i = idx % kTX;
    double s = 0.0;
    for (int k = 0; k <= 2 * r; ++k) s += t.w[k] * ext[j * E + i + k];
    htmp[j * kTX + i] = s;
  }
  __syncthreads();
  vpass_store(htmp, out + plane, W, H, x0, y0, t);
}

// the ten products of imaging.cpp:126-135 (reference signs and operand order)
template <int P>
__device__ __forceinline__ double product(double fx, double fy, double ft, double f) {
  if (P == 0) return fx * fx;
  if (P == 1) return fx * fy;
  if (P == 2) return -fx * f;
  if (P == 3) return fy * fy;
  if (P == 4) return -fy * f;
  if (P == 5) return f * f;
  if (P == 6) return -fx * ft;
  if (P == 7) return -fy * ft;
  if (P == 8) return f * ft;
  return ft * ft;
}

template <int P>
__device__ __forceinline__ void term_plane(const double* D, double* htmp, double* __restrict__ out,
                                           int W, int H, int x0, int y0, const Taps& t) {
  const int r = t.r, E = ext_of(r), EE = E * E;
  for (int idx = threadIdx.x; idx < E * kTX; idx += kTileThreads) {
    const int j = idx / kTX, i = idx % kTX;
    const double* d = D + j * E + i;
    double s = 0.0;
    for (int k = 0; k <= 2 * r; ++k)
      s += t.w[k] * product<P>(d[k], d[EE + k], d[2 * EE + k], d[3 * EE + k]);
    htmp[j * kTX + i] = s;
  }
  __syncthreads();
  vpass_store(htmp, out + static_cast<size_t>(P) * W * H, W, H, x0, y0, t);
}

// build_data_terms (imaging.cpp:108-138) fused with compute_derivatives (imaging.cpp:78-103):
// the four derivative planes of the folded neighbourhood are staged once (from the smoothed
// frames, or from given derivative planes), then each of the ten products is formed on the
// fly inside the horizontal pass, smoothed and stored. The two horizontal buffers alternate
// so one barrier per plane suffices. 16 B/px in, 80 B/px out (vs 480 B/px for the separate
// product + row/column passes).
template <bool kFrom4>
__global__ void __launch_bounds__(kTileThreads)
    k_terms_tile(const double* __restrict__ a, const double* __restrict__ b,
                 const double* __restrict__ c, const double* __restrict__ d4,
                 double* __restrict__ out10, int W, int H, Taps t) {
  extern __shared__ __align__(16) double sm[];
  const int r = t.r, E = ext_of(r), EE = E * E;
  double* D = sm;                 // fx, fy, ft, f over the neighbourhood
  double* h0 = sm + 4 * EE;       // two horizontal buffers (E rows x kTX)
  double* h1 = h0 + E * kTX;
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  for (int idx = threadIdx.x; idx < EE; idx += kTileThreads) {
    const int j = idx / E, i = idx % E;
    const int gx = fold(x0 - r + i, W), gy = fold(y0 - r + j, H);
    double fx, fy, ft, f;
    if (kFrom4) {
      const size_t g = static_cast<size_t>(gy) * W + gx;
      fx = __ldg(a + g);
      fy = __ldg(b + g);
      ft = __ldg(c + g);
      f = __ldg(d4 + g);
    } else {
      deriv_at(a, b, W, H, gx, gy, fx, fy, ft, f);
    }
    D[idx] = fx;
    D[EE + idx] = fy;
    D[2 * EE + idx] = ft;
    D[3 * EE + idx] = f;
  }
  __syncthreads();
  term_plane<0>(D, h0, out10, W, H, x0, y0, t);
  // a buffer is rewritten two planes later: every thread has passed the barrier in between,
  // so its vertical pass over that buffer is done
  term_plane<1>(D, h1, out10, W, H, x0, y0, t);
  term_plane<2>(D, h0, out10, W, H, x0, y0, t);
  term_plane<3>(D, h1, out10, W, H, x0, y0, t);
  term_plane<4>(D, h0, out10, W, H, x0, y0, t);
  term_plane<5>(D, h1, out10, W, H, x0, y0, t);
  term_plane<6>(D, h0, out10, W, H, x0, y0, t);
  term_plane<7>(D, h1, out10, W, H, x0, y0, t);
  term_plane<8>(D, h0, out10, W, H, x0, y0, t);
  term_plane<9>(D, h1, out10, W, H, x0, y0, t);
}

size_t smooth_smem(int r) { return sizeof(double) * (ext_of(r) * ext_of(r) + ext_of(r) * kTX); }
size_t terms_smem(int r) {
  return sizeof(double) * (4 * ext_of(r) * ext_of(r) + 2 * ext_of(r) * kTX);
}

template <class K>
void allow_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    FFB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
}

dim3 tile_grid(int W, int H, int planes) {
  return dim3((W + kTX - 1) / kTX, (H + kTY - 1) / kTY, planes);
}

}  // namespace

void smooth_planes(const double* in, double* out, double* tmp, int W, int H, int planes,
                   double sigma, cudaStream_t st) {
  const size_t bytes = static_cast<size_t>(W) * H * planes * sizeof(double);
  if (!(sigma > 0.0)) {  // imaging.cpp:34
    if (out != in) FFB_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, st));
    return;
  }
  const Taps t = make_taps(sigma);
  if (t.r <= kTileMaxR) {
    const size_t sm = smooth_smem(t.r);
    allow_smem(k_smooth_tile, sm);
    k_smooth_tile<<<tile_grid(W, H, planes), kTileThreads, sm, st>>>(in, out, W, H, t);
    FFB_LAUNCHED();
    return;
  }
  dim3 grid((W + kRowThreads - 1) / kRowThreads, H, planes);
  k_smooth_h<<<grid, kRowThreads, 0, st>>>(in, tmp, W, H, t);
  FFB_LAUNCHED();
  k_smooth_v<<<grid, kRowThreads, 0, st>>>(tmp, out, W, H, t);
  FFB_LAUNCHED();
}

void data_terms(const double* s0, const double* s1, double* t10, double* prod, double* tmp,
                int W, int H, double rho, cudaStream_t st) {
  const Taps t = make_taps(rho > 0.0 ? rho : 1.0);
  if (rho > 0.0 && t.r <= kTileMaxR) {
    const size_t sm = terms_smem(t.r);
    allow_smem(k_terms_tile<false>, sm);
    k_terms_tile<false><<<tile_grid(W, H, 1), kTileThreads, sm, st>>>(s0, s1, nullptr, nullptr,
                                                                     t10, W, H, t);
    FFB_LAUNCHED();
    return;
  }
  // rho <= 0 (the products unsmoothed, imaging.cpp:34) or a radius beyond the tile
  dim3 grid((W + kRowThreads - 1) / kRowThreads, H);
  if (!(rho > 0.0)) prod = t10;
  k_deriv_products<<<grid, kRowThreads, 0, st>>>(s0, s1, prod, W, H);
  FFB_LAUNCHED();
  if (rho > 0.0) smooth_planes(prod, t10, tmp, W, H, 10, rho, st);
}

void derivatives4(const double* s0, const double* s1, double* fx, double* fy, double* ft,
                  double* f, int W, int H, cudaStream_t st) {
  dim3 grid((W + kRowThreads - 1) / kRowThreads, H);
  k_deriv4<<<grid, kRowThreads, 0, st>>>(s0, s1, fx, fy, ft, f, W, H);
  FFB_LAUNCHED();
}

void data_terms_from4(const double* fx, const double* fy, const double* ft, const double* f,
                      double* t10, double* prod, double* tmp, int W, int H, double rho,
                      cudaStream_t st) {
  const Taps t = make_taps(rho > 0.0 ? rho : 1.0);
  if (rho > 0.0 && t.r <= kTileMaxR) {
    const size_t sm = terms_smem(t.r);
    allow_smem(k_terms_tile<true>, sm);
    k_terms_tile<true><<<tile_grid(W, H, 1), kTileThreads, sm, st>>>(fx, fy, ft, f, t10, W, H, t);
    FFB_LAUNCHED();
    return;
  }
  const size_t n = static_cast<size_t>(W) * H;
  if (!(rho > 0.0)) prod = t10;
  k_products4<<<(n + 255) / 256, 256, 0, st>>>(fx, fy, ft, f, prod, n);
  FFB_LAUNCHED();
  if (rho > 0.0) smooth_planes(prod, t10, tmp, W, H, 10, rho, st);
}

}  // namespace ffb
