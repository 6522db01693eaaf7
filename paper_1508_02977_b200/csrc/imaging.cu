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

}  // namespace

void smooth_planes(const double* in, double* out, double* tmp, int W, int H, int planes,
                   double sigma, cudaStream_t st) {
  const size_t bytes = static_cast<size_t>(W) * H * planes * sizeof(double);
  if (!(sigma > 0.0)) {  // imaging.cpp:34
    if (out != in) FFB_CUDA(cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, st));
    return;
  }
  const Taps t = make_taps(sigma);
  dim3 grid((W + kRowThreads - 1) / kRowThreads, H, planes);
  k_smooth_h<<<grid, kRowThreads, 0, st>>>(in, tmp, W, H, t);
  FFB_LAUNCHED();
  k_smooth_v<<<grid, kRowThreads, 0, st>>>(tmp, out, W, H, t);
  FFB_LAUNCHED();
}

void deriv_products(const double* s0, const double* s1, double* prod10, int W, int H,
                    cudaStream_t st) {
  dim3 grid((W + kRowThreads - 1) / kRowThreads, H);
  k_deriv_products<<<grid, kRowThreads, 0, st>>>(s0, s1, prod10, W, H);
  FFB_LAUNCHED();
}

void derivatives4(const double* s0, const double* s1, double* fx, double* fy, double* ft,
                  double* f, int W, int H, cudaStream_t st) {
  dim3 grid((W + kRowThreads - 1) / kRowThreads, H);
  k_deriv4<<<grid, kRowThreads, 0, st>>>(s0, s1, fx, fy, ft, f, W, H);
  FFB_LAUNCHED();
}

void products_from4(const double* fx, const double* fy, const double* ft, const double* f,
                    double* prod10, int W, int H, cudaStream_t st) {
  const size_t n = static_cast<size_t>(W) * H;
  k_products4<<<(n + 255) / 256, 256, 0, st>>>(fx, fy, ft, f, prod10, n);
  FFB_LAUNCHED();
}

}  // namespace ffb
