// Validation-side kernels: angular-spectrum
// propagation / reconstruction and the box-window SSIM, so the
// SSIM >= 0.999 check of a 4096^2 hologram runs on the device instead of a
// CPU fp64 FFT.
//
//   * K6 restates build_kernel / propagate / reconstruct
//     (angular_spectrum.cpp:11-61) and fft_2d (fft.cpp:45-68): fp64
//     throughout like the reference. The 2-D DFTs are the hand-written fp64
//     row FFTs + transposes of wcgh_fftk.cu; the transfer function is evaluated on the fly in
//     the spectral-product kernel (no n^2 kernel array), in the reference's
//     operation order ((2 pi) z_signed) sqrt(s), evanescent samples zeroed;
//     the inverse transform is scaled by 1/n^2 as fft_2d does.
//   * K7 restates ssim (metrics.cpp:49-85): mean over every unit-stride
//     window of the luminance/contrast/structure product. The reference uses
//     summed-area tables; here the five window sums come from a separable
//     two-pass direct summation (row sums, then column sums of row sums) in
//     fp64, and the per-window scores are reduced in a fixed order, so the
//     result is deterministic and differs from the reference only by fp64
//     rounding.
#include <cuda_runtime.h>

#include <string>

#include "wcgh_internal.cuh"

namespace wcgh {
namespace {

constexpr double kPi = 3.14159265358979323846;

__global__ void k_widen(const float2* __restrict__ in, size_t n, double2* __restrict__ out) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_double2(in[i].x, in[i].y);
}

// Transfer sample at DFT index (ix, iy) (angular_spectrum.cpp:17-31).
__device__ __forceinline__ double2 transfer_at(int ix, int iy, int n, double df,
                                               double inv_lambda_sq, double z_signed) {
  const int my = iy < n / 2 ? iy : iy - n;
  const int mx = ix < n / 2 ? ix : ix - n;
  const double fy = my * df, fx = mx * df;
  const double s = inv_lambda_sq - fx * fx - fy * fy;
  if (s >= 0.0) {
    double sn, cs;
    sincos(2.0 * kPi * z_signed * sqrt(s), &sn, &cs);
    return make_double2(cs, sn);
  }
  return make_double2(0.0, 0.0);
}

__global__ void k_transfer(int n, double df, double inv_lambda_sq, double z_signed,
                           double2* __restrict__ out) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size_t(n) * n) return;
  out[i] = transfer_at(int(i % n), int(i / n), n, df, inv_lambda_sq, z_signed);
}

// spectrum *= transfer (propagate, angular_spectrum.cpp:41-43)
__global__ void k_apply_transfer(int n, double df, double inv_lambda_sq, double z_signed,
                                 double2* __restrict__ spec) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size_t(n) * n) return;
  const double2 t = transfer_at(int(i % n), int(i / n), n, df, inv_lambda_sq, z_signed);
  const double2 v = spec[i];
  spec[i] = make_double2(v.x * t.x - v.y * t.y, v.x * t.y + v.y * t.x);
}

__global__ void k_scale(double2* __restrict__ v, size_t n, double scale) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = make_double2(v[i].x * scale, v[i].y * scale);
}

// fft_2d's 1/n^2 inverse scaling then |.| or |.|^2 (angular_spectrum.cpp:54-58)
__global__ void k_magnitude(const double2* __restrict__ v, size_t n, double scale, int intensity,
                            double* __restrict__ out) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double re = v[i].x * scale, im = v[i].y * scale;
  out[i] = intensity ? re * re + im * im : hypot(re, im);
}

// Pass 1: horizontal window sums of a, b, a^2, b^2, ab; out[k][y][x], x < wo.
__global__ void k_ssim_rows(const double* __restrict__ a, const double* __restrict__ b, int w,
                            int h, int win, int wo, double* __restrict__ out) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size_t(h) * wo) return;
  const int x = int(i % wo), y = int(i / wo);
  const double* ra = a + size_t(y) * w + x;
  const double* rb = b + size_t(y) * w + x;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
  for (int k = 0; k < win; ++k) {
    const double va = ra[k], vb = rb[k];
    s0 += va;
    s1 += vb;
    s2 += va * va;
    s3 += vb * vb;
    s4 += va * vb;
  }
  const size_t plane = size_t(h) * wo;
  out[i] = s0;
  out[plane + i] = s1;
  out[2 * plane + i] = s2;
  out[3 * plane + i] = s3;
  out[4 * plane + i] = s4;
}

// Pass 2: vertical sums of the row sums -> per-window score -> per-block sum.
__global__ void k_ssim_cols(const double* __restrict__ rows, int h, int wo, int ho, int win,
                            double inv_n, double c1, double c2, double* __restrict__ partial) {
  __shared__ double s_red[32];
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  double score = 0.0;
  if (i < size_t(ho) * wo) {
    const int x = int(i % wo), y = int(i / wo);
    const size_t plane = size_t(h) * wo;
    double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < win; ++k) {
      const size_t at = size_t(y + k) * wo + x;
#pragma unroll
      for (int q = 0; q < 5; ++q) s[q] += rows[q * plane + at];
    }
    const double mu_a = s[0] * inv_n, mu_b = s[1] * inv_n;
    const double var_a = s[2] * inv_n - mu_a * mu_a;
    const double var_b = s[3] * inv_n - mu_b * mu_b;
    const double cov = s[4] * inv_n - mu_a * mu_b;
    score = ((2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2)) /
            ((mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2));
  }
  for (int o = 16; o > 0; o >>= 1) score += __shfl_down_sync(0xffffffffu, score, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_red[wid] = score;
  __syncthreads();
  if (wid == 0) {
    double v = lane < int(blockDim.x >> 5) ? s_red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) partial[blockIdx.x] = v;
  }
}

// Fixed-order sum of n partials (one CTA).
__global__ void k_sum_fixed(const double* __restrict__ partial, int n, double* __restrict__ out) {
  __shared__ double s_red[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += partial[i];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < int(blockDim.x >> 5) ? s_red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (lane == 0) *out = t;
  }
}

unsigned blocks_for(size_t n, int threads) { return unsigned((n + threads - 1) / threads); }

void ensure_plan(ReconPlan& rp, int n, cudaStream_t s) {
  rp.tw.ensure(n, s);
  rp.n = n;
}

}  // namespace

double2* recon_field(ReconPlan& rp, int n) {
  return static_cast<double2*>(rp.field.reserve(sizeof(double2) * size_t(n) * n));
}

void load_field(ReconPlan& rp, const void* dev_in, bool single, int n, cudaStream_t s) {
  double2* f = recon_field(rp, n);
  const size_t nn = size_t(n) * n;
  if (single) {
    k_widen<<<blocks_for(nn, 256), 256, 0, s>>>(static_cast<const float2*>(dev_in), nn, f);
    WCGH_CHECK_LAUNCH();
  } else if (dev_in != f) {
    WCGH_CUDA(cudaMemcpyAsync(f, dev_in, sizeof(double2) * nn, cudaMemcpyDeviceToDevice, s));
  }
}

int launch_fft2d(ReconPlan& rp, int n, bool inverse, cudaStream_t s) {
  ensure_plan(rp, n, s);
  double2* f = rp.field.as<double2>();
  int launches = fftk::fft2d_f64(f, n, inverse, rp.tw, rp.s1, rp.split, s);
  if (inverse) {
    const size_t nn = size_t(n) * n;
    k_scale<<<blocks_for(nn, 256), 256, 0, s>>>(f, nn, 1.0 / (double(n) * double(n)));
    WCGH_CHECK_LAUNCH();
    ++launches;
  }
  return launches;
}

int launch_transfer(int n, double wavelength, double pitch, double z_signed, double2* out,
                    cudaStream_t s) {
  const size_t nn = size_t(n) * n;
  k_transfer<<<blocks_for(nn, 256), 256, 0, s>>>(n, 1.0 / (double(n) * pitch),
                                                  1.0 / (wavelength * wavelength), z_signed, out);
  WCGH_CHECK_LAUNCH();
  return 1;
}

int launch_propagate(ReconPlan& rp, int n, double wavelength, double pitch, double z_signed,
                     bool scaled, cudaStream_t s) {
  ensure_plan(rp, n, s);
  double2* f = rp.field.as<double2>();
  const size_t nn = size_t(n) * n;
  int launches = fftk::fft2d_f64(f, n, false, rp.tw, rp.s1, rp.split, s);
  k_apply_transfer<<<blocks_for(nn, 256), 256, 0, s>>>(n, 1.0 / (double(n) * pitch),
                                                        1.0 / (wavelength * wavelength), z_signed, f);
  WCGH_CHECK_LAUNCH();
  launches += 1 + fftk::fft2d_f64(f, n, true, rp.tw, rp.s1, rp.split, s);
  if (scaled) {  // fft_2d's 1/n^2 (reconstruct folds it into the magnitude pass)
    k_scale<<<blocks_for(nn, 256), 256, 0, s>>>(f, nn, 1.0 / (double(n) * double(n)));
    WCGH_CHECK_LAUNCH();
    ++launches;
  }
  return launches;
}

int launch_reconstruct(ReconPlan& rp, int n, double wavelength, double pitch, double z,
                       bool intensity, double* out, cudaStream_t s) {
  int launches = launch_propagate(rp, n, wavelength, pitch, -z, false, s);
  const size_t nn = size_t(n) * n;
  k_magnitude<<<blocks_for(nn, 256), 256, 0, s>>>(rp.field.as<double2>(), nn,
                                                   1.0 / (double(n) * double(n)), intensity ? 1 : 0,
                                                   out);
  WCGH_CHECK_LAUNCH();
  return launches + 1;
}

int launch_ssim(const double* a, const double* b, int w, int h, int window, double k1, double k2,
                double dynamic_range, DevBuf& scratch, double* result, cudaStream_t s) {
  const int wo = w - window + 1, ho = h - window + 1;
  const size_t rows_elems = 5 * size_t(h) * wo;
  const size_t outs = size_t(ho) * wo;
  constexpr int kThreads = 256;
  const unsigned nb = blocks_for(outs, kThreads);
  double* buf = static_cast<double*>(scratch.reserve(sizeof(double) * (rows_elems + nb + 1)));
  double* partial = buf + rows_elems;
  k_ssim_rows<<<blocks_for(size_t(h) * wo, kThreads), kThreads, 0, s>>>(a, b, w, h, window, wo, buf);
  WCGH_CHECK_LAUNCH();
  const double c1 = (k1 * dynamic_range) * (k1 * dynamic_range);
  const double c2 = (k2 * dynamic_range) * (k2 * dynamic_range);
  k_ssim_cols<<<nb, kThreads, 0, s>>>(buf, h, wo, ho, window,
                                      1.0 / (double(window) * double(window)), c1, c2, partial);
  WCGH_CHECK_LAUNCH();
  k_sum_fixed<<<1, 1024, 0, s>>>(partial, int(nb), result);
  WCGH_CHECK_LAUNCH();
  return 3;
}

}  // namespace wcgh

WCGH_CHK_TU(wcgh_recon)
