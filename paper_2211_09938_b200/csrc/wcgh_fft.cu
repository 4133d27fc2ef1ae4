// FFT-convolution synthesis: the same hologram as
// the direct and LUT methods, H = A_eff (*) F with F the single-point fringe
// (fringe_lut.cpp:27-32), evaluated as a circular correlation on an
// L x L = 2Nh x 2Nh grid (L >= Nh + No - 1, so no wrap-around reaches the
// output window). O(L^2 log L) instead of O(P Nh^2): an algorithm-class
// alternative for dense objects, with cuFFT doing the transforms (library
// code, like cuBLAS) and hand-written kernels for the fp64 fringe grid, the
// scatter, the spectral product and the band extraction. Per-layer fringe
// spectra are computed once per job (precompute, like the LUTs).
#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdlib>
#include <string>

#include "wcgh_internal.cuh"

namespace wcgh {
namespace {

#define WCGH_CUFFT(call)                                                                       \
  do {                                                                                         \
    cufftResult r_ = (call);                                                                   \
    if (r_ != CUFFT_SUCCESS)                                                                   \
      throw RuntimeError(std::string("cuFFT error ") + std::to_string(int(r_)) + " at " +     \
                         __FILE__ + ":" + std::to_string(__LINE__));                           \
  } while (0)

// F at every residue of the L x L grid: offsets d in [-(Nh-1), Nh-1] per axis
// (the residue L/2 = Nh is never reached and stays zero). fp64 evaluation,
// complex64 store — the B = 1 LUT (CGHL payload) laid out circularly.
__global__ void k_fringe_grid(double wavelength, double pitch, double z, int nh, int L,
                              float2* __restrict__ g) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size_t(L) * L) return;
  const int cx = int(i % L), cy = int(i / L);
  const int dx = cx < nh ? cx : cx - L;
  const int dy = cy < nh ? cy : cy - L;
  if (cx == nh || cy == nh) {
    g[i] = make_float2(0.f, 0.f);
    return;
  }
  const double px = double(dx) * pitch, py = double(dy) * pitch;
  const double r = sqrt(px * px + py * py + z * z);
  const double k = 2.0 * 3.14159265358979323846 / wavelength;
  double s, c;
  sincos(k * r, &s, &c);
  g[i] = make_float2(float(c / r), float(s / r));
}

// A_eff (No x No fp32, one layer; a_im: imaginary part or NULL) -> the L x L
// grid at (off+y, off+x).
__global__ void k_scatter(const float* __restrict__ a, const float* __restrict__ a_im, int no,
                          int off, int L, float2* __restrict__ grid) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size_t(no) * no) return;
  const int x = int(i % no), y = int(i / no);
  grid[size_t(off + y) * L + off + x] = make_float2(a[i], a_im ? a_im[i] : 0.f);
}

// acc (+)= fa * ff (complex), elementwise.
__global__ void k_spec_mul(const float2* __restrict__ fa, const float2* __restrict__ ff, size_t n,
                           int accumulate, float2* __restrict__ acc) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float2 a = fa[i], b = ff[i];
  float2 r = make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  if (accumulate) {
    r.x += acc[i].x;
    r.y += acc[i].y;
  }
  acc[i] = r;
}

// out (rows x nh) = grid[row0 + y][x] / L^2.
__global__ void k_extract(const float2* __restrict__ grid, int L, int nh, int row0, int rows,
                          float scale, float2* __restrict__ out, PeerPlanes peers) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size_t(rows) * nh) return;
  const int x = int(i % nh), y = int(i / nh);
  const float2 v = grid[size_t(row0 + y) * L + x];
  const float2 r = make_float2(v.x * scale, v.y * scale);
  out[i] = r;
  store_peers(peers, i, r);  // fused row-tile gather
}

// Two pixels per thread (nh and L even): float4 grid loads, float4 complex64 stores.
__global__ void k_extract2(const float4* __restrict__ grid, int L2h, int nh2, int row0, int rows,
                           float scale, float4* __restrict__ out, PeerPlanes peers) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size_t(rows) * nh2) return;
  const int x = int(i % nh2), y = int(i / nh2);
  const float4 v = grid[size_t(row0 + y) * L2h + x];
  const float4 r = make_float4(v.x * scale, v.y * scale, v.z * scale, v.w * scale);
  out[i] = r;
  store_peers2(peers, 2 * i, r);  // fused row-tile gather
}

inline unsigned blocks_for(size_t n) { return unsigned((n + 255) / 256); }

// WCGH_SYNC_DEBUG=1: synchronize after every step and name the failing one.
void dbg(cudaStream_t s, const char* tag) {
  static const bool on = std::getenv("WCGH_SYNC_DEBUG") != nullptr;
  if (!on) return;
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) throw RuntimeError(std::string("fft step '") + tag + "': " + cudaGetErrorString(e));
}

}  // namespace

FftPlan::~FftPlan() {
  if (plan) cufftDestroy(plan);
}

void fft_prepare(FftPlan& fp, const wcgh_layer* layers, int n_layers, int nh, cudaStream_t s) {
  const int L = 2 * nh;
  const size_t L2 = size_t(L) * L;
  fp.L = L;
  fp.n_layers = n_layers;
  if (!fp.plan) WCGH_CUFFT(cufftPlan2d(&fp.plan, L, L, CUFFT_C2C));
  WCGH_CUFFT(cufftSetStream(fp.plan, s));
  float2* spec = static_cast<float2*>(fp.fringe_spec.reserve(sizeof(float2) * L2 * n_layers));
  fp.grid.reserve(sizeof(float2) * L2);
  fp.acc.reserve(sizeof(float2) * L2);
  for (int l = 0; l < n_layers; ++l) {
    float2* g = spec + L2 * l;
    k_fringe_grid<<<blocks_for(L2), 256, 0, s>>>(layers[l].wavelength, layers[l].pitch, layers[l].z,
                                                  nh, L, g);
    WCGH_CHECK_LAUNCH();
    dbg(s, "fringe_grid");
    WCGH_CUFFT(cufftExecC2C(fp.plan, reinterpret_cast<cufftComplex*>(g),
                            reinterpret_cast<cufftComplex*>(g), CUFFT_FORWARD));
    dbg(s, "fringe_fft");
  }
}

int launch_fft_synthesis(FftPlan& fp, const float* a_eff, int no, int off, int nh, int row0,
                         int rows, float2* out, cudaStream_t s, DirectTiming* timing,
                         const PeerPlanes* peers, const float* a_im) {
  const int L = fp.L;
  const size_t L2 = size_t(L) * L;
  WCGH_CUFFT(cufftSetStream(fp.plan, s));
  float2* grid = fp.grid.as<float2>();
  float2* acc = fp.acc.as<float2>();
  int launches = 0;
  if (timing) WCGH_CUDA(cudaEventRecord(timing->begin(), s));
  for (int l = 0; l < fp.n_layers; ++l) {
    WCGH_CUDA(cudaMemsetAsync(grid, 0, sizeof(float2) * L2, s));
    k_scatter<<<blocks_for(size_t(no) * no), 256, 0, s>>>(
        a_eff + size_t(no) * no * l, a_im ? a_im + size_t(no) * no * l : nullptr, no, off, L, grid);
    WCGH_CHECK_LAUNCH();
    dbg(s, "scatter");
    WCGH_CUFFT(cufftExecC2C(fp.plan, reinterpret_cast<cufftComplex*>(grid),
                            reinterpret_cast<cufftComplex*>(grid), CUFFT_FORWARD));
    dbg(s, "object_fft");
    k_spec_mul<<<blocks_for(L2), 256, 0, s>>>(grid, fp.fringe_spec.as<float2>() + L2 * l, L2, l > 0, acc);
    WCGH_CHECK_LAUNCH();
    launches += 3;
  }
  dbg(s, "spec_mul");
  WCGH_CUFFT(cufftExecC2C(fp.plan, reinterpret_cast<cufftComplex*>(acc),
                          reinterpret_cast<cufftComplex*>(acc), CUFFT_INVERSE));
  dbg(s, "inverse_fft");
  const PeerPlanes pp = peers ? *peers : PeerPlanes{};
  if (nh % 2 == 0 && L % 2 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(acc) % 16 == 0 && peers_aligned16(pp))
    k_extract2<<<blocks_for(size_t(rows) * nh / 2), 256, 0, s>>>(
        reinterpret_cast<const float4*>(acc), L / 2, nh / 2, row0, rows, float(1.0 / double(L2)),
        reinterpret_cast<float4*>(out), pp);
  else
    k_extract<<<blocks_for(size_t(rows) * nh), 256, 0, s>>>(acc, L, nh, row0, rows,
                                                            float(1.0 / double(L2)), out, pp);
  WCGH_CHECK_LAUNCH();
  if (timing) WCGH_CUDA(cudaEventRecord(timing->end(), s));
  return launches + 2;
}

}  // namespace wcgh

WCGH_CHK_TU(wcgh_fft)
