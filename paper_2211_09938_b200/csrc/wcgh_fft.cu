// FFT-convolution synthesis: the same hologram as
// the direct and LUT methods, H = A_eff (*) F with F the single-point fringe
// (fringe_lut.cpp:27-32), evaluated as a circular correlation on an
// L x L = 2Nh x 2Nh grid (L >= Nh + No - 1, so no wrap-around reaches the
// output window). O(L^2 log L) instead of O(P Nh^2): an algorithm-class
// alternative for dense objects. Every kernel is hand-written: the fp64
// fringe grid here, the transforms in wcgh_fftk.cu (shared-memory Stockham
// row FFTs + tiled transposes, spectra kept in the transposed layout, the
// object's zero padding, the spectral product and the band extraction fused
// into the row passes). Per-layer fringe spectra are computed once per job
// (precompute, like the LUTs).
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "wcgh_internal.cuh"

namespace wcgh {
namespace {

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

inline unsigned blocks_for(size_t n) { return unsigned((n + 255) / 256); }

// WCGH_SYNC_DEBUG=1: synchronize after every step and name the failing one.
void dbg(cudaStream_t s, const char* tag) {
  static const bool on = std::getenv("WCGH_SYNC_DEBUG") != nullptr;
  if (!on) return;
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) throw RuntimeError(std::string("fft step '") + tag + "': " + cudaGetErrorString(e));
}

}  // namespace

void fft_prepare(FftPlan& fp, const wcgh_layer* layers, int n_layers, int nh, cudaStream_t s) {
  const int L = 2 * nh;
  const size_t L2 = size_t(L) * L;
  fp.L = L;
  fp.n_layers = n_layers;
  fp.tw.ensure(L, s);
  float2* spec = static_cast<float2*>(fp.fringe_spec.reserve(sizeof(float2) * L2 * n_layers));
  float2* g = static_cast<float2*>(fp.grid.reserve(sizeof(float2) * L2));
  if (n_layers > 1) fp.acc.reserve(sizeof(float2) * L2);
  for (int l = 0; l < n_layers; ++l) {
    k_fringe_grid<<<blocks_for(L2), 256, 0, s>>>(layers[l].wavelength, layers[l].pitch, layers[l].z,
                                                  nh, L, g);
    WCGH_CHECK_LAUNCH();
    dbg(s, "fringe_grid");
    fftk::forward_full(g, L, fp.tw, spec + L2 * l, fp.s1, fp.split, s);
    dbg(s, "fringe_fft");
  }
}

int launch_fft_synthesis(FftPlan& fp, const float* a_eff, int no, int off, int nh, int row0,
                         int rows, float2* out, cudaStream_t s, DirectTiming* timing,
                         const PeerPlanes* peers, const float* a_im) {
  const int L = fp.L;
  const size_t L2 = size_t(L) * L;
  float2* grid = fp.grid.as<float2>();
  int launches = 0;
  if (timing) WCGH_CUDA(cudaEventRecord(timing->begin(), s));
  const size_t nn = size_t(no) * no;
  for (int l = 0; l < fp.n_layers; ++l) {
    launches += fftk::forward_object(a_eff + nn * l, a_im ? a_im + nn * l : nullptr, no, off, L, fp.tw,
                                     grid, fp.s1, fp.s2, fp.split, s);
    dbg(s, "object_fft");
    if (fp.n_layers > 1) {  // sum_l A_l F_l, then one inverse
      k_spec_mul<<<blocks_for(L2), 256, 0, s>>>(grid, fp.fringe_spec.as<float2>() + L2 * l, L2, l > 0,
                                                fp.acc.as<float2>());
      WCGH_CHECK_LAUNCH();
      launches += 1;
    }
  }
  dbg(s, "spec_mul");
  const PeerPlanes pp = peers ? *peers : PeerPlanes{};
  // one layer: the spectral product rides on the inverse's first pass
  const bool one = fp.n_layers == 1;
  launches += fftk::inverse_band(one ? grid : fp.acc.as<float2>(), one ? fp.fringe_spec.as<float2>() : nullptr,
                                 L, nh, row0, rows, fp.tw, out, pp, fp.s1, fp.s2, fp.split, s);
  dbg(s, "inverse_fft");
  if (timing) WCGH_CUDA(cudaEventRecord(timing->end(), s));
  return launches;
}

}  // namespace wcgh

WCGH_CHK_TU(wcgh_fft)
