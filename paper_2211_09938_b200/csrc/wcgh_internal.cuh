// Internal declarations shared by the wcgh CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/wcgh.h"

namespace wcgh {

// Error types mirroring the reference's ValidationError / IoError
// (errors.hpp:10-20); mapped to WCGH_EVALIDATION / WCGH_ERUNTIME at the ABI.
struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define WCGH_CUDA(call)                                                                     \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      throw ::wcgh::RuntimeError(std::string("CUDA error ") + cudaGetErrorString(e_) +     \
                                 " at " + __FILE__ + ":" + std::to_string(__LINE__));       \
  } while (0)

#define WCGH_CHECK_LAUNCH() WCGH_CUDA(cudaGetLastError())

inline void require(bool ok, const std::string& what) {
  if (!ok) throw ValidationError(what);
}

// Tuning / test overrides from the environment: unset or empty = default.
inline int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}

// ---- checked build (-DWCGH_CHECKED, libwcgh_checked.so; test use only) -------
// compute-sanitizer is not available on the GPU pool, so a separate build of
// the same sources carries its own checks: WCGH_DCHECK(cond) in the kernels
// records the first failing source line in a per-translation-unit device
// flag (the kernel continues; the offending access is still performed only
// where it is provably inside an allocation); every C-ABI call collects the
// flags after its work (abi::guard) and turns a hit into WCGH_ERUNTIME
// "checked build: ...". Scratch allocations are poisoned with 0xFF bytes
// (NaN floats, -1 ints), so a read of memory no kernel wrote shows up in
// the results. The product library (libwcgh.so) compiles none of this.
#ifdef WCGH_CHECKED
namespace chk {
static __device__ unsigned int d_fail;
static __device__ unsigned int d_line;
__device__ __forceinline__ void fail(unsigned line) {
  if (atomicCAS(&d_fail, 0u, 1u) == 0u) d_line = line;
}
// reads and clears this translation unit's flag; throws on a hit
inline void collect_tu(const char* tu) {
  cudaDeviceSynchronize();  // the ABI's streams are non-blocking; the flag is read on the legacy stream
  unsigned f = 0, l = 0;
  const cudaError_t e = cudaMemcpyFromSymbol(&f, d_fail, sizeof(f));
  if (e != cudaSuccess)
    throw RuntimeError(std::string("checked build: cannot read the check flag of ") + tu + ": " +
                       cudaGetErrorString(e));
  if (!f) return;
  cudaMemcpyFromSymbol(&l, d_line, sizeof(l));
  const unsigned zero = 0;
  cudaMemcpyToSymbol(d_fail, &zero, sizeof(zero));
  throw RuntimeError(std::string("checked build: device bounds check failed at ") + tu + ":" +
                     std::to_string(l));
}
void collect_all();  // every translation unit (wcgh_abi.cu)
}  // namespace chk
#define WCGH_DCHECK(cond)                                   \
  do {                                                      \
    if (!(cond)) ::wcgh::chk::fail(unsigned(__LINE__));     \
  } while (0)
#define WCGH_CHK_TU(NAME) \
  namespace wcgh { namespace chk { void collect_##NAME() { collect_tu(#NAME ".cu"); } } }
#else
#define WCGH_DCHECK(cond) \
  do {                    \
  } while (0)
#define WCGH_CHK_TU(NAME)
#endif

// RAII device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  // Grows to at least n bytes (contents not preserved).
  void* reserve(size_t n) {
    if (n <= bytes && p) return p;
    release();
    if (n == 0) n = 16;
    WCGH_CUDA(cudaMalloc(&p, n));
    bytes = n;
#ifdef WCGH_CHECKED
    // poison: reads of unwritten scratch show up as NaN / -1. The legacy
    // stream does not order against the ABI's non-blocking streams: finish
    // the fill before any stream work can touch the buffer.
    WCGH_CUDA(cudaMemset(p, 0xFF, n));
    WCGH_CUDA(cudaDeviceSynchronize());
#endif
    return p;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// ---- fused row-tile gather -------------------------------------------------
// Full-plane buffers of every rank (device pointers valid in this process,
// e.g. CUDA-IPC-mapped over NVLink): the kernel that produces a band's final
// values also stores each value into every listed plane at its global
// position (offset = row0 * Nh elements), so the all-gather rides on the
// epilogue's stores instead of a separate collective.
constexpr int kMaxPeers = 16;
struct PeerPlanes {
  float2* p[kMaxPeers];
  int n = 0;
  size_t offset = 0;
  size_t limit = 0;  // elements in each full plane (plane_size^2)
};
__device__ __forceinline__ void store_peers(const PeerPlanes& pp, size_t i, float2 v) {
  if (pp.n) WCGH_DCHECK(pp.offset + i < pp.limit);
  for (int k = 0; k < pp.n; ++k) pp.p[k][pp.offset + i] = v;
}
// two adjacent pixels (i even, offset even, peer planes 16-byte aligned) as one float4
__device__ __forceinline__ void store_peers2(const PeerPlanes& pp, size_t i, float4 v) {
  if (pp.n) WCGH_DCHECK(pp.offset + i + 1 < pp.limit);
  for (int k = 0; k < pp.n; ++k) *reinterpret_cast<float4*>(pp.p[k] + pp.offset + i) = v;
}
inline bool peers_aligned16(const PeerPlanes& pp) {
  if (pp.offset % 2) return false;
  for (int k = 0; k < pp.n; ++k)
    if (reinterpret_cast<uintptr_t>(pp.p[k]) % 16) return false;
  return true;
}

// Chunks of fixed-order partial sums per launch group (direct K3 and LUT K4).
// Each group's reduction rounds the running plane to fp32, so the group
// boundaries are part of the summation order: they are sized from the FULL
// plane (nh^2), never from the row band, so every band — any GPU count —
// adds its chunks in the same groups and the gathered plane is bitwise the
// single-GPU plane. Budget: 2 GiB of fp32 complex partial planes, or
// WCGH_PARTIAL_BYTES (tests force several groups with a small value).
int partial_group(int n_chunks, int nh);

// copy a finished band into the peer planes (used where no fused epilogue exists)
int launch_band_to_peers(const float2* band_dev, size_t count, const PeerPlanes& peers,
                         cudaStream_t stream);

// ---- direct accumulation (K3) ---------------------------------------------

constexpr int kMaxLayers = 16;
constexpr int kMaxCorr = 8;  // phase-correction series terms b_2 .. b_9

// Per-layer constants of the fixed-point phase evaluation. Total phase in
// cycles: z/lambda * sqrt(1 + u), u = s p^2/z^2, s = dx^2 + dy^2, split as
//   frac(z/lambda)  +  s * alpha  +  (z/lambda) * g(u),
//   alpha = p^2 / (2 lambda z),  g(u) = sqrt(1+u) - 1 - u/2 = sum_{n>=2} C(1/2,n) u^n.
// The first two are exact 32-/64-bit fixed point; g is an fp32 series.
struct DirectLayer {
  uint32_t a_hi, a_lo;   // frac(alpha) in 0.64 fixed point
  uint32_t phi0;         // frac(z/lambda) in 0.32 fixed point
  uint32_t dd;           // frac(2*32^2*alpha): second difference along a thread's pixels
  float c;               // p^2 / z^2
  float inv_z;           // 1/z
  float corr[kMaxCorr];  // 2*pi*(z/lambda)*C(1/2, n+2): radians per u^(n+2)
  float amp[4];          // C(-1/2, n+1): (1+u)^(-1/2) = 1 + sum amp[n] u^(n+1)
  // recurrence form (k_direct_rec): derivatives of the correction series,
  // d/du: sum dcorr[n] u^(n+1), d2/du2: sum ddcorr[n] u^n (radians), and the
  // quadratic phase's second difference between adjacent pixels, 2 alpha
  // cycles, centred and in radians.
  float dcorr[kMaxCorr], ddcorr[kMaxCorr];
  float dq, dq3, sr0;     // dq, dq - dq^3/6, -c + dq (dq - dq^3/6) - dq^2/2
  uint32_t t_ab, d_ab;    // frac(240 alpha), frac(32 alpha): run B from run A (L = 16)
  uint32_t t_abq;         // frac(256 alpha): the same for the chirp-factored form
  double wavelength, pitch, z, k;  // fp64 phase mode
};

struct DirectPlan {
  int n_corr;      // phase-series terms used (2, 3, 5 or 8)
  int amp_degree;  // (1+u)^(-1/2): polynomial degree 1, 2 or 3, or 0 = MUFU.RSQ
  double u_max;
  int rec;         // 0 per-pixel (k_direct_fixed); angle-addition recurrence along
                   // 16-pixel runs: 1 k_direct_rec, 2 chirp-factored k_direct_chirp
  int hold = 1;    // k_direct_chirp: steps the run multiplier is held for (1, 2 or 4)
};

// CUDA-event pairs around each launch of a kernel family (for per-kernel
// device time inside a run); events are created lazily and reused.
struct DirectTiming {
  std::vector<cudaEvent_t> ev;
  size_t used = 0;
  int extra = 0;  // launches inside timed intervals beyond one each (K4 chunk launches)
  int form = -1, hold = 0;  // launch_direct's choice for the last run (DirectPlan::rec, ::hold)
  cudaEvent_t next() {
    if (used == ev.size()) {
      cudaEvent_t e;
      WCGH_CUDA(cudaEventCreate(&e));
      ev.push_back(e);
    }
    return ev[used++];
  }
  cudaEvent_t begin() { return next(); }
  cudaEvent_t end() { return next(); }
  void reset() { used = 0; extra = 0; }
  // Sum of the pair durations (call after the stream has synchronized).
  float elapsed_ms() const {
    float total = 0.f;
    for (size_t i = 0; i + 1 < used; i += 2) {
      float ms = 0.f;
      WCGH_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      total += ms;
    }
    return total;
  }
  int launches() const { return int(used / 2) + extra; }
  ~DirectTiming() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

// Chooses the series length and amplitude evaluation for a maximal u;
// throws ValidationError when the fixed-point mode cannot reach 1e-7 rad.
DirectPlan plan_direct(const wcgh_layer* layers, int n_layers, double max_dx, double max_dy);
DirectLayer make_direct_layer(const wcgh_layer& L);

// Launches K3 (and the chunk reductions) on `stream`. pts: device, sorted by
// layer; layer_begin: host array (n_layers + 1). out: device rows x nh
// complex64. Returns the number of kernel launches; if `timing` is given,
// brackets every K3 launch with an event pair. pim (device, optional): the
// points' imaginary amplitudes (complex objects; pts[i].a is the real part).
struct DirectScratch {
  DevBuf partial;
  DevBuf polar;  // complex amplitudes as (x, y, |a|, phase) records
};
int launch_direct(const wcgh_point* pts_dev, const int64_t* layer_begin_host, int n_layers,
                  const wcgh_layer* layers, int nh, int row0, int rows, int phase_mode,
                  double max_dx, double max_dy, float2* out_dev, DirectScratch& scratch,
                  cudaStream_t stream, DirectTiming* timing, double* updates_out,
                  const PeerPlanes* peers = nullptr, const float* pim = nullptr);

// ---- analysis (K1 + K2) ----------------------------------------------------

constexpr int kOpReplicas = 256;
struct AnalysisOut {
  // device outputs (nullptr = not requested), per layer strided by n^2-type sizes
  double* pyramid = nullptr;  // layer stride: pyr_len(n)
  double* sal_pyr = nullptr;  // layer stride: (n/2)^2 + (n/4)^2 + (n/8)^2
  uint8_t* masks = nullptr;   // layer stride: (n/4)^2 + (n/2)^2 + n^2
  float* a_eff = nullptr;     // layer stride n^2 (required)
  float* w_stage = nullptr;   // LUT weights: base (n/8)^2, ll (n/4)^2, l (n/2)^2, full n^2
  int* seg_counts = nullptr;  // nonzero A_eff per (layer, row, 128-px segment)
  unsigned long long* ops = nullptr;  // per layer 5 counters (device)
  // optional: kOpReplicas x layers x 5 zeroed partial counters. The uint8 K1
  // spreads its per-warp counts over them (same-address atomics from every
  // warp serialised in L2: 25% of the front end at 16384^2) and a fold
  // kernel adds them into `ops` and re-zeroes them.
  unsigned long long* ops_rep = nullptr;
  int* err = nullptr;                 // validation flags (device)
};

__host__ __device__ inline size_t pyr_len(int n) {
  const size_t n2 = size_t(n) * n;
  return n2 / 64 + 3 * (n2 / 4 + n2 / 16 + n2 / 64);
}
__host__ __device__ inline size_t salpyr_len(int n) {
  const size_t n2 = size_t(n) * n;
  return n2 / 4 + n2 / 16 + n2 / 64;
}
__host__ __device__ inline size_t masks_len(int n) {
  const size_t n2 = size_t(n) * n;
  return n2 / 16 + n2 / 4 + n2;
}
__host__ __device__ inline size_t wstage_len(int n) {
  const size_t n2 = size_t(n) * n;
  return n2 / 64 + n2 / 16 + n2 / 4 + n2;
}
__host__ __device__ inline int seg_per_row(int n) { return (n + 127) / 128; }

// Error flag bits written by the analysis kernel.
enum : int { kErrObjectNonFinite = 1, kErrSaliencyRange = 2 };

// WCGH_C128: analyses one part of the complex object; `obj` points at the
// first real part (or, 8 bytes on, the first imaginary part).
int launch_analysis(const void* obj, int obj_dtype, double obj_scale, const void* sal,
                    int sal_dtype, int n, int n_layers, const wcgh_plan& plan,
                    const AnalysisOut& out, cudaStream_t stream);
// Exclusive scan of `count` ints into `offsets` (count + 1 entries, last = total).
// Exclusive scan, offsets[count] = total. With `scratch`, long arrays use a
// multi-CTA scan (3 launches); otherwise one CTA.
int launch_scan(const int* counts, int* offsets, int count, cudaStream_t stream,
                DevBuf* scratch = nullptr);
// Ordered compaction of nonzero A_eff into points (hologram coordinates).
// With a_im (complex objects): kept where either part is nonzero, imaginary
// parts written to p_im in point order.
int launch_compact_points(const float* a_eff, const int* offsets, int n, int n_layers,
                          int offset, int layer0, wcgh_point* points, cudaStream_t stream,
                          const float* a_im = nullptr, float* p_im = nullptr);
// Ordered compaction of nonzero mask bytes into cell indices y*m+x.
int launch_mask_counts(const uint8_t* mask, int m, int* seg_counts, cudaStream_t stream);
// Stage s's amplitude contribution image (snapshots of the direct/FFT methods).
int launch_stage_delta(const float* w_stage, int n, int n_layers, int stage, float* out,
                       cudaStream_t stream);
int launch_seg_counts_f32(const float* img, int n, int n_layers, int* counts, cudaStream_t stream,
                          const float* img_im = nullptr);
int launch_compact_mask(const uint8_t* mask, int m, const int* offsets, uint32_t* cells,
                        cudaStream_t stream);

// Generic L-level Haar analysis (levels != 3); scratch holds 2 n^2 doubles.
int launch_haar_levels(const void* image, int dtype, double scale, int n, int levels,
                       double* pyramid, double* scratch, int* err, cudaStream_t stream);
// refine(): residual expansion + strict gate into dense weights (2m x 2m).
int launch_refine_gate(const double* h, const double* v, const double* d, int m,
                       const double* sal, double t, float* w, uint8_t* mask,
                       unsigned long long* count, cudaStream_t stream);
// Residual expansion of host-provided bands (wcgh_expand_residual).
int launch_expand_residual(const double* h, const double* v, const double* d, int m, double* out,
                           cudaStream_t stream);

// ---- LUT path (K4 + K5) ------------------------------------------------------

// ---- FFT-convolution method ---------------------------------------------------

// Hand-written FFTs (wcgh_fftk.cu): twiddle tables e^{-2 pi i t / len} in
// fp64 and fp32 for len = L, L/2, L/4 (the split path's sub-rows).
namespace fftk {
struct Twiddles {
  int L = 0;
  DevBuf f32, f64;
  void ensure(int L_, cudaStream_t s);
  // the table of length len (L, L/2 or L/4)
  template <typename C>
  const C* table(int len) const {
    const C* base;
    if constexpr (sizeof(C) == 8) base = f32.as<C>();
    else base = f64.as<C>();
    size_t o = 0;  // per length: plain table (len) + stage tables (< len)
    for (int l = L; l > len; l /= 2) o += 2 * size_t(l);
    return base + o;
  }
};
// FFT method (complex64): object / fringe spectra in the transposed layout,
// the inverse restricted to a row band and the first nh columns (+ peers).
// split: two scratch buffers (radix-2 pre-pass levels for rows > 8192)
int forward_object(const float* re, const float* im, int no, int off, int L, const Twiddles& tw,
                   float2* spec_t, DevBuf& s1, DevBuf& s2, DevBuf* split, cudaStream_t s);
int forward_full(const float2* grid, int L, const Twiddles& tw, float2* spec_t, DevBuf& s1,
                 DevBuf* split, cudaStream_t s);
int inverse_band(const float2* spec_t, const float2* fringe_t, int L, int nh, int row0, int rows,
                 const Twiddles& tw, float2* out, const PeerPlanes& peers, DevBuf& s1, DevBuf& s2,
                 DevBuf* split, cudaStream_t s);
// fp64 2-D DFT of an n x n field in place (natural layout), inverse unscaled.
int fft2d_f64(double2* f, int n, bool inverse, const Twiddles& tw, DevBuf& s1, DevBuf* split,
              cudaStream_t s);
}  // namespace fftk

struct FftPlan {
  int L = 0, n_layers = 0;
  fftk::Twiddles tw;
  DevBuf fringe_spec, grid, acc, s1, s2, split[2];
  FftPlan() = default;
  FftPlan(const FftPlan&) = delete;
  FftPlan& operator=(const FftPlan&) = delete;
};
// Per-layer fringe spectra on the 2Nh x 2Nh grid (precompute).
void fft_prepare(FftPlan& fp, const wcgh_layer* layers, int n_layers, int nh, cudaStream_t stream);
// out (rows x nh) = band of sum_layers A_eff_l (*) F_l; a_im (optional): the
// imaginary part of a complex A_eff.
int launch_fft_synthesis(FftPlan& fp, const float* a_eff, int no, int off, int nh, int row0,
                         int rows, float2* out, cudaStream_t stream, DirectTiming* timing,
                         const PeerPlanes* peers = nullptr, const float* a_im = nullptr);

// ---- reconstruction and SSIM (K6, K7) --------------
struct ReconPlan {
  int n = 0;
  fftk::Twiddles tw;         // fp64 tables for n
  DevBuf field, s1, split[2];  // n x n double2 working field + FFT scratch
  ReconPlan() = default;
  ReconPlan(const ReconPlan&) = delete;
  ReconPlan& operator=(const ReconPlan&) = delete;
};
double2* recon_field(ReconPlan& rp, int n);
// field <- device input (complex64 if single, else complex128)
void load_field(ReconPlan& rp, const void* dev_in, bool single, int n, cudaStream_t s);
int launch_fft2d(ReconPlan& rp, int n, bool inverse, cudaStream_t s);
int launch_transfer(int n, double wavelength, double pitch, double z_signed, double2* out,
                    cudaStream_t s);
// field <- IDFT(DFT(field) * transfer), scaled by 1/n^2 when `scaled`
int launch_propagate(ReconPlan& rp, int n, double wavelength, double pitch, double z_signed,
                     bool scaled, cudaStream_t s);
int launch_reconstruct(ReconPlan& rp, int n, double wavelength, double pitch, double z,
                       bool intensity, double* out, cudaStream_t s);
// *result = sum of window scores (divide by the window count on the host)
int launch_ssim(const double* a, const double* b, int w, int h, int window, double k1, double k2,
                double dynamic_range, DevBuf& scratch, double* result, cudaStream_t s);

// LUT supports live in guarded allocations: zeroed guard rows before
// (prefetch below row 0: <= B*(D+1)+1 rows) and after (a CTA's last row
// groups overhang the band by < B*R*W rows; they compute on guard data and are
// never stored) plus kLutPadCols zeroed tail elements, so the superposition
// kernel's register window never needs bounds checks.
constexpr int kLutGuardBefore = 64;
constexpr int kLutGuardAfter = 8 * 8 * 8 + 16;  // B*R*W for the compiled shapes (W <= 8)
constexpr int kLutPadCols = 256;
inline size_t lut_alloc_bytes(int n) {
  const size_t span = size_t(2 * n - 1);
  return ((span + kLutGuardBefore + kLutGuardAfter) * span + kLutPadCols) * sizeof(float2);
}
// Zeroes the allocation and returns the pointer to support element (0, 0).
inline float2* lut_in_alloc(DevBuf& buf, int n, cudaStream_t s) {
  buf.reserve(lut_alloc_bytes(n));
  WCGH_CUDA(cudaMemsetAsync(buf.p, 0, lut_alloc_bytes(n), s));
  return buf.as<float2>() + size_t(kLutGuardBefore) * size_t(2 * n - 1);
}

// Builds the (2n-1)^2 complex64 support of block size B (fp64 sums).
int launch_build_lut(const wcgh_layer& scene, int n, int block, float2* lut, DevBuf& scratch,
                     cudaStream_t stream);
// Run lists of one stage's m x m cell grid (column-major): runs of nonzero
// cells (gaps <= the kernel's window height stepped through) as int4
// (c_x, c_y start, steps, dense offset) plus the dense per-step weights.
// Host totals (n_runs, n_dense, nnz) are filled after stage_cells_totals_async
// has completed.
struct StageCells {
  int m = 0;
  int gap = 0;  // run gap threshold (the window height R) the lists were built with
  int n_runs = 0, n_dense = 0, nnz = 0;
  DevBuf counts, offsets, runs, dense;
  // host copies of the run list (the K4 chunk kernel takes each chunk's runs
  // and weights as a kernel parameter block); valid after stage_cells_fetch
  bool host_valid = false;
  std::vector<int4> h_runs;
  std::vector<float> h_dense;
};
int launch_stage_cells(const float* w, int m, StageCells& sc, cudaStream_t stream);
void stage_cells_totals_async(const StageCells& sc, int* host3, cudaStream_t stream);
// Copies the run list (n_runs, n_dense filled) to the host; blocks until the
// stream has produced it.
void stage_cells_fetch(StageCells& sc, cudaStream_t stream);
// out (rows x nh complex64, overwritten) = superposition of the stage's
// listed cells with the block-B LUT; object grid offset `off` on the plane.
// accumulate: out += instead; rotate: out += i * superposition (the
// imaginary weights of a complex object, by linearity).
int launch_lut_stage(const float2* lut, int nh, int block, StageCells& sc, int off, int row0,
                     int rows, float2* out, DevBuf& partial, cudaStream_t stream,
                     DirectTiming* timing, bool accumulate, bool rotate = false);
// Dense weight grid convenience: builds the list, reads nnz (synchronizes),
// superposes.
int launch_lut_dense(const float2* lut, int nh, int block, const float* w, int m, int off,
                     int row0, int rows, float2* out, StageCells& sc, DevBuf& partial,
                     cudaStream_t stream, long long* nnz_out, bool accumulate = false,
                     bool rotate = false);

}  // namespace wcgh
