// Hand-written FFTs for the FFT synthesis method and
// the fp64 reconstruction (fft_2d, fft.cpp:10-68): no cuFFT.
//
// Building block: k_fft_rows — batched 1-D FFTs along the rows of an array,
// each row of L = 2^m complex values held in shared memory (one CTA per row,
// or several short rows per CTA), Stockham autosort stages of radix 16 (then
// 8/4/2 for the remaining bits) done in registers: every thread owns 16
// elements per stage (EPT = min(16, L)), reads them, synchronises, applies
// the stage twiddles (a precomputed fp64-accurate table e^{-2 pi i t / L})
// and an in-register radix-R DFT, and writes them back in place. Shared
// memory is padded by one element per 16 so the strided stores of the early
// stages spread over the banks. Loads and stores go through functors, so the
// zero-padding of the object, the spectral product and the band extraction
// (with the fused row-tile gather) ride on the row passes instead of extra
// passes over HBM. Rows longer than fit in shared memory (fp32 L = 32768,
// fp64 L = 16384) take one radix-2 decimation-in-frequency pre-pass and two
// half-length sub-rows.
//
// A 2-D transform is rows -> transpose -> rows (-> transpose): the FFT
// method keeps spectra in the transposed layout (the pointwise product does
// not care), so forward and inverse are 3 passes each, and it prunes: the
// forward pass transforms only the No object rows, the second pass reads
// only the No nonzero columns, the inverse keeps only the band's rows and the
// first Nh columns.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <utility>

#include "wcgh_internal.cuh"

namespace wcgh {
namespace fftk {
namespace {

// ---- complex helpers (float2 / double2) -------------------------------------
template <typename C> struct Real;
template <> struct Real<float2> { using T = float; };
template <> struct Real<double2> { using T = double; };
template <typename C> __device__ __forceinline__ C mk(typename Real<C>::T x, typename Real<C>::T y) {
  C r;
  r.x = x;
  r.y = y;
  return r;
}
template <typename C> __device__ __forceinline__ C add(C a, C b) { return mk<C>(a.x + b.x, a.y + b.y); }
template <typename C> __device__ __forceinline__ C sub(C a, C b) { return mk<C>(a.x - b.x, a.y - b.y); }
template <typename C> __device__ __forceinline__ C mul(C a, C b) {
  return mk<C>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b) (inverse-transform twiddles from the forward table)
template <typename C> __device__ __forceinline__ C mulc(C a, C b) {
  return mk<C>(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

// cos / sin (2 pi j / 16), j = 0..15
__device__ __constant__ double c_c16[16] = {
    1.0, 0.92387953251128673848, 0.70710678118654752440, 0.38268343236508977173,
    0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128673848,
    -1.0, -0.92387953251128673848, -0.70710678118654752440, -0.38268343236508977173,
    0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128673848};
__device__ __constant__ double c_s16[16] = {
    0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128673848,
    1.0, 0.92387953251128673848, 0.70710678118654752440, 0.38268343236508977173,
    0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128673848,
    -1.0, -0.92387953251128673848, -0.70710678118654752440, -0.38268343236508977173};

// x * e^{-+ 2 pi i j / 16} (INV: +), exact for the quarter turns
template <int J, bool INV, typename C>
__device__ __forceinline__ C rot16(C x) {
  constexpr int j = J & 15;
  if constexpr (j == 0) {
    return x;
  } else if constexpr (j == 4) {  // -i (fwd) / +i (inv)
    return INV ? mk<C>(-x.y, x.x) : mk<C>(x.y, -x.x);
  } else if constexpr (j == 8) {
    return mk<C>(-x.x, -x.y);
  } else if constexpr (j == 12) {
    return INV ? mk<C>(x.y, -x.x) : mk<C>(-x.y, x.x);
  } else {
    using T = typename Real<C>::T;
    const T c = T(c_c16[j]), s = T(INV ? c_s16[j] : -c_s16[j]);
    return mk<C>(x.x * c - x.y * s, x.x * s + x.y * c);
  }
}

template <int R>
__host__ __device__ constexpr int bitrev(int v) {
  int r = 0;
  for (int b = 1; b < R; b <<= 1) {
    r = (r << 1) | (v & 1);
    v >>= 1;
  }
  return r;
}

// In-register DFT of length R (2, 4, 8, 16): radix-2 DIT on the bit-reversed
// input, output in natural order.
template <int R, int I>
struct BitRev {
  static constexpr int value = bitrev<R>(I);
};

template <int R, typename C, int... I>
__device__ __forceinline__ void bitrev_copy(const C (&x)[R], C (&y)[R], std::integer_sequence<int, I...>) {
  ((y[I] = x[BitRev<R, I>::value]), ...);  // compile-time permutation: registers only
}

template <int R>
constexpr int ilog2c() {
  int r = 0;
  while ((1 << r) < R) ++r;
  return r;
}

template <int R, bool INV, typename C>
__device__ __forceinline__ void dft(C (&x)[R]) {
  C y[R];
  bitrev_copy<R>(x, y, std::make_integer_sequence<int, R>{});
  constexpr int S = ilog2c<R>();
#pragma unroll
  for (int st = 0; st < S; ++st) {  // counted loops: fully unrolled, static indices
    const int len = 2 << st;
#pragma unroll
    for (int i = 0; i < R; i += len) {
#pragma unroll
      for (int k = 0; k < len / 2; ++k) {
        C v = y[i + k + len / 2];
        // twiddle e^{-+2 pi i k / len} = rot16<k * 16 / len>
        switch (k * (16 / len)) {
          case 0: break;
          case 1: v = rot16<1, INV>(v); break;
          case 2: v = rot16<2, INV>(v); break;
          case 3: v = rot16<3, INV>(v); break;
          case 4: v = rot16<4, INV>(v); break;
          case 5: v = rot16<5, INV>(v); break;
          case 6: v = rot16<6, INV>(v); break;
          case 7: v = rot16<7, INV>(v); break;
          default: break;
        }
        const C u = y[i + k];
        y[i + k] = add(u, v);
        y[i + k + len / 2] = sub(u, v);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) x[i] = y[i];
}

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }
__host__ __device__ __forceinline__ int pad_len(int L) { return L + L / 16 + 1; }

// One Stockham stage of radix R over a row in shared memory: the thread's
// EPT elements = EPT/R butterflies j = t + b * tpr.
template <int R, int EPT, bool INV, typename C>
__device__ __forceinline__ void stage(C* s, int L, int Ns, int t, int tpr, const C* __restrict__ tw) {
  constexpr int NB = EPT / R;
  C x[NB][R];
  const int LR = L / R;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + b * tpr;
#pragma unroll
    for (int r = 0; r < R; ++r) x[b][r] = s[pad(j + r * LR)];
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + b * tpr;
    const int k = j & (Ns - 1);
    if (Ns > 1) {
      // the stage's own table tw[(r-1) Ns + k] = e^{-2 pi i r k / (Ns R)}:
      // consecutive k across the lanes, so every load is coalesced
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const C w = tw[(r - 1) * Ns + k];
        x[b][r] = INV ? mulc(x[b][r], w) : mul(x[b][r], w);
      }
    }
    dft<R, INV>(x[b]);
    const int base = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) s[pad(base + r * Ns)] = x[b][r];
  }
  __syncthreads();
}

// The whole row transform in shared memory (all stages).
// tw: the row length's stage tables (Twiddles::stages), one per stage with
// Ns > 1, consumed in order ((R - 1) Ns entries each)
template <int EPT, bool INV, typename C>
__device__ void row_fft(C* s, int L, int log2L, int t, int tpr, const C* __restrict__ tw) {
  int Ns = 1, bits = log2L;
  while (bits > 0) {
    const int rb = bits >= 4 ? 4 : bits;
    if constexpr (EPT >= 16) {
      if (rb == 4) {
        stage<16, EPT, INV>(s, L, Ns, t, tpr, tw);
        if (Ns > 1) tw += 15 * Ns;
        Ns <<= 4; bits -= 4; continue;
      }
    }
    if constexpr (EPT >= 8) {
      if (rb == 3) {
        stage<8, EPT, INV>(s, L, Ns, t, tpr, tw);
        if (Ns > 1) tw += 7 * Ns;
        Ns <<= 3; bits -= 3; continue;
      }
    }
    if constexpr (EPT >= 4) {
      if (rb == 2) {
        stage<4, EPT, INV>(s, L, Ns, t, tpr, tw);
        if (Ns > 1) tw += 3 * Ns;
        Ns <<= 2; bits -= 2; continue;
      }
    }
    stage<2, EPT, INV>(s, L, Ns, t, tpr, tw);
    if (Ns > 1) tw += Ns;
    Ns <<= 1;
    bits -= 1;
  }
}

// Batched row FFTs with load / store functors: ld(row, e) -> C, st(row, e, C).
template <int EPT, bool INV, typename C, class Ld, class St>
__global__ void __launch_bounds__(512) k_fft_rows(int L, int log2L, int rows, const C* __restrict__ tw,
                                                   Ld ld, St st) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tpr = L / EPT;
  const int rpc = blockDim.x / tpr;
  const int lr = threadIdx.x / tpr, t = threadIdx.x - lr * tpr;
  const int row = blockIdx.x * rpc + lr;
  C* s = reinterpret_cast<C*>(smem_raw) + size_t(lr) * pad_len(L);
  const bool active = row < rows;
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int e = t + i * tpr;
    s[pad(e)] = active ? ld(row, e) : mk<C>(0, 0);
  }
  __syncthreads();
  row_fft<EPT, INV>(s, L, log2L, t, tpr, tw);
  if (!active) return;
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int e = t + i * tpr;
    st(row, e, s[pad(e)]);
  }
}

// Radix-2 DIF pre-pass for rows too long for shared memory: y0[n] = a + b,
// y1[n] = (a - b) w^n (w = e^{-+2 pi i / L}), a = x[n], b = x[n + L/2];
// out row = [y0 | y1]; X[2k] = DFT(y0)[k], X[2k+1] = DFT(y1)[k].
template <bool INV, typename C, class Ld>
__global__ void k_split2(int L, int rows, const C* __restrict__ tw, Ld ld, C* __restrict__ out) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int h = L / 2;
  if (i >= size_t(rows) * h) return;
  const int row = int(i / h), n = int(i % h);
  const C a = ld(row, n), b = ld(row, n + h);
  const C w = tw[n];
  const C d = sub(a, b);
  out[size_t(row) * L + n] = add(a, b);
  out[size_t(row) * L + h + n] = INV ? mulc(d, w) : mul(d, w);
}

// ---- functors -------------------------------------------------------------
template <typename C> struct LdRows {  // plain rows of a strided array
  const C* p;
  size_t stride;
  __device__ C operator()(int r, int e) const { return p[size_t(r) * stride + e]; }
};
template <typename C> struct StRows {
  C* p;
  size_t stride;
  __device__ void operator()(int r, int e, C v) const { p[size_t(r) * stride + e] = v; }
};
// sub-row p of row r (2 rows per original row) -> out position 2e + p
template <typename C, class St> struct StInterleave {
  St st;
  __device__ void operator()(int r, int e, C v) const { st(r >> 1, 2 * e + (r & 1), v); }
};

// forward pass 1: object row r of the layer's A_eff (re [, im]) zero-padded
// into [off, off + no) of an L-row
struct LdAeffRow {
  const float* re;
  const float* im;
  int no, off;
  __device__ float2 operator()(int r, int e) const {
    const int x = e - off;
    if (x < 0 || x >= no) return make_float2(0.f, 0.f);
    const size_t i = size_t(r) * no + x;
    return make_float2(re[i], im ? im[i] : 0.f);
  }
};
// forward pass 2: column q of the pass-1 result, transposed (L x no),
// zero-padded into [off, off + no)
struct LdPadded {
  const float2* p;
  int no, off;
  __device__ float2 operator()(int r, int e) const {
    const int x = e - off;
    if (x < 0 || x >= no) return make_float2(0.f, 0.f);
    return p[size_t(r) * no + x];
  }
};
// inverse pass 1: the accumulated spectrum (transposed layout) times, for a
// single layer, the fringe spectrum (spectral product fused into the load)
struct LdSpec {
  const float2* a;
  const float2* f;  // nullptr: `a` already holds the product (multi-layer sum)
  size_t stride;
  __device__ float2 operator()(int r, int e) const {
    const size_t i = size_t(r) * stride + e;
    const float2 v = a[i];
    if (!f) return v;
    const float2 w = f[i];
    return make_float2(v.x * w.x - v.y * w.y, v.x * w.y + v.y * w.x);
  }
};
// inverse pass 1 store: keep y in [row0, row0 + rows) -> (L x rows)
struct StBandRows {
  float2* p;
  int row0, rows;
  __device__ void operator()(int r, int e, float2 v) const {
    const int y = e - row0;
    if (y >= 0 && y < rows) p[size_t(r) * rows + y] = v;
  }
};
// inverse pass 2 store: x in [0, nh) of band row r, scaled by 1/L^2, into
// the band and every peer plane (fused row-tile gather)
struct StBandOut {
  float2* out;
  int nh;
  float scale;
  PeerPlanes peers;
  __device__ void operator()(int r, int e, float2 v) const {
    if (e >= nh) return;
    const size_t i = size_t(r) * nh + e;
    const float2 o = make_float2(v.x * scale, v.y * scale);
    out[i] = o;
    store_peers(peers, i, o);
  }
};

// ---- pipelined row FFTs (complex64, rows of 512..8192) -----------------------
// A persistent CTA per SM walks rows r = blockIdx.x, += gridDim.x. While a
// row's stages run, the NEXT row's raw input is already streaming into a
// staging buffer with cp.async (no registers held), so HBM latency and
// bandwidth overlap the shared-memory stages instead of stalling the CTA
// (one 512-thread CTA per SM: 128 registers per thread). Staged loaders copy
// raw bytes and build elements from them: plain rows, the spectral product
// of two rows, the zero-padded object column block, the A_eff row.
__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_bytes(char* dst, const char* src, size_t bytes, int tid, int nt) {
  for (size_t c = size_t(tid); c < bytes / 16; c += size_t(nt)) cp16(dst + 16 * c, src + 16 * c);
}

struct PfRows {
  const float2* p;
  size_t stride;
  static size_t bytes(int L, int) { return size_t(L) * 8; }
  __device__ void prefetch(int r, char* st, int L, int tid, int nt) const {
    cp_bytes(st, reinterpret_cast<const char*>(p + size_t(r) * stride), size_t(L) * 8, tid, nt);
  }
  __device__ float2 get(const char* st, int e) const { return reinterpret_cast<const float2*>(st)[e]; }
};
struct PfSpec {  // spectrum row (times the fringe spectrum row when f != nullptr)
  const float2* a;
  const float2* f;
  size_t stride;
  static size_t bytes(int L, int two) { return size_t(L) * 8 * (two ? 2 : 1); }
  __device__ void prefetch(int r, char* st, int L, int tid, int nt) const {
    cp_bytes(st, reinterpret_cast<const char*>(a + size_t(r) * stride), size_t(L) * 8, tid, nt);
    if (f) cp_bytes(st + size_t(L) * 8, reinterpret_cast<const char*>(f + size_t(r) * stride), size_t(L) * 8, tid, nt);
  }
  __device__ float2 get(const char* st, int e, int L) const {
    const float2 v = reinterpret_cast<const float2*>(st)[e];
    if (!f) return v;
    const float2 w = reinterpret_cast<const float2*>(st)[L + e];
    return make_float2(v.x * w.x - v.y * w.y, v.x * w.y + v.y * w.x);
  }
};
struct PfPadded {  // (L x no) rows, zero-padded into [off, off + no)
  const float2* p;
  int no, off;
  static size_t bytes(int, int no) { return size_t(no) * 8; }
  __device__ void prefetch(int r, char* st, int, int tid, int nt) const {
    cp_bytes(st, reinterpret_cast<const char*>(p + size_t(r) * no), size_t(no) * 8, tid, nt);
  }
  __device__ float2 get(const char* st, int e) const {
    const int x = e - off;
    return (x >= 0 && x < no) ? reinterpret_cast<const float2*>(st)[x] : make_float2(0.f, 0.f);
  }
};
struct PfAeff {  // A_eff row r (re, optional im), zero-padded into [off, off + no)
  const float* re;
  const float* im;
  int no, off;
  static size_t bytes(int, int no) { return size_t(no) * 8; }
  __device__ void prefetch(int r, char* st, int, int tid, int nt) const {
    cp_bytes(st, reinterpret_cast<const char*>(re + size_t(r) * no), size_t(no) * 4, tid, nt);
    if (im) cp_bytes(st + size_t(no) * 4, reinterpret_cast<const char*>(im + size_t(r) * no), size_t(no) * 4, tid, nt);
  }
  __device__ float2 get(const char* st, int e) const {
    const int x = e - off;
    if (x < 0 || x >= no) return make_float2(0.f, 0.f);
    return make_float2(reinterpret_cast<const float*>(st)[x], im ? reinterpret_cast<const float*>(st)[no + x] : 0.f);
  }
};
template <class Ld> __device__ __forceinline__ float2 pf_get(const Ld& ld, const char* st, int e, int) { return ld.get(st, e); }
template <> __device__ __forceinline__ float2 pf_get<PfSpec>(const PfSpec& ld, const char* st, int e, int L) { return ld.get(st, e, L); }

template <bool INV, class Ld, class St>
__global__ void __launch_bounds__(512) k_fft_rows_pf(int L, int log2L, int rows, const float2* __restrict__ tw,
                                                     Ld ld, St st) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* F = reinterpret_cast<float2*>(smem_raw);
  char* stg = reinterpret_cast<char*>(smem_raw) + (size_t(pad_len(L)) * 8 + 15) / 16 * 16;
  const int t = threadIdx.x, tpr = blockDim.x;  // tpr = L / 16
  int row = blockIdx.x;
  if (row < rows) ld.prefetch(row, stg, L, t, tpr);
  cp_commit();
  for (; row < rows; row += gridDim.x) {
    cp_wait_all();
    __syncthreads();  // staged row complete; previous row's stores done
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int e = t + i * tpr;
      F[pad(e)] = pf_get(ld, stg, e, L);
    }
    __syncthreads();  // staging free: stream the next row in behind the stages
    const int nxt = row + gridDim.x;
    if (nxt < rows) ld.prefetch(nxt, stg, L, t, tpr);
    cp_commit();
    row_fft<16, INV>(F, L, log2L, t, tpr, tw);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int e = t + i * tpr;
      st(row, e, F[pad(e)]);
    }
  }
}

// ---- transpose ------------------------------------------------------------
template <typename C>
__global__ void k_transpose(const C* __restrict__ in, int rows, int cols, C* __restrict__ out) {
  __shared__ C tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int y = by + threadIdx.y + k, x = bx + threadIdx.x;
    if (y < rows && x < cols) tile[threadIdx.y + k][threadIdx.x] = in[size_t(y) * cols + x];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int x = by + threadIdx.x, y = bx + threadIdx.y + k;  // out is cols x rows
    if (y < cols && x < rows) out[size_t(y) * rows + x] = tile[threadIdx.x][threadIdx.y + k];
  }
}

__global__ void k_twiddles(int L, double2* __restrict__ d, float2* __restrict__ f) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L) return;
  double s, c;
  sincospi(-2.0 * double(t) / double(L), &s, &c);
  d[t] = make_double2(c, s);
  f[t] = make_float2(float(c), float(s));
}

__global__ void k_stage_twiddles(int Ns, int R, double2* __restrict__ d, float2* __restrict__ f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (R - 1) * Ns) return;
  const int r = i / Ns + 1, k = i % Ns;
  double s, c;
  sincospi(-2.0 * double(r) * double(k) / (double(Ns) * double(R)), &s, &c);
  d[i] = make_double2(c, s);
  f[i] = make_float2(float(c), float(s));
}

int ilog2(int v) {
  int r = 0;
  while ((1 << r) < v) ++r;
  return r;
}

// longest row kept in shared memory (512 threads x 16 elements; 70 KB fp32,
// 139 KB fp64); longer rows are split by radix-2 DIF pre-passes
constexpr int kMaxRowL = 8192;

template <typename C, bool INV, int EPT, class Ld, class St>
void launch_rows_ept(int L, int rows, const C* tw, Ld ld, St st, cudaStream_t s) {
  const int tpr = L / EPT;
  const int rpc = std::max(1, 256 / tpr);
  const int threads = tpr * rpc;
  const size_t smem = sizeof(C) * size_t(pad_len(L)) * rpc;
  auto kern = k_fft_rows<EPT, INV, C, Ld, St>;
  if (smem > 48 * 1024) WCGH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const unsigned blocks = unsigned((rows + rpc - 1) / rpc);
  kern<<<blocks, threads, smem, s>>>(L, ilog2(L), rows, tw, ld, st);
  WCGH_CHECK_LAUNCH();
}

}  // namespace

// Row-FFT driver: direct in shared memory, or radix-2 split + half rows.
template <typename C, bool INV, int DEPTH = 0, class Ld, class St>
int fft_rows(int L, int rows, const Twiddles& tws, Ld ld, St st, DevBuf* split, cudaStream_t s) {
  const C* tw = tws.table<C>(L);
  if (L <= kMaxRowL) {
    const C* st_tw = tw + L;  // the stage tables follow the plain table
    if (L >= 16) launch_rows_ept<C, INV, 16>(L, rows, st_tw, ld, st, s);
    else if (L == 8) launch_rows_ept<C, INV, 8>(L, rows, st_tw, ld, st, s);
    else if (L == 4) launch_rows_ept<C, INV, 4>(L, rows, st_tw, ld, st, s);
    else launch_rows_ept<C, INV, 2>(L, rows, st_tw, ld, st, s);
    return 1;
  }
  if constexpr (DEPTH < 2) {
    // DIF radix-2 split into [y0 | y1], then 2 * rows rows of L/2 whose
    // outputs interleave (row 2r+p = half p of row r -> positions 2k+p)
    C* y = static_cast<C*>(split[DEPTH].reserve(sizeof(C) * size_t(L) * rows));
    const size_t n = size_t(rows) * (L / 2);
    k_split2<INV, C, Ld><<<unsigned((n + 255) / 256), 256, 0, s>>>(L, rows, tw, ld, y);
    WCGH_CHECK_LAUNCH();
    return 1 + fft_rows<C, INV, DEPTH + 1>(L / 2, 2 * rows, tws, LdRows<C>{y, size_t(L / 2)},
                                           StInterleave<C, St>{st}, split, s);
  } else {
    throw ValidationError("fft: length above 4 x 8192 not supported");
  }
}

void Twiddles::ensure(int L_, cudaStream_t s) {
  if (L == L_) return;
  require(L_ >= 2 && (L_ & (L_ - 1)) == 0, "fft: length must be a power of two");
  L = L_;
  // for len = L, L/2, L/4 (the split path's sub-rows), back to back: the plain
  // table e^{-2 pi i t / len} (len entries, the split pre-pass) followed by the
  // per-stage tables of row_fft's stage schedule (< len entries), each
  // [r - 1][k] = e^{-2 pi i r k / (Ns R)}, all from fp64 sincospi
  double2* d = static_cast<double2*>(f64.reserve(sizeof(double2) * 4 * size_t(L)));
  float2* f = static_cast<float2*>(f32.reserve(sizeof(float2) * 4 * size_t(L)));
  size_t o = 0;
  for (int len = L; len >= 2 && len * 4 >= L; len /= 2) {
    k_twiddles<<<unsigned((len + 255) / 256), 256, 0, s>>>(len, d + o, f + o);
    WCGH_CHECK_LAUNCH();
    size_t so = o + size_t(len);
    int Ns = 1, bits = ilog2(len);
    while (bits > 0) {
      const int rb = bits >= 4 ? 4 : bits, R = 1 << rb;
      if (Ns > 1) {
        const int cnt = (R - 1) * Ns;
        k_stage_twiddles<<<unsigned((cnt + 255) / 256), 256, 0, s>>>(Ns, R, d + so, f + so);
        WCGH_CHECK_LAUNCH();
        so += size_t(cnt);
      }
      Ns <<= rb;
      bits -= rb;
    }
    o += 2 * size_t(len);
  }
}

template <typename C>
int transpose(const C* in, int rows, int cols, C* out, cudaStream_t s) {
  dim3 grid(unsigned((cols + 31) / 32), unsigned((rows + 31) / 32));
  k_transpose<C><<<grid, dim3(32, 8), 0, s>>>(in, rows, cols, out);
  WCGH_CHECK_LAUNCH();
  return 1;
}

// ---- the FFT method's transforms (complex64) ---------------------------------

// Object spectrum, transposed layout (L x L, row = x-frequency): the layer's
// A_eff zero-padded into [off, off + no)^2 of the L x L grid.
// rows of 512..8192 take the pipelined kernel, other lengths the plain one
inline bool use_pf(int L) { return L >= 512 && L <= kMaxRowL; }

template <bool INV, class Pf, class St>
int launch_rows_pf(int L, int rows, const Twiddles& tws, Pf ld, St st, size_t stage_bytes, cudaStream_t s) {
  const float2* tw = tws.table<float2>(L) + L;  // stage tables
  const size_t smem = (size_t(pad_len(L)) * 8 + 15) / 16 * 16 + stage_bytes;
  auto kern = k_fft_rows_pf<INV, Pf, St>;
  if (smem > 48 * 1024) WCGH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0, dev = 0, sms = 0;
  WCGH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L / 16, smem));
  WCGH_CUDA(cudaGetDevice(&dev));
  WCGH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = std::max(1, std::min(rows, std::max(1, per_sm) * sms));
  kern<<<grid, L / 16, smem, s>>>(L, ilog2(L), rows, tw, ld, st);
  WCGH_CHECK_LAUNCH();
  return 1;
}

int forward_object(const float* re, const float* im, int no, int off, int L, const Twiddles& tw,
                   float2* spec_t, DevBuf& s1, DevBuf& s2, DevBuf* split, cudaStream_t s) {
  float2* rowsft = static_cast<float2*>(s1.reserve(sizeof(float2) * size_t(no) * L));
  float2* tr = static_cast<float2*>(s2.reserve(sizeof(float2) * size_t(no) * L));
  int n = 0;
  if (use_pf(L) && no % 4 == 0)
    n += launch_rows_pf<false>(L, no, tw, PfAeff{re, im, no, off}, StRows<float2>{rowsft, size_t(L)},
                               size_t(no) * 8, s);
  else
    n += fft_rows<float2, false>(L, no, tw, LdAeffRow{re, im, no, off}, StRows<float2>{rowsft, size_t(L)},
                                 split, s);
  n += transpose(rowsft, no, L, tr, s);  // (no x L) -> (L x no)
  if (use_pf(L) && no % 2 == 0)
    n += launch_rows_pf<false>(L, L, tw, PfPadded{tr, no, off}, StRows<float2>{spec_t, size_t(L)},
                               size_t(no) * 8, s);
  else
    n += fft_rows<float2, false>(L, L, tw, LdPadded{tr, no, off}, StRows<float2>{spec_t, size_t(L)}, split, s);
  return n;
}

// Spectrum of a full L x L grid (the fringe), transposed layout.
int forward_full(const float2* grid, int L, const Twiddles& tw, float2* spec_t, DevBuf& s1,
                 DevBuf* split, cudaStream_t s) {
  float2* a = static_cast<float2*>(s1.reserve(sizeof(float2) * size_t(L) * L));
  int n = fft_rows<float2, false>(L, L, tw, LdRows<float2>{grid, size_t(L)}, StRows<float2>{a, size_t(L)},
                                  split, s);
  n += transpose(a, L, L, spec_t, s);
  n += fft_rows<float2, false>(L, L, tw, LdRows<float2>{spec_t, size_t(L)}, StRows<float2>{spec_t, size_t(L)},
                               split, s);
  return n;
}

// Inverse of spec_t (times fringe_t when given) restricted to the band rows
// [row0, row0 + rows) and columns [0, nh), scaled by 1/L^2, into out (+ peers).
int inverse_band(const float2* spec_t, const float2* fringe_t, int L, int nh, int row0, int rows,
                 const Twiddles& tw, float2* out, const PeerPlanes& peers, DevBuf& s1, DevBuf& s2,
                 DevBuf* split, cudaStream_t s) {
  float2* g = static_cast<float2*>(s1.reserve(sizeof(float2) * size_t(L) * rows));
  float2* gt = static_cast<float2*>(s2.reserve(sizeof(float2) * size_t(L) * rows));
  int n = 0;
  if (use_pf(L))
    n += launch_rows_pf<true>(L, L, tw, PfSpec{spec_t, fringe_t, size_t(L)}, StBandRows{g, row0, rows},
                              size_t(L) * 8 * (fringe_t ? 2 : 1), s);
  else
    n += fft_rows<float2, true>(L, L, tw, LdSpec{spec_t, fringe_t, size_t(L)}, StBandRows{g, row0, rows},
                                split, s);
  n += transpose(g, L, rows, gt, s);  // (L x rows) -> (rows x L)
  const float scale = float(1.0 / (double(L) * double(L)));
  if (use_pf(L))
    n += launch_rows_pf<true>(L, rows, tw, PfRows{gt, size_t(L)}, StBandOut{out, nh, scale, peers},
                              size_t(L) * 8, s);
  else
    n += fft_rows<float2, true>(L, rows, tw, LdRows<float2>{gt, size_t(L)}, StBandOut{out, nh, scale, peers},
                                split, s);
  return n;
}

// fft_2d (fft.cpp:45-68) in fp64, natural layout, in place; inverse unscaled.
int fft2d_f64(double2* f, int n, bool inverse, const Twiddles& tw, DevBuf& s1, DevBuf* split,
              cudaStream_t s) {
  double2* t = static_cast<double2*>(s1.reserve(sizeof(double2) * size_t(n) * n));
  int k = 0;
  if (inverse) {
    k += fft_rows<double2, true>(n, n, tw, LdRows<double2>{f, size_t(n)}, StRows<double2>{f, size_t(n)}, split, s);
    k += transpose(f, n, n, t, s);
    k += fft_rows<double2, true>(n, n, tw, LdRows<double2>{t, size_t(n)}, StRows<double2>{t, size_t(n)}, split, s);
  } else {
    k += fft_rows<double2, false>(n, n, tw, LdRows<double2>{f, size_t(n)}, StRows<double2>{f, size_t(n)}, split, s);
    k += transpose(f, n, n, t, s);
    k += fft_rows<double2, false>(n, n, tw, LdRows<double2>{t, size_t(n)}, StRows<double2>{t, size_t(n)}, split, s);
  }
  k += transpose(t, n, n, f, s);
  return k;
}

}  // namespace fftk
}  // namespace wcgh

WCGH_CHK_TU(wcgh_fftk)
