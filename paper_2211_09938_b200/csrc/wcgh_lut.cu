// K5: block-LUT construction and K4: LUT fringe superposition.
//
// K5 restates build_block_lut (core/src/fringe_lut.cpp:53-93): the extended
// single-point grid F(dx, dy) = polar(1/r, k r) (fringe_lut.cpp:27-32) in
// fp64, then the B x B box sum in the reference's (pv, pu) order in fp64,
// stored as complex64 — the CGHL cache payload (fringe_lut.cpp:107-113),
// which is what every LUT the reference's `generate` uses has passed through
// (pipeline.cpp:174-177).
//
// K4 restates apply_cells -> apply_block_unchecked (synthesis.cpp:18-42,
// 55-69): plane(x, y) += w_c * S_B(x - a_x, y - a_y), anchors a = off + B*cell,
// for the nonzero-weight gated cells of one stage (zero weights add nothing,
// synthesis.cpp:20). The reference streams 16 B of LUT and 16 B of plane per
// update (its hot loop, synthesis.cpp:33); here the plane stays in registers
// and LUT samples are reused from registers:
//   * cells are listed column-major (per cell column c_x, ascending c_y);
//   * a thread owns R pixel rows at stride B and PX pixel columns at stride
//     32 (default R = 8, PX = 2); the W = 4 warps of a CTA share one row
//     residue mod B and take consecutive row groups, so a LUT row one warp
//     loads is the row the next warp needs R steps later (L1 reuse);
//   * for cell (c_x, c_y) pixel row j reads LUT row y_j - a_y, and
//     (y_j + B) - (a_y + B) is the same row: stepping c_y -> c_y + 1 shifts
//     the R-row register window by one, so each step loads one new LUT row
//     segment (PX samples, prefetched D steps ahead) and performs R*PX
//     complex-by-real MACs, one packed FFMA2 (fma.rn.f32x2) each;
//   * runs of cells closer than R rows are stepped through; longer gaps
//     restart the window.
// Cells are split into fixed chunks of the column-major list; each
// (tile, chunk) CTA writes a partial plane and a fixed-order reduction sums
// them, so the result does not depend on the launch or the row-band split.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "wcgh_internal.cuh"

namespace wcgh {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__global__ void k_point_grid(double wavelength, double pitch, double z, int ext, int lo,
                             double2* __restrict__ base) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size_t(ext) * ext) return;
  const int col = int(i % ext), row = int(i / ext);
  const double px = double(lo + col) * pitch;
  const double py = double(lo + row) * pitch;
  const double r = sqrt(px * px + py * py + z * z);
  const double k = 2.0 * 3.14159265358979323846 / wavelength;
  double s, c;
  sincos(k * r, &s, &c);
  const double m = 1.0 / r;
  base[i] = make_double2(m * c, m * s);
}

__global__ void k_box_sum(const double2* __restrict__ base, int ext, int span, int block,
                          float2* __restrict__ lut) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size_t(span) * span) return;
  const int col = int(i % span), row = int(i / span);
  double sr = 0.0, si = 0.0;
  for (int pv = 0; pv < block; ++pv) {
    const double2* src = base + size_t(row - pv + block - 1) * ext;
    for (int pu = 0; pu < block; ++pu) {
      const double2 v = src[col - pu + block - 1];
      sr += v.x;
      si += v.y;
    }
  }
  lut[i] = make_float2(float(sr), float(si));
}

// Run lists of a dense m x m weight grid (one warp per cell column c_x):
// nonzero cells in ascending c_y are grouped into runs whose consecutive
// gaps are <= R (the superposition kernel steps through such gaps with its
// register window); each run gets a record (c_x, c_y start, length, offset
// into a dense weight array holding every step's weight, zeros in gaps).
__global__ void k_runs_count(const float* __restrict__ w, int m, int R, int* __restrict__ n_runs,
                             int* __restrict__ n_dense, int* __restrict__ n_nnz) {
  const int lane = threadIdx.x & 31;
  const int cx = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (cx >= m) return;
  int last = -(1 << 29), runs = 0, dense = 0, nnz = 0, start = 0;
  for (int base = 0; base < m; base += 32) {
    const int cy = base + lane;
    const float v = cy < m ? w[size_t(cy) * m + cx] : 0.0f;
    unsigned mask = __ballot_sync(kFull, v != 0.0f);
    while (mask) {
      const int c = base + __ffs(mask) - 1;
      mask &= mask - 1;
      ++nnz;
      if (c - last > R) {
        if (runs) dense += last - start + 1;
        ++runs;
        start = c;
      }
      last = c;
    }
  }
  if (runs) dense += last - start + 1;
  if (lane == 0) {
    n_runs[cx] = runs;
    n_dense[cx] = dense;
    n_nnz[cx] = nnz;
  }
}

__global__ void k_runs_fill(const float* __restrict__ w, int m, int R, const int* __restrict__ run_off,
                            const int* __restrict__ dense_off, int4* __restrict__ runs,
                            float* __restrict__ dense) {
  const int lane = threadIdx.x & 31;
  const int cx = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (cx >= m) return;
  int rp = run_off[cx], dp = dense_off[cx];
  int cur = -1, start = 0, last = -(1 << 29), wofs = 0;
  for (int base = 0; base < m; base += 32) {
    const int cy = base + lane;
    const float v = cy < m ? w[size_t(cy) * m + cx] : 0.0f;
    unsigned mask = __ballot_sync(kFull, v != 0.0f);
    while (mask) {
      const int b = __ffs(mask) - 1;
      mask &= mask - 1;
      const int c = base + b;
      const float vc = __shfl_sync(kFull, v, b);
      if (c - last > R) {  // a new run
        if (cur >= 0) {
          if (lane == 0) runs[cur].z = last - start + 1;
          dp = wofs + (last - start + 1);
        }
        cur = rp++;
        start = c;
        wofs = dp;
        if (lane == 0) runs[cur] = make_int4(cx, c, 0, wofs);
      }
      if (lane == 0) dense[wofs + (c - start)] = vc;
      last = c;
    }
  }
  if (cur >= 0 && lane == 0) runs[cur].z = last - start + 1;
}

// acc + w * v on both lanes of a complex sample: one packed FFMA2
// (fma.rn.f32x2, sm_100a) -- per lane the same IEEE fma as fmaf, so results
// are bit-identical to the scalar form at half the issued instructions.
__device__ __forceinline__ float2 ffma2(float w, float2 v, float2 a) {
  float2 r;
  asm("{\n .reg .b64 pv, pw, pa, pr;\n mov.b64 pv, {%2, %3};\n mov.b64 pw, {%4, %4};\n"
      " mov.b64 pa, {%5, %6};\n fma.rn.f32x2 pr, pw, pv, pa;\n mov.b64 {%0, %1}, pr;\n}\n"
      : "=f"(r.x), "=f"(r.y)
      : "f"(v.x), "f"(v.y), "f"(w), "f"(a.x), "f"(a.y));
  return r;
}

// Resident CTAs per SM the register budget is sized for: accumulators
// (2 R PX) + ring (2 (R + D) PX) + ~24 for addressing, per thread.
constexpr int lut_min_blocks(int R, int PX, int D, int W) {
  return 65536 / (W * 32 * (4 * R * PX + 2 * D * PX + 24)) > 0
             ? 65536 / (W * 32 * (4 * R * PX + 2 * D * PX + 24))
             : 1;
}

template <int B, int R, int PX, int D, int W>
__global__ void __launch_bounds__(W * 32, lut_min_blocks(R, PX, D, W))
    k_lut_stage(const float2* __restrict__ lut, int nh, const int4* __restrict__ runs,
                int n_runs, const float* __restrict__ dense, int off, int row0, int rows,
                int tiles_x, int chunk0, int chunk_steps, float2* __restrict__ out,
                size_t out_stride) {
  extern __shared__ float s_w[];
  constexpr int S = R + D;  // ring: R live diagonals + D prefetched
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx = blockIdx.x % tiles_x, tyc = blockIdx.x / tiles_x;
  // The W warps of a CTA share one row residue r (mod B) and take consecutive
  // row groups (R rows at stride B each), so the LUT rows one warp loads are
  // the rows the next warp needs R steps later (L1 reuse at every B).
  const int r = tyc % B;
  const int g = (tyc / B) * W + warp;
  const int yb = g * (B * R) + r;  // band row of pixel row 0
  const int x0 = tx * (32 * PX) + lane;
  const int span = 2 * nh - 1;
  const int d_lo = (chunk0 + blockIdx.y) * chunk_steps;
  const int d_hi = d_lo + chunk_steps;

  // runs starting in [d_lo, d_hi) of the dense step array (runs are ordered by offset)
  auto lower_bound = [&](int key) {
    int lo = 0, hi = n_runs;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(&runs[mid].w) < key) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const int r_lo = lower_bound(d_lo), r_hi = lower_bound(d_hi);
  int w_lo = 0;
#ifdef WCGH_CHECKED
  unsigned smem_floats;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(smem_floats));
  smem_floats /= 4;
  // the guarded LUT allocation (lut_alloc_bytes): every window / prefetch read
  const float2* lut_lo = lut - size_t(kLutGuardBefore) * span;
  const float2* lut_hi = lut + size_t(span + kLutGuardAfter) * span + kLutPadCols;
#define WCGH_LUT_IN(ptr) WCGH_DCHECK((ptr) >= lut_lo && (ptr) + 32 * (PX - 1) < lut_hi)
#else
#define WCGH_LUT_IN(ptr)
#endif
  if (r_lo < r_hi) {
    w_lo = __ldg(&runs[r_lo].w);
    const int4 lr = __ldg(runs + r_hi - 1);
    const int w_n = lr.w + lr.z - w_lo;
    WCGH_DCHECK(w_n + S - 1 <= int(smem_floats));  // incl. the remainder's up-front reads
    for (int i = threadIdx.x; i < w_n; i += W * 32) s_w[i] = __ldg(dense + w_lo + i);
  }
  __syncthreads();

  float2 acc[R][PX];
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int i = 0; i < PX; ++i) acc[j][i] = make_float2(0.f, 0.f);

  // LUT row of pixel row j at cell row cy: (row0 + yb + jB) - off - B cy + nh - 1.
  // `lut` points into a guarded allocation (guard rows before and
  // after, kLutPadCols elements of tail padding), so the window and the
  // prefetch never need clamping; out-of-plane pixels read guard data and
  // are never stored.
  const int rho_base = row0 + yb - off + nh - 1;
  const long long row_step = (long long)B * span;  // one cell row down the LUT
  int4 next = r_lo < r_hi ? __ldg(runs + r_lo) : make_int4(0, 0, 0, 0);
  for (int ri = r_lo; ri < r_hi; ++ri) {
    const int4 run = next;  // (c_x, c_y start, steps, dense offset)
    if (ri + 1 < r_hi) next = __ldg(runs + ri + 1);  // one run ahead
    const int cx = run.x, cy_s = run.y, n_steps = run.z;
    const float* ws = s_w + (run.w - w_lo);
    const float2* rp = lut + (x0 - off - B * cx + nh - 1) + (long long)(rho_base - B * cy_s) * span;
    // ring slot (t mod S) holds diagonal t: LUT row rho0 + B t
    float2 ring[S][PX];
    {
      const float2* rt = rp - D * row_step;
#pragma unroll
      for (int t = -D; t < R; ++t) {
        WCGH_LUT_IN(rt);
#pragma unroll
        for (int i = 0; i < PX; ++i) ring[(t + S) % S][i] = __ldg(rt + 32 * i);
        rt += row_step;
      }
    }
    // prefetch pointer: diagonal -(D + 1), then one row lower per step
    const float2* pf = rp - (D + 1) * row_step;
    // one step: MAC the listed weight (zero in gaps), then refill the dead slot
#define WCGH_LUT_STEP(uu, u) WCGH_LUT_STEP_W(uu, ws[u])
#define WCGH_LUT_STEP_W(uu, wexpr)                                              \
  {                                                                             \
    const float wv = (wexpr);                                                   \
    if (wv != 0.f) {                                                            \
      _Pragma("unroll") for (int j = 0; j < R; ++j)                             \
      _Pragma("unroll") for (int i = 0; i < PX; ++i) {                          \
        acc[j][i] = ffma2(wv, ring[(j - (uu) + 2 * S) % S][i], acc[j][i]);      \
      }                                                                         \
    }                                                                           \
    WCGH_LUT_IN(pf);                                                            \
    _Pragma("unroll") for (int i = 0; i < PX; ++i)                              \
      ring[(R - 1 - (uu) + S) % S][i] = __ldg(pf + 32 * i);                     \
    pf -= row_step;                                                             \
  }
    const int full = n_steps - n_steps % S;
    for (int ub = 0; ub < full; ub += S) {
#pragma unroll
      for (int uu = 0; uu < S; ++uu) WCGH_LUT_STEP(uu, ub + uu)
    }
    // remainder (< S steps): weights read up front (the shared array has
    // >= 32 slack slots past the chunk's last run), one uniform branch per step
    const int rem = n_steps - full;
    if (rem > 0) {
      float wt[S - 1];
#pragma unroll
      for (int k = 0; k < S - 1; ++k) wt[k] = ws[full + k];
      // ptxas if-converts a straight-line remainder block (each step guarded
      // by uu < rem), so a block costs all its step slots whatever rem is:
      // three blocks of 1/3, 2/3 and all of the S - 1 slots keep the
      // predicated-off slots under a third of the block (config 2 K4 29.73 ->
      // 29.39 ms; one block per remainder length via a jump table measured
      // the same, 29.39 ms, at twice the code).
      constexpr int T1 = (S - 1) / 3, T2 = 2 * (S - 1) / 3;
      if (rem <= T1) {
#pragma unroll
        for (int uu = 0; uu < T1; ++uu) {
          if (uu < rem) WCGH_LUT_STEP_W(uu, wt[uu])
        }
      } else if (rem <= T2) {
#pragma unroll
        for (int uu = 0; uu < T2; ++uu) {
          if (uu < rem) WCGH_LUT_STEP_W(uu, wt[uu])
        }
      } else {
#pragma unroll
        for (int uu = 0; uu < S - 1; ++uu) {
          if (uu < rem) WCGH_LUT_STEP_W(uu, wt[uu])
        }
      }
    }
#undef WCGH_LUT_STEP_W
#undef WCGH_LUT_STEP
  }

#undef WCGH_LUT_IN
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int row = yb + j * B;
    if (row < rows) {
      float2* dst = out + size_t(blockIdx.y) * out_stride + size_t(row) * nh;
#pragma unroll
      for (int i = 0; i < PX; ++i) {
        const int x = x0 + 32 * i;
        WCGH_DCHECK(size_t(blockIdx.y) * out_stride + size_t(row) * nh + x < size_t(gridDim.y) * out_stride ||
                    x >= nh);
        if (x < nh) dst[x] = acc[j][i];
      }
    }
  }
}

// One chunk of a stage's run list as a kernel parameter block (the default
// K4 form). The weights then come from the constant bank through uniform
// registers (LDCU), and an FFMA2 whose scalar operand is a uniform register
// reads only its two register pairs: one even and one odd register each, so
// it issues at the pipe rate. With the weight in a regular register (the
// shared-memory form above) the third read conflicts in the register banks
// whenever the operand-reuse cache misses: tools/microbench_operands.cu
// measures 125-127 lane-FMA/clk/SM for the uniform/constant operand against
// 110-111 for the register operand (128 = the FP32 pipe).
//   d[2i]     = c_x | c_y << 16      (run i: cell column, first cell row)
//   d[2i + 1] = steps | woff << 16   (its step count, first weight at d[w_base + woff])
//   d[w_base ...] = the dense per-step weights (zeros in gaps), then >= S zeros.
constexpr int kChunkInts = 8160;
struct LutChunk {
  int n_runs;
  int w_base;
  int d[kChunkInts];
};
static_assert(sizeof(LutChunk) + 64 <= 32764, "kernel parameter space");

template <int B, int R, int PX, int D, int W>
__global__ void __launch_bounds__(W * 32, lut_min_blocks(R, PX, D, W))
    k_lut_chunk(const float2* __restrict__ lut, int nh, int off, int row0, int rows, int tiles_x,
                float2* __restrict__ out, const __grid_constant__ LutChunk ck) {
  constexpr int S = R + D;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx = blockIdx.x % tiles_x, tyc = blockIdx.x / tiles_x;
  const int r = tyc % B;
  const int g = (tyc / B) * W + warp;
  const int yb = g * (B * R) + r;
  const int x0 = tx * (32 * PX) + lane;
  const int span = 2 * nh - 1;
#ifdef WCGH_CHECKED
  const float2* lut_lo = lut - size_t(kLutGuardBefore) * span;
  const float2* lut_hi = lut + size_t(span + kLutGuardAfter) * span + kLutPadCols;
#define WCGH_LUT_IN(ptr) WCGH_DCHECK((ptr) >= lut_lo && (ptr) + 32 * (PX - 1) < lut_hi)
#else
#define WCGH_LUT_IN(ptr)
#endif
  float2 acc[R][PX];
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int i = 0; i < PX; ++i) acc[j][i] = make_float2(0.f, 0.f);

  const int rho_base = row0 + yb - off + nh - 1;
  const long long row_step = (long long)B * span;
  for (int ri = 0; ri < ck.n_runs; ++ri) {
    const unsigned rx = unsigned(ck.d[2 * ri]), ry = unsigned(ck.d[2 * ri + 1]);
    const int cx = int(rx & 0xffffu), cy_s = int(rx >> 16), n_steps = int(ry & 0xffffu);
    const int wo = ck.w_base + int(ry >> 16);
    WCGH_DCHECK(wo + n_steps + S - 1 <= kChunkInts);
    const float2* rp = lut + (x0 - off - B * cx + nh - 1) + (long long)(rho_base - B * cy_s) * span;
    float2 ring[S][PX];
    {
      const float2* rt = rp - D * row_step;
#pragma unroll
      for (int t = -D; t < R; ++t) {
        WCGH_LUT_IN(rt);
#pragma unroll
        for (int i = 0; i < PX; ++i) ring[(t + S) % S][i] = __ldg(rt + 32 * i);
        rt += row_step;
      }
    }
    const float2* pf = rp - (D + 1) * row_step;
    // one step: MAC the listed weight (zeros in gaps are multiplied, not
    // predicated: a predicated-off FFMA2 occupies the pipe all the same, and
    // the predicate would need the weight in a regular register)
#define WCGH_LUT_STEP_W(uu, wexpr)                                              \
  {                                                                             \
    const float wv = (wexpr);                                                   \
    _Pragma("unroll") for (int j = 0; j < R; ++j)                               \
    _Pragma("unroll") for (int i = 0; i < PX; ++i) {                            \
      acc[j][i] = ffma2(wv, ring[(j - (uu) + 2 * S) % S][i], acc[j][i]);        \
    }                                                                           \
    WCGH_LUT_IN(pf);                                                            \
    _Pragma("unroll") for (int i = 0; i < PX; ++i)                              \
      ring[(R - 1 - (uu) + S) % S][i] = __ldg(pf + 32 * i);                     \
    pf -= row_step;                                                             \
  }
    const int full = n_steps - n_steps % S;
    for (int ub = 0; ub < full; ub += S) {
#pragma unroll
      for (int uu = 0; uu < S; ++uu) WCGH_LUT_STEP_W(uu, __int_as_float(ck.d[wo + ub + uu]))
    }
    const int rem = n_steps - full;
    if (rem > 0) {
      // the parameter block holds >= S zero weights past its last run
      constexpr int T1 = (S - 1) / 3, T2 = 2 * (S - 1) / 3;
      const int wr = wo + full;
      if (rem <= T1) {
#pragma unroll
        for (int uu = 0; uu < T1; ++uu) {
          if (uu < rem) WCGH_LUT_STEP_W(uu, __int_as_float(ck.d[wr + uu]))
        }
      } else if (rem <= T2) {
#pragma unroll
        for (int uu = 0; uu < T2; ++uu) {
          if (uu < rem) WCGH_LUT_STEP_W(uu, __int_as_float(ck.d[wr + uu]))
        }
      } else {
#pragma unroll
        for (int uu = 0; uu < S - 1; ++uu) {
          if (uu < rem) WCGH_LUT_STEP_W(uu, __int_as_float(ck.d[wr + uu]))
        }
      }
    }
#undef WCGH_LUT_STEP_W
  }
#undef WCGH_LUT_IN
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int row = yb + j * B;
    if (row < rows) {
      float2* dst = out + size_t(row) * nh;
#pragma unroll
      for (int i = 0; i < PX; ++i) {
        const int x = x0 + 32 * i;
        if (x < nh) dst[x] = acc[j][i];
      }
    }
  }
}

// out (+)= sum of `n` partial planes in order, fp64 accumulation. rotate:
// out += i * sum (imaginary LUT weights of a complex object).
__global__ void k_reduce_partials(const float2* __restrict__ partial, int n, size_t count,
                                  int accumulate, int rotate, float2* __restrict__ out) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double re = 0.0, im = 0.0;
  if (rotate) {
    for (int c = 0; c < n; ++c) {
      const float2 v = partial[size_t(c) * count + i];
      re += v.x;
      im += v.y;
    }
    out[i] = make_float2(float(double(out[i].x) - im), float(double(out[i].y) + re));
    return;
  }
  if (accumulate) {
    re = out[i].x;
    im = out[i].y;
  }
  for (int c = 0; c < n; ++c) {
    const float2 v = partial[size_t(c) * count + i];
    re += v.x;
    im += v.y;
  }
  out[i] = make_float2(float(re), float(im));
}

constexpr int kMaxChunkSteps = 4096;

// Register-window shape: R rows x PX columns per thread, D rows of prefetch,
// W warps per CTA. Default 16 x 2 x 2 x 4 (168 registers, 12 warps/SM: one
// LUT row segment feeds 32 FFMA2s, half the loads per MAC of the 8-row window;
// config 2 K4 26.86 -> 25.14 ms, profiles/s5_k4_chunk_sweep.md);
// WCGH_LUT_VARIANT="R,PX,D,W" selects another compiled shape (tuning only;
// results equal up to fp32 rounding).
struct LutVariant {
  int R, PX, D, W;
};
LutVariant lut_variant() {
  static const LutVariant v = [] {
    LutVariant d{16, 2, 2, 4};
    if (const char* e = std::getenv("WCGH_LUT_VARIANT"); e && *e) {
      int r = 0, px = 0, dd = 0, w = 4;
      const int got = std::sscanf(e, "%d,%d,%d,%d", &r, &px, &dd, &w);
      if (got >= 3) d = LutVariant{r, px, dd, w};
    }
    return d;
  }();
  return v;
}
// Largest gap (in cell rows) a run steps through with zero weights; a wider
// gap starts a new run (window reload). WCGH_LUT_GAP overrides (tuning).
int lut_gap() {
  static const int g = std::max(1, env_int("WCGH_LUT_GAP", std::min(4, lut_variant().R)));
  return g;
}
int lut_chunk_target() {
  static const int t = std::max(1, env_int("WCGH_LUT_CHUNKS", 8));
  return t;
}

template <int B, int R, int PX, int D, int W>
void launch_stage_v(const float2* lut, int nh, const StageCells& sc, int off, int row0, int rows,
                    int tiles_x, dim3 grid, int chunk0, int chunk_steps, float2* out,
                    size_t stride, cudaStream_t s) {
  const size_t smem = sizeof(float) * size_t(chunk_steps + sc.m + 32);
  k_lut_stage<B, R, PX, D, W><<<grid, W * 32, smem, s>>>(
      lut, nh, sc.runs.as<int4>(), sc.n_runs, sc.dense.as<float>(), off, row0, rows, tiles_x,
      chunk0, chunk_steps, out, stride);
}

template <int B>
void launch_stage_b(const LutVariant& v, const float2* lut, int nh, const StageCells& sc, int off,
                    int row0, int rows, int tiles_x, dim3 grid, int chunk0, int chunk_steps,
                    float2* out, size_t stride, cudaStream_t s) {
#define WCGH_V(R_, PX_, D_, W_)                                                             \
  if (v.R == R_ && v.PX == PX_ && v.D == D_ && v.W == W_) {                                 \
    launch_stage_v<B, R_, PX_, D_, W_>(lut, nh, sc, off, row0, rows, tiles_x, grid, chunk0, \
                                       chunk_steps, out, stride, s);                        \
    return;                                                                                 \
  }
  WCGH_V(8, 2, 2, 4)
  WCGH_V(8, 2, 1, 4)
  WCGH_V(8, 2, 3, 4)
  WCGH_V(8, 2, 4, 4)
  WCGH_V(8, 2, 2, 8)
  WCGH_V(8, 4, 2, 4)
  WCGH_V(16, 2, 2, 4)
#undef WCGH_V
  throw ValidationError("WCGH_LUT_VARIANT: shape not compiled");
}

template <int B, int R, int PX, int D, int W>
void launch_chunk_v(const float2* lut, int nh, int off, int row0, int rows, int tiles_x, int grid,
                    float2* out, const LutChunk& ck, cudaStream_t s) {
  k_lut_chunk<B, R, PX, D, W><<<grid, W * 32, 0, s>>>(lut, nh, off, row0, rows, tiles_x, out, ck);
}

template <int B>
void launch_chunk_b(const LutVariant& v, const float2* lut, int nh, int off, int row0, int rows,
                    int tiles_x, int grid, float2* out, const LutChunk& ck, cudaStream_t s) {
#define WCGH_V(R_, PX_, D_, W_)                                                                \
  if (v.R == R_ && v.PX == PX_ && v.D == D_ && v.W == W_) {                                    \
    launch_chunk_v<B, R_, PX_, D_, W_>(lut, nh, off, row0, rows, tiles_x, grid, out, ck, s);   \
    return;                                                                                    \
  }
  WCGH_V(8, 2, 2, 4)
  WCGH_V(8, 2, 1, 4)
  WCGH_V(8, 2, 3, 4)
  WCGH_V(16, 2, 2, 4)
#ifdef WCGH_LUT_SWEEP
  WCGH_V(16, 2, 1, 4)
  WCGH_V(16, 2, 3, 4)
  WCGH_V(12, 2, 2, 4)
  WCGH_V(16, 1, 2, 4)
  WCGH_V(16, 2, 2, 2)
  WCGH_V(24, 1, 2, 2)
  WCGH_V(32, 1, 2, 2)
  WCGH_V(24, 2, 2, 2)
  WCGH_V(20, 2, 2, 2)
#endif
#undef WCGH_V
  throw ValidationError("WCGH_LUT_VARIANT: shape not compiled for the chunk kernel");
}

// K4 form: 1 = run-list chunks as kernel parameter blocks (default), 0 = the
// shared-memory form (weights staged per CTA, predicated zero steps).
bool lut_params() {
  static const bool p = env_int("WCGH_LUT_PARAMS", 1) != 0;
  return p;
}

// Side streams the chunk launches of one stage are spread over, so that a
// launch's last partial wave overlaps the next launch (per host thread and
// device; created once).
constexpr int kSideStreams = 4;
struct SideStreams {
  int dev = -1;
  cudaStream_t st[kSideStreams];
  cudaEvent_t fork, join[kSideStreams];
};
SideStreams& side_streams() {
  thread_local std::vector<std::unique_ptr<SideStreams>> pools;
  int dev = 0;
  WCGH_CUDA(cudaGetDevice(&dev));
  for (auto& p : pools)
    if (p->dev == dev) return *p;
  auto p = std::make_unique<SideStreams>();
  p->dev = dev;
  for (int k = 0; k < kSideStreams; ++k) {
    WCGH_CUDA(cudaStreamCreateWithFlags(&p->st[k], cudaStreamNonBlocking));
    WCGH_CUDA(cudaEventCreateWithFlags(&p->join[k], cudaEventDisableTiming));
  }
  WCGH_CUDA(cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming));
  pools.push_back(std::move(p));
  return *pools.back();
}

// Splits a stage's run list into parameter blocks, in list order. A chunk
// closes once it holds `target` weights (so a stage has >= kMinChunks chunks
// to spread over the side streams) or when the next record would not fit;
// a run longer than the room left is split (its remainder restarts the
// window at the next cell row). Depends on the run list only, never on the
// row band, so the partial planes and their reduction are band-invariant.
constexpr int kMinChunks = 4;
void build_chunks(const StageCells& sc, int S, std::vector<LutChunk>& out) {
  out.clear();
  const int cap = kChunkInts - S;  // records + weights (S zero weights of slack after)
  const int target =
      std::min(cap, std::max(16 * S, (sc.n_dense + kMinChunks - 1) / kMinChunks));
  std::vector<int> recs;
  std::vector<float> ws;
  auto flush = [&] {
    if (recs.empty()) return;
    out.emplace_back();
    LutChunk& c = out.back();
    const int nr = int(recs.size() / 2);
    c.n_runs = nr;
    c.w_base = 2 * nr;
    std::copy(recs.begin(), recs.end(), c.d);
    std::memcpy(c.d + c.w_base, ws.data(), ws.size() * sizeof(float));
    std::fill(c.d + c.w_base + ws.size(), c.d + kChunkInts, 0);
    recs.clear();
    ws.clear();
  };
  for (int i = 0; i < sc.n_runs; ++i) {
    const int4 run = sc.h_runs[size_t(i)];
    int cy = run.y, n = run.z;
    size_t wofs = size_t(run.w);
    require(run.x < 65536 && cy + n <= 65536, "LUT superposition: cell grid too large");
    while (n > 0) {
      if (int(ws.size()) >= target) flush();
      const int room = cap - int(recs.size()) - 2 - int(ws.size());
      if (room < std::min(n, S) && !recs.empty()) {
        flush();
        continue;
      }
      const int take = std::min(n, room);
      recs.push_back(run.x | (cy << 16));
      recs.push_back(take | (int(ws.size()) << 16));
      ws.insert(ws.end(), sc.h_dense.begin() + wofs, sc.h_dense.begin() + wofs + take);
      cy += take;
      wofs += size_t(take);
      n -= take;
    }
  }
  flush();
}

int launch_lut_chunks(const float2* lut, int nh, int block, const StageCells& sc, int off,
                      int row0, int rows, float2* out, DevBuf& partial, cudaStream_t s,
                      DirectTiming* timing, bool accumulate, bool rotate) {
  const LutVariant v = lut_variant();
  thread_local std::vector<LutChunk> chunks;
  build_chunks(sc, v.R + v.D, chunks);
  const size_t band = size_t(rows) * nh;
  const int n_chunks = int(chunks.size());
  const int group = partial_group(n_chunks, nh);
  float2* part = static_cast<float2*>(partial.reserve(band * group * sizeof(float2)));
  const int tiles_x = (nh + 32 * v.PX - 1) / (32 * v.PX);
  const int groups = (rows + block * v.R - 1) / (block * v.R);
  const int tiles_y = block * ((groups + v.W - 1) / v.W);
  const int grid = tiles_x * tiles_y;
  SideStreams& ss = side_streams();
  int launches = 0;
  for (int g0 = 0; g0 < n_chunks; g0 += group) {
    const int ng = std::min(group, n_chunks - g0);
    const int nside = std::min(ng, kSideStreams);
    if (timing) WCGH_CUDA(cudaEventRecord(timing->begin(), s));
    WCGH_CUDA(cudaEventRecord(ss.fork, s));
    for (int k = 0; k < nside; ++k) WCGH_CUDA(cudaStreamWaitEvent(ss.st[k], ss.fork, 0));
    for (int c = 0; c < ng; ++c) {
      cudaStream_t sk = ss.st[c % nside];
      float2* o = part + band * size_t(c);
      const LutChunk& ck = chunks[size_t(g0 + c)];
      switch (block) {
        case 1: launch_chunk_b<1>(v, lut, nh, off, row0, rows, tiles_x, grid, o, ck, sk); break;
        case 2: launch_chunk_b<2>(v, lut, nh, off, row0, rows, tiles_x, grid, o, ck, sk); break;
        case 4: launch_chunk_b<4>(v, lut, nh, off, row0, rows, tiles_x, grid, o, ck, sk); break;
        case 8: launch_chunk_b<8>(v, lut, nh, off, row0, rows, tiles_x, grid, o, ck, sk); break;
        default: throw ValidationError("LUT superposition: unsupported block size");
      }
      WCGH_CHECK_LAUNCH();
    }
    for (int k = 0; k < nside; ++k) {
      WCGH_CUDA(cudaEventRecord(ss.join[k], ss.st[k]));
      WCGH_CUDA(cudaStreamWaitEvent(s, ss.join[k], 0));
    }
    if (timing) {
      WCGH_CUDA(cudaEventRecord(timing->end(), s));
      timing->extra += ng - 1;
    }
    k_reduce_partials<<<unsigned((band + 255) / 256), 256, 0, s>>>(part, ng, band,
                                                                  accumulate || g0 > 0, rotate, out);
    WCGH_CHECK_LAUNCH();
    launches += ng + 1;
  }
  return launches;
}

}  // namespace

int launch_build_lut(const wcgh_layer& scene, int n, int block, float2* lut, DevBuf& scratch,
                     cudaStream_t s) {
  require(block == 1 || block == 2 || block == 4 || block == 8,
          "build_block_lut: unsupported block size " + std::to_string(block));
  require(block <= n, "build_block_lut: block size exceeds plane size");
  const int span = 2 * n - 1;
  const int ext = span + block - 1;
  const int lo = -(n - 1) - (block - 1);
  double2* base = static_cast<double2*>(scratch.reserve(sizeof(double2) * size_t(ext) * ext));
  const size_t ne = size_t(ext) * ext, ns = size_t(span) * span;
  k_point_grid<<<unsigned((ne + 255) / 256), 256, 0, s>>>(scene.wavelength, scene.pitch, scene.z,
                                                           ext, lo, base);
  WCGH_CHECK_LAUNCH();
  k_box_sum<<<unsigned((ns + 255) / 256), 256, 0, s>>>(base, ext, span, block, lut);
  WCGH_CHECK_LAUNCH();
  return 2;
}

int launch_stage_cells(const float* w, int m, StageCells& sc, cudaStream_t s) {
  sc.m = m;
  sc.host_valid = false;
  int* c = static_cast<int*>(sc.counts.reserve(sizeof(int) * 3 * (size_t(m) + 1)));
  int* o = static_cast<int*>(sc.offsets.reserve(sizeof(int) * 3 * (size_t(m) + 1)));
  const size_t mm = size_t(m) * m;
  sc.runs.reserve(sizeof(int4) * (mm + 1));
  sc.dense.reserve(sizeof(float) * (mm + 1));
  WCGH_CUDA(cudaMemsetAsync(sc.dense.p, 0, sizeof(float) * (mm + 1), s));
  const unsigned g = unsigned((m + 7) / 8);
  const int R = lut_gap();
  sc.gap = R;
  k_runs_count<<<g, 256, 0, s>>>(w, m, R, c, c + (m + 1), c + 2 * (m + 1));
  WCGH_CHECK_LAUNCH();
  for (int k = 0; k < 3; ++k) launch_scan(c + k * (m + 1), o + k * (m + 1), m, s);
  k_runs_fill<<<g, 256, 0, s>>>(w, m, R, o, o + (m + 1), sc.runs.as<int4>(), sc.dense.as<float>());
  WCGH_CHECK_LAUNCH();
  return 5;
}

void stage_cells_totals_async(const StageCells& sc, int* host3, cudaStream_t s) {
  const int m = sc.m;
  const int* o = sc.offsets.as<int>();
  for (int k = 0; k < 3; ++k)
    WCGH_CUDA(cudaMemcpyAsync(host3 + k, o + k * (m + 1) + m, sizeof(int), cudaMemcpyDeviceToHost, s));
}

void stage_cells_fetch(StageCells& sc, cudaStream_t s) {
  sc.h_runs.resize(size_t(sc.n_runs));
  sc.h_dense.resize(size_t(sc.n_dense));
  if (sc.n_runs > 0) {
    WCGH_CUDA(cudaMemcpyAsync(sc.h_runs.data(), sc.runs.p, sizeof(int4) * size_t(sc.n_runs),
                              cudaMemcpyDeviceToHost, s));
    WCGH_CUDA(cudaMemcpyAsync(sc.h_dense.data(), sc.dense.p, sizeof(float) * size_t(sc.n_dense),
                              cudaMemcpyDeviceToHost, s));
  }
  WCGH_CUDA(cudaStreamSynchronize(s));
  sc.host_valid = true;
}

int launch_lut_stage(const float2* lut, int nh, int block, StageCells& sc, int off, int row0,
                     int rows, float2* out, DevBuf& partial, cudaStream_t s, DirectTiming* timing,
                     bool accumulate, bool rotate) {
  const size_t band = size_t(rows) * nh;
  require(!rotate || accumulate, "LUT superposition: a rotated stage accumulates");
  if (sc.n_runs == 0) {
    if (!accumulate) WCGH_CUDA(cudaMemsetAsync(out, 0, band * sizeof(float2), s));
    return 0;
  }
  // chunk size depends on the stage's step count only (never on the row band)
  const LutVariant v = lut_variant();
  require(sc.gap >= 1, "LUT superposition: run lists not built");
  require(block * v.R * v.W <= kLutGuardAfter - 16 && block * (v.D + 1) + 1 <= kLutGuardBefore,
          "LUT superposition: window shape exceeds the LUT guard rows");
  if (lut_params()) {
    if (!sc.host_valid) stage_cells_fetch(sc, s);
    return launch_lut_chunks(lut, nh, block, sc, off, row0, rows, out, partial, s, timing,
                             accumulate, rotate);
  }
  const int target = lut_chunk_target();
  int chunk_steps = std::min(kMaxChunkSteps, std::max(256, (sc.n_dense + target - 1) / target));
  chunk_steps = (chunk_steps + 127) / 128 * 128;
  const int n_chunks = (sc.n_dense + chunk_steps - 1) / chunk_steps;
  const int group = partial_group(n_chunks, nh);
  float2* part = static_cast<float2*>(partial.reserve(band * group * sizeof(float2)));
  const int tiles_x = (nh + 32 * v.PX - 1) / (32 * v.PX);
  const int groups = (rows + block * v.R - 1) / (block * v.R);  // per row residue
  const int tiles_y = block * ((groups + v.W - 1) / v.W);
  int launches = 0;
  for (int g0 = 0; g0 < n_chunks; g0 += group) {
    const int ng = std::min(group, n_chunks - g0);
    dim3 grid(unsigned(tiles_x * tiles_y), unsigned(ng));
    if (timing) WCGH_CUDA(cudaEventRecord(timing->begin(), s));
    switch (block) {
      case 1: launch_stage_b<1>(v, lut, nh, sc, off, row0, rows, tiles_x, grid, g0, chunk_steps, part, band, s); break;
      case 2: launch_stage_b<2>(v, lut, nh, sc, off, row0, rows, tiles_x, grid, g0, chunk_steps, part, band, s); break;
      case 4: launch_stage_b<4>(v, lut, nh, sc, off, row0, rows, tiles_x, grid, g0, chunk_steps, part, band, s); break;
      case 8: launch_stage_b<8>(v, lut, nh, sc, off, row0, rows, tiles_x, grid, g0, chunk_steps, part, band, s); break;
      default: throw ValidationError("LUT superposition: unsupported block size");
    }
    WCGH_CHECK_LAUNCH();
    if (timing) WCGH_CUDA(cudaEventRecord(timing->end(), s));
    k_reduce_partials<<<unsigned((band + 255) / 256), 256, 0, s>>>(part, ng, band,
                                                                  accumulate || g0 > 0, rotate, out);
    WCGH_CHECK_LAUNCH();
    launches += 2;
  }
  return launches;
}

int launch_lut_dense(const float2* lut, int nh, int block, const float* w, int m, int off,
                     int row0, int rows, float2* out, StageCells& sc, DevBuf& partial,
                     cudaStream_t s, long long* nnz_out, bool accumulate, bool rotate) {
  int launches = launch_stage_cells(w, m, sc, s);
  int tot[3];
  stage_cells_totals_async(sc, tot, s);
  WCGH_CUDA(cudaStreamSynchronize(s));
  sc.n_runs = tot[0];
  sc.n_dense = tot[1];
  sc.nnz = tot[2];
  if (nnz_out) *nnz_out = sc.nnz;
  return launches + launch_lut_stage(lut, nh, block, sc, off, row0, rows, out, partial, s, nullptr,
                                    accumulate || rotate, rotate);
}

}  // namespace wcgh

WCGH_CHK_TU(wcgh_lut)
