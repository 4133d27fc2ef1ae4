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
//     32 (a CTA of 8 warps covers 8R rows x 32PX columns);
//   * for cell (c_x, c_y) pixel row j reads LUT row y_j - a_y, and
//     (y_j + B) - (a_y + B) is the same row: stepping c_y -> c_y + 1 shifts
//     the R-row register window by one, so each step loads one new LUT row
//     segment (PX samples) and performs R*PX complex-by-real MACs (2 FFMA each);
//   * runs of cells closer than R rows are stepped through; longer gaps
//     restart the window.
// Cells are split into fixed chunks of the column-major list; each
// (tile, chunk) CTA writes a partial plane and a fixed-order reduction sums
// them, so the result does not depend on the launch or the row-band split.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
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

// Column-major compaction of a dense m x m weight grid: one warp per cell
// column, ascending c_y, nonzero weights only.
__global__ void k_col_counts(const float* __restrict__ w, int m, int* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int cx = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (cx >= m) return;
  int c = 0;
  for (int cy = lane; cy < m; cy += 32) c += w[size_t(cy) * m + cx] != 0.0f;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  if (lane == 0) cnt[cx] = c;
}

__global__ void k_col_fill(const float* __restrict__ w, int m, const int* __restrict__ off,
                           int2* __restrict__ ent) {
  const int lane = threadIdx.x & 31;
  const int cx = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (cx >= m) return;
  int pos = off[cx];
  for (int base = 0; base < m; base += 32) {
    const int cy = base + lane;
    const float v = cy < m ? w[size_t(cy) * m + cx] : 0.0f;
    const unsigned b = __ballot_sync(kFull, v != 0.0f);
    if (v != 0.0f) ent[pos + __popc(b & ((1u << lane) - 1u))] = make_int2(cy, __float_as_int(v));
    pos += __popc(b);
  }
}

constexpr int kThreads = 256;

// Dynamic shared memory: the chunk's column-major entries (cy, w bits).
template <int B, int R, int PX, int D>
__global__ void __launch_bounds__(kThreads, 2)
    k_lut_stage(const float2* __restrict__ lut, int nh, const int* __restrict__ col_off,
                const int2* __restrict__ ent, int m, int off, int row0, int rows, int tiles_x,
                int chunk0, int chunk_entries, int nnz, float2* __restrict__ out,
                size_t out_stride) {
  extern __shared__ int2 s_ent[];
  constexpr int BW = B < 8 ? B : 8;  // row residues spread over the 8 warps
  constexpr int S = R + D;           // ring: R live diagonals + D prefetched
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = warp % BW, q = warp / BW;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int yb = ty * (8 * R) + q * (R * B) + r;  // band row of pixel row j = 0
  const int x0 = tx * (32 * PX) + lane;
  const int span = 2 * nh - 1;
  const int e_lo = (chunk0 + blockIdx.y) * chunk_entries;
  const int e_hi = min(e_lo + chunk_entries, nnz);

  float2 acc[R][PX];
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int i = 0; i < PX; ++i) acc[j][i] = make_float2(0.f, 0.f);

  for (int e = e_lo + threadIdx.x; e < e_hi; e += kThreads) s_ent[e - e_lo] = __ldg(ent + e);
  __syncthreads();

  if (e_lo < e_hi) {
    // first cell column of the chunk: col_off[cx] <= e_lo < col_off[cx + 1]
    int lo = 0, hi = m;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(col_off + mid) <= e_lo) lo = mid; else hi = mid;
    }
    // LUT row of pixel row j at cell row cy: (row0 + yb + jB) - off - B cy + nh - 1.
    // `lut` points into a guarded allocation (kLutGuardRows rows before and
    // after, kLutPadCols elements of tail padding), so the window and the
    // prefetch never need clamping; out-of-plane pixels read guard data and
    // are never stored.
    const int rho_base = row0 + yb - off + nh - 1;
    const long long row_step = (long long)B * span;  // one cell row down the LUT
    int ce_prev = __ldg(col_off + lo);
    for (int cx = lo; cx < m; ++cx) {
      const int ce_abs = __ldg(col_off + cx + 1);
      const int cb = max(ce_prev, e_lo) - e_lo;
      const int ce = min(ce_abs, e_hi) - e_lo;
      ce_prev = ce_abs;
      if (cb >= e_hi - e_lo) break;
      if (cb >= ce) continue;
      const float2* cp = lut + (x0 - off - B * cx + nh - 1);  // this thread's column 0
      int k = cb;
      while (k < ce) {
        // run: entries k..k_end-1 whose consecutive cy gaps are <= R
        int k_end = k + 1;
        int cy_prev = s_ent[k].x;
        while (k_end < ce) {
          const int cy_n = s_ent[k_end].x;
          if (cy_n - cy_prev > R) break;
          cy_prev = cy_n;
          ++k_end;
        }
        const int cy_s = s_ent[k].x;
        const int n_steps = cy_prev - cy_s + 1;
        // ring slot (t mod S) holds diagonal t: LUT row rho0 + B t
        const float2* rp = cp + (long long)(rho_base - B * cy_s) * span;
        float2 ring[S][PX];
        {
          const float2* rt = rp - D * row_step;
#pragma unroll
          for (int t = -D; t < R; ++t) {
#pragma unroll
            for (int i = 0; i < PX; ++i) ring[(t + S) % S][i] = __ldg(rt + 32 * i);
            rt += row_step;
          }
        }
        // prefetch pointer: diagonal -(D + 1), then one row lower per step
        const float2* pf = rp - (D + 1) * row_step;
        int2 nx = s_ent[k];
        int cy = cy_s;
        const int full = n_steps - n_steps % S;
        // one step: MAC if cell (cx, cy) is listed, then refill the dead slot
#define WCGH_LUT_STEP(uu)                                                          \
  {                                                                                \
    if (nx.x == cy) {                                                              \
      const float wv = __int_as_float(nx.y);                                       \
      ++k;                                                                         \
      nx = k < k_end ? s_ent[k] : make_int2(-1, 0);                                \
      _Pragma("unroll") for (int j = 0; j < R; ++j)                                \
      _Pragma("unroll") for (int i = 0; i < PX; ++i) {                             \
        const float2 v = ring[(j - (uu) + 2 * S) % S][i];                          \
        acc[j][i].x = fmaf(wv, v.x, acc[j][i].x);                                  \
        acc[j][i].y = fmaf(wv, v.y, acc[j][i].y);                                  \
      }                                                                            \
    }                                                                              \
    _Pragma("unroll") for (int i = 0; i < PX; ++i)                                 \
      ring[(R - 1 - (uu) + S) % S][i] = __ldg(pf + 32 * i);                        \
    pf -= row_step;                                                                \
    ++cy;                                                                          \
  }
        for (int ub = 0; ub < full; ub += S) {
#pragma unroll
          for (int uu = 0; uu < S; ++uu) WCGH_LUT_STEP(uu)
        }
#pragma unroll
        for (int uu = 0; uu < S - 1; ++uu) {
          if (full + uu < n_steps) WCGH_LUT_STEP(uu)
        }
#undef WCGH_LUT_STEP
        k = k_end;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int row = yb + j * B;
    if (row < rows) {
      float2* dst = out + size_t(blockIdx.y) * out_stride + size_t(row) * nh;
#pragma unroll
      for (int i = 0; i < PX; ++i) {
        const int x = x0 + 32 * i;
        if (x < nh) dst[x] = acc[j][i];
      }
    }
  }
}

// out (+)= sum of `n` partial planes in order, fp64 accumulation.
__global__ void k_reduce_partials(const float2* __restrict__ partial, int n, size_t count,
                                  int accumulate, float2* __restrict__ out) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double re = 0.0, im = 0.0;
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

constexpr int kR = 8, kPX = 2, kD = 2;
constexpr int kMaxChunkEntries = 4096;
constexpr size_t kPartialBytes = 2ull << 30;

template <int B>
void launch_stage_b(const float2* lut, int nh, const int* col_off, const int2* ent, int m,
                    int off, int row0, int rows, int tiles_x, dim3 grid, int chunk0,
                    int chunk_entries, int nnz, float2* out, size_t stride, cudaStream_t s) {
  k_lut_stage<B, kR, kPX, kD><<<grid, kThreads, sizeof(int2) * chunk_entries, s>>>(
      lut, nh, col_off, ent, m, off, row0, rows, tiles_x, chunk0, chunk_entries, nnz, out, stride);
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
  int* cnt = static_cast<int*>(sc.counts.reserve(sizeof(int) * (size_t(m) + 1)));
  int* off = static_cast<int*>(sc.offsets.reserve(sizeof(int) * (size_t(m) + 1)));
  sc.entries.reserve(sizeof(int2) * size_t(m) * m);
  const unsigned g = unsigned((m + 7) / 8);
  k_col_counts<<<g, 256, 0, s>>>(w, m, cnt);
  WCGH_CHECK_LAUNCH();
  launch_scan(cnt, off, m, s);
  k_col_fill<<<g, 256, 0, s>>>(w, m, off, sc.entries.as<int2>());
  WCGH_CHECK_LAUNCH();
  return 3;
}

int launch_lut_stage(const float2* lut, int nh, int block, const StageCells& sc, int nnz,
                     int off, int row0, int rows, float2* out, DevBuf& partial, cudaStream_t s,
                     DirectTiming* timing) {
  const size_t band = size_t(rows) * nh;
  if (nnz == 0) {
    WCGH_CUDA(cudaMemsetAsync(out, 0, band * sizeof(float2), s));
    return 0;
  }
  // chunk size depends on nnz only (never on the row band): ~48+ chunks
  int chunk_entries = std::min(kMaxChunkEntries, std::max(256, (nnz + 47) / 48));
  chunk_entries = (chunk_entries + 127) / 128 * 128;
  const int n_chunks = (nnz + chunk_entries - 1) / chunk_entries;
  const int group = int(std::max<size_t>(1, std::min<size_t>(n_chunks, kPartialBytes / (band * sizeof(float2)))));
  float2* part = static_cast<float2*>(partial.reserve(band * group * sizeof(float2)));
  const int tiles_x = (nh + 32 * kPX - 1) / (32 * kPX);
  const int tiles_y = (rows + 8 * kR - 1) / (8 * kR);
  const int* col_off = sc.offsets.as<int>();
  const int2* ent = sc.entries.as<int2>();
  int launches = 0;
  for (int g0 = 0; g0 < n_chunks; g0 += group) {
    const int ng = std::min(group, n_chunks - g0);
    dim3 grid(unsigned(tiles_x * tiles_y), unsigned(ng));
    if (timing) WCGH_CUDA(cudaEventRecord(timing->begin(), s));
    switch (block) {
      case 1: launch_stage_b<1>(lut, nh, col_off, ent, sc.m, off, row0, rows, tiles_x, grid, g0, chunk_entries, nnz, part, band, s); break;
      case 2: launch_stage_b<2>(lut, nh, col_off, ent, sc.m, off, row0, rows, tiles_x, grid, g0, chunk_entries, nnz, part, band, s); break;
      case 4: launch_stage_b<4>(lut, nh, col_off, ent, sc.m, off, row0, rows, tiles_x, grid, g0, chunk_entries, nnz, part, band, s); break;
      case 8: launch_stage_b<8>(lut, nh, col_off, ent, sc.m, off, row0, rows, tiles_x, grid, g0, chunk_entries, nnz, part, band, s); break;
      default: throw ValidationError("LUT superposition: unsupported block size");
    }
    WCGH_CHECK_LAUNCH();
    if (timing) WCGH_CUDA(cudaEventRecord(timing->end(), s));
    k_reduce_partials<<<unsigned((band + 255) / 256), 256, 0, s>>>(part, ng, band, g0 > 0, out);
    WCGH_CHECK_LAUNCH();
    launches += 2;
  }
  return launches;
}

int launch_lut_dense(const float2* lut, int nh, int block, const float* w, int m, int off,
                     int row0, int rows, float2* out, StageCells& sc, DevBuf& partial,
                     cudaStream_t s, long long* nnz_out) {
  launch_stage_cells(w, m, sc, s);
  int nnz = 0;
  WCGH_CUDA(cudaMemcpyAsync(&nnz, sc.offsets.as<int>() + m, sizeof(int), cudaMemcpyDeviceToHost, s));
  WCGH_CUDA(cudaStreamSynchronize(s));
  if (nnz_out) *nnz_out = nnz;
  return 4 + launch_lut_stage(lut, nh, block, sc, nnz, off, row0, rows, out, partial, s, nullptr);
}

}  // namespace wcgh
