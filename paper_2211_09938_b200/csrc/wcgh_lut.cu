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
// 55-69): plane(x, y) += w_c * S_B(x - a_x, y - a_y), anchors a = off + B*cell.
// Output-stationary: a CTA owns an 8-row x 32P-column tile; lane l of warp w
// owns pixels (x_b + l + 32 i, y_0 + w). For a cell row c_y and a phase
// phi in [0, 32/B), the cells c_x = phi + (32/B) k all read LUT row
// y - a_y at columns x_i - a_x = const + 32 (i - k): stepping k slides a
// P-sample register window by one, so each 8-byte LUT load feeds P complex
// MACs (2P FFMA) — the fringe tile is reused from registers instead of being
// re-streamed per cell (the reference's hot loop streams 16 B of LUT and
// 16 B of plane per update, synthesis.cpp:33).
#include <cuda_runtime.h>

#include <cmath>

#include "wcgh_internal.cuh"

namespace wcgh {
namespace {

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

__global__ void k_row_nnz(const float* __restrict__ w, int m, int* __restrict__ row_nnz) {
  const int row = blockIdx.x;
  int c = 0;
  for (int x = threadIdx.x; x < m; x += blockDim.x) c += w[size_t(row) * m + x] != 0.0f;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ int s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int k = 0; k < (blockDim.x + 31) / 32; ++k) t += s[k];
    row_nnz[row] = t;
  }
}

constexpr int kThreads = 256;

// One cell-row chunk per blockIdx.y; writes (not accumulates) its partial
// plane so the reduction order is fixed.
template <int P>
__global__ void __launch_bounds__(kThreads, 2)
    k_lut_superpose(const float2* __restrict__ lut, int nh, int block, const float* __restrict__ w,
                    int m, int off, int row0, int rows, int tiles_x, int rows_per_chunk,
                    const int* __restrict__ row_nnz, float2* __restrict__ out,
                    size_t out_chunk_stride) {
  extern __shared__ float w_row[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int tx = blockIdx.x % tiles_x;
  const int ty = blockIdx.x / tiles_x;
  const int row = ty * 8 + warp;
  const int y = row0 + row;
  const int xb = tx * 32 * P + lane;
  const int span = 2 * nh - 1;
  const int steps_per_phase = 32 / block;  // cells per 32 columns
  const int cy0 = blockIdx.y * rows_per_chunk;
  const int cy1 = min(cy0 + rows_per_chunk, m);

  float re[P], im[P];
#pragma unroll
  for (int i = 0; i < P; ++i) re[i] = im[i] = 0.0f;

  for (int cy = cy0; cy < cy1; ++cy) {
    if (row_nnz[cy] == 0) continue;  // uniform across the CTA
    __syncthreads();
    for (int x = threadIdx.x; x < m; x += kThreads) w_row[x] = w[size_t(cy) * m + x];
    __syncthreads();
    const int ay = off + block * cy;
    const int dyi = y - ay + nh - 1;  // LUT row, in [0, span) for valid rows
    const float2* lrow = lut + size_t(min(max(dyi, 0), span - 1)) * span;
    for (int phi = 0; phi < steps_per_phase; ++phi) {
      // cells cx = phi + steps_per_phase * k, k = 0..K-1
      const int K = (m - phi + steps_per_phase - 1) / steps_per_phase;
      if (K <= 0) continue;
      // LUT column of pixel i at step k: x_i - off - B*cx = c0 + 32 (i - k) + (nh - 1)
      const int c0 = xb - off - block * phi + nh - 1;
      // Circular register window: sample j (column c0 + 32 j) lives in slot
      // j mod P; at step k pixel i reads j = i - k, and after the step the
      // slot of j = P-1-k (no longer needed) receives j = -(k+1).
      float2 win[P];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int col = c0 + 32 * i;
        win[i] = (col >= 0 && col < span) ? __ldg(lrow + col) : make_float2(0.f, 0.f);
      }
      for (int kb = 0; kb < K; kb += P) {
#pragma unroll
        for (int kk = 0; kk < P; ++kk) {
          const int k = kb + kk;
          if (k < K) {
            const float wk = w_row[phi + steps_per_phase * k];
            if (wk != 0.0f) {
#pragma unroll
              for (int i = 0; i < P; ++i) {
                const float2 v = win[(i - kk + P) % P];
                re[i] = fmaf(wk, v.x, re[i]);
                im[i] = fmaf(wk, v.y, im[i]);
              }
            }
            const int col = c0 - 32 * (k + 1);
            win[(P - 1 - kk) % P] =
                (col >= 0 && col < span) ? __ldg(lrow + col) : make_float2(0.f, 0.f);
          }
        }
      }
    }
  }
  if (row < rows) {
    float2* dst = out + blockIdx.y * out_chunk_stride + size_t(row) * nh;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int x = xb + 32 * i;
      if (x < nh) dst[x] = make_float2(re[i], im[i]);
    }
  }
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

int launch_row_nnz(const float* w, int m, int* row_nnz, cudaStream_t s) {
  k_row_nnz<<<m, 256, 0, s>>>(w, m, row_nnz);
  WCGH_CHECK_LAUNCH();
  return 1;
}

// Writes one stage's contribution for the row band into `plane` (rows x nh,
// overwritten); the caller sums the stage planes in stage order.
int launch_lut_superpose(const float2* lut, int nh, int block, const float* w, int m, int off,
                         int row0, int rows, float2* plane, cudaStream_t s, double* updates,
                         const int* row_nnz) {
  const int P = nh >= 512 ? 16 : (nh >= 256 ? 8 : 4);
  const int tiles_x = (nh + 32 * P - 1) / (32 * P);
  const int tiles_y = (rows + 7) / 8;
  dim3 grid(unsigned(tiles_x * tiles_y), 1);
  const size_t smem = sizeof(float) * size_t(m);
  if (P == 16)
    k_lut_superpose<16><<<grid, kThreads, smem, s>>>(lut, nh, block, w, m, off, row0, rows, tiles_x, m, row_nnz, plane, 0);
  else if (P == 8)
    k_lut_superpose<8><<<grid, kThreads, smem, s>>>(lut, nh, block, w, m, off, row0, rows, tiles_x, m, row_nnz, plane, 0);
  else
    k_lut_superpose<4><<<grid, kThreads, smem, s>>>(lut, nh, block, w, m, off, row0, rows, tiles_x, m, row_nnz, plane, 0);
  WCGH_CHECK_LAUNCH();
  (void)updates;
  return 1;
}

}  // namespace wcgh
