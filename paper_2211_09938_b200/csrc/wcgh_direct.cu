// K3: pixel-owning direct point-source accumulation,
//   H(x,y) = sum_j A_j * exp(i k r_j) / r_j,  r_j = sqrt(((x-x_j)^2 + (y-y_j)^2) p^2 + z^2),
// the sum the reference's pointwise_sum forms (tests/support/oracles.cpp:12-36)
// and the production LUT path reproduces (synthesis.cpp:255-286; telescoping,
// test_synthesis.cpp:193-203), evaluated over the compacted A_eff points.
//
// Work decomposition: a CTA of 8 warps owns an 8-row x 32P-column tile; lane
// l of warp w owns pixels (x_b + l + 32 i, y_0 + w), i < P, and keeps their
// complex sums in registers. Points stream through shared memory in batches
// of 256 16-byte records and are broadcast to all threads. The point list is
// split into chunks whose boundaries depend only on the point count, each
// chunk producing a partial plane that a fixed-order reduction sums: the
// per-pixel summation order is independent of the launch and of the row-band
// split across GPUs (the GPU analogue of accumulate_deterministic,
// parallel.cpp:49-98), so results are bitwise identical for any GPU count.
//
// Phase (fixed mode): cycles = frac(z/lambda) + s*alpha + (z/lambda) g(u), with
// the quadratic term in exact 0.64/0.32 fixed point and advanced along a
// thread's pixels by an exact second-order recurrence (two IADDs), and the
// small higher-order term g(u) = sqrt(1+u)-1-u/2 as an fp32 series. fp32
// k*r would lose the phase entirely (k r ~ 2.4e6 rad); see SURVEY.md App. A.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "wcgh_internal.cuh"

namespace wcgh {

__constant__ DirectLayer c_layers[kMaxLayers];

namespace {

constexpr int kBatch = 256;
constexpr int kThreads = 256;
constexpr float kTwoPi = 6.283185307179586f;
constexpr float kNegThreePi = -9.42477796076938f;

// int -> float for |v| < 2^22 on the ALU+FMA pipes (avoids the XU-pipe I2F).
__device__ __forceinline__ float i2f_small(int v) {
  return __int_as_float(v + 0x4B400000) - 12582912.0f;
}

template <int P, int NC, bool POLY_AMP>
__global__ void __launch_bounds__(kThreads, 2)
    k_direct_fixed(const int4* __restrict__ pts, const long long* __restrict__ layer_begin,
                   int n_layers, long long chunk, long long n_points, int nh, int row0, int rows,
                   int tiles_x, float2* __restrict__ out, size_t out_chunk_stride) {
  __shared__ int4 sp[kBatch];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int tx = blockIdx.x % tiles_x;
  const int ty = blockIdx.x / tiles_x;
  const int row = ty * 8 + warp;  // row within the band
  const int y = row0 + row;       // hologram row
  const int xb = tx * 32 * P + lane;
  const long long p0 = (long long)blockIdx.y * chunk;
  const long long p1 = min(p0 + chunk, n_points);

  float tre[P], tim[P];
#pragma unroll
  for (int i = 0; i < P; ++i) tre[i] = tim[i] = 0.0f;

  for (int l = 0; l < n_layers; ++l) {
    const long long s0 = max(p0, layer_begin[l]);
    const long long s1 = min(p1, layer_begin[l + 1]);
    if (s0 >= s1) continue;
    const DirectLayer& L = c_layers[l];
    const uint32_t a_hi = L.a_hi, a_lo = L.a_lo, phi0 = L.phi0, dd = L.dd;
    const float c = L.c, inv_z = L.inv_z;
    const float c64 = 64.0f * c, c1024 = 1024.0f * c, ddu = 2048.0f * c;
    float corr[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) corr[k] = L.corr[k];
    const float am1 = L.amp[0], am2 = L.amp[1], am3 = L.amp[2];

    for (long long b = s0; b < s1; b += kBatch) {
      const int nb = int(min((long long)kBatch, s1 - b));
      __syncthreads();
      if (threadIdx.x < nb) sp[threadIdx.x] = pts[b + threadIdx.x];
      __syncthreads();

      float re[P], im[P];
#pragma unroll
      for (int i = 0; i < P; ++i) re[i] = im[i] = 0.0f;

#pragma unroll 1
      for (int j = 0; j < nb; ++j) {
        const int4 q = sp[j];
        const int dx0 = xb - q.x;
        const int dy = y - q.y;
        const int s = dx0 * dx0 + dy * dy;  // exact: |dx|,|dy| < 2^15
        const int s_1 = s + 64 * dx0 + 1024;  // pixel i = 1 (x + 32)
        uint32_t t = uint32_t(s) * a_hi + __umulhi(uint32_t(s), a_lo) + phi0;
        const uint32_t t1 = uint32_t(s_1) * a_hi + __umulhi(uint32_t(s_1), a_lo) + phi0;
        uint32_t D = t1 - t;
        const float fdx = i2f_small(dx0), fdy = i2f_small(dy);
        float u = fmaf(fdx * c, fdx, fdy * fdy * c);
        float du = fmaf(fdx, c64, c1024);
        const float a0 = __int_as_float(q.z) * inv_z;
        const float a1 = a0 * am1, a2 = a0 * am2, a3 = a0 * am3;
#pragma unroll
        for (int i = 0; i < P; ++i) {
          // [1,2) cycles from the top 23 fraction bits of the fixed-point phase
          const float phf = __int_as_float((t >> 9) | 0x3f800000u);
          const float u2 = u * u;
          float pc = corr[NC - 1];
#pragma unroll
          for (int k = NC - 2; k >= 0; --k) pc = fmaf(pc, u, corr[k]);
          // radians in [-pi, pi) + correction: (phf - 1.5) * 2pi + u^2 * pc
          const float ph = fmaf(phf, kTwoPi, fmaf(u2, pc, kNegThreePi));
          float am;
          if constexpr (POLY_AMP) {
            am = fmaf(fmaf(fmaf(a3, u, a2), u, a1), u, a0);
          } else {
            am = a0 * rsqrtf(1.0f + u);
          }
          float sn, cs;
          __sincosf(ph, &sn, &cs);
          re[i] = fmaf(am, cs, re[i]);
          im[i] = fmaf(am, sn, im[i]);
          t += D;
          D += dd;
          u += du;
          du += ddu;
        }
      }
#pragma unroll
      for (int i = 0; i < P; ++i) {
        tre[i] += re[i];
        tim[i] += im[i];
      }
    }
  }

  if (row < rows) {
    float2* dst = out + blockIdx.y * out_chunk_stride + size_t(row) * nh;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int x = xb + 32 * i;
      if (x < nh) dst[x] = make_float2(tre[i], tim[i]);
    }
  }
}

// Double-phase option: r and k*r in fp64, reduced to [-pi, pi] in fp64, then
// fp32 sin/cos. Accuracy mode (FP64 pipe bound).
template <int P>
__global__ void __launch_bounds__(kThreads)
    k_direct_fp64(const int4* __restrict__ pts, const long long* __restrict__ layer_begin,
                  int n_layers, long long chunk, long long n_points, int nh, int row0, int rows,
                  int tiles_x, float2* __restrict__ out, size_t out_chunk_stride) {
  __shared__ int4 sp[kBatch];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int tx = blockIdx.x % tiles_x;
  const int ty = blockIdx.x / tiles_x;
  const int row = ty * 8 + warp;
  const int y = row0 + row;
  const int xb = tx * 32 * P + lane;
  const long long p0 = (long long)blockIdx.y * chunk;
  const long long p1 = min(p0 + chunk, n_points);
  const double two_pi = 6.283185307179586476925286766559;

  float tre[P], tim[P];
#pragma unroll
  for (int i = 0; i < P; ++i) tre[i] = tim[i] = 0.0f;

  for (int l = 0; l < n_layers; ++l) {
    const long long s0 = max(p0, layer_begin[l]);
    const long long s1 = min(p1, layer_begin[l + 1]);
    if (s0 >= s1) continue;
    const double pitch = c_layers[l].pitch, z = c_layers[l].z, k = c_layers[l].k;
    const double z2 = z * z;
    for (long long b = s0; b < s1; b += kBatch) {
      const int nb = int(min((long long)kBatch, s1 - b));
      __syncthreads();
      if (threadIdx.x < nb) sp[threadIdx.x] = pts[b + threadIdx.x];
      __syncthreads();
      float re[P], im[P];
#pragma unroll
      for (int i = 0; i < P; ++i) re[i] = im[i] = 0.0f;
#pragma unroll 1
      for (int j = 0; j < nb; ++j) {
        const int4 q = sp[j];
        const double ddy = double(y - q.y) * pitch;
        const double a = double(__int_as_float(q.z));
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const double ddx = double(xb + 32 * i - q.x) * pitch;
          const double r = sqrt(ddx * ddx + ddy * ddy + z2);
          const double kr = k * r;
          const double red = kr - two_pi * rint(kr * (1.0 / two_pi));
          const float am = float(a / r);
          float sn, cs;
          __sincosf(float(red), &sn, &cs);
          re[i] = fmaf(am, cs, re[i]);
          im[i] = fmaf(am, sn, im[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < P; ++i) {
        tre[i] += re[i];
        tim[i] += im[i];
      }
    }
  }
  if (row < rows) {
    float2* dst = out + blockIdx.y * out_chunk_stride + size_t(row) * nh;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int x = xb + 32 * i;
      if (x < nh) dst[x] = make_float2(tre[i], tim[i]);
    }
  }
}

// Fixed-order chunk reduction in fp64: out = sum_c partial[c].
__global__ void k_reduce_chunks(const float2* __restrict__ partial, int n_chunks, size_t count,
                                float2* __restrict__ out) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double re = 0.0, im = 0.0;
  for (int c = 0; c < n_chunks; ++c) {
    const float2 v = partial[size_t(c) * count + i];
    re += v.x;
    im += v.y;
  }
  out[i] = make_float2(float(re), float(im));
}

// binom(a, n) for real a.
double binom(double a, int n) {
  double r = 1.0;
  for (int i = 0; i < n; ++i) r *= (a - i) / (i + 1);
  return r;
}

template <int P, int NC, bool POLY>
void launch_fixed(dim3 grid, cudaStream_t s, const int4* pts, const long long* lb, int L,
                  long long chunk, long long np, int nh, int row0, int rows, int tiles_x,
                  float2* out, size_t stride) {
  k_direct_fixed<P, NC, POLY><<<grid, kThreads, 0, s>>>(pts, lb, L, chunk, np, nh, row0, rows,
                                                        tiles_x, out, stride);
}

template <int P>
void launch_fixed_nc(const DirectPlan& plan, dim3 grid, cudaStream_t s, const int4* pts,
                     const long long* lb, int L, long long chunk, long long np, int nh, int row0,
                     int rows, int tiles_x, float2* out, size_t stride) {
#define WCGH_LF(NC, POLY) \
  launch_fixed<P, NC, POLY>(grid, s, pts, lb, L, chunk, np, nh, row0, rows, tiles_x, out, stride)
  if (plan.n_corr <= 3) {
    if (plan.poly_amp) WCGH_LF(3, true); else WCGH_LF(3, false);
  } else if (plan.n_corr <= 5) {
    if (plan.poly_amp) WCGH_LF(5, true); else WCGH_LF(5, false);
  } else {
    if (plan.poly_amp) WCGH_LF(8, true); else WCGH_LF(8, false);
  }
#undef WCGH_LF
}

}  // namespace

DirectLayer make_direct_layer(const wcgh_layer& L) {
  DirectLayer d{};
  const double lam = L.wavelength, p = L.pitch, z = L.z;
  const double alpha = p * p / (2.0 * lam * z);
  const double fa = alpha - std::floor(alpha);
  const double hi = std::floor(std::ldexp(fa, 32));
  const double lo = std::floor(std::ldexp(std::ldexp(fa, 32) - hi, 32));
  d.a_hi = uint32_t(hi);
  d.a_lo = uint32_t(lo);
  const double K = z / lam;
  d.phi0 = uint32_t(uint64_t(std::llround(std::ldexp(K - std::floor(K), 32))) & 0xffffffffu);
  const double ddc = 2048.0 * alpha;
  d.dd = uint32_t(uint64_t(std::llround(std::ldexp(ddc - std::floor(ddc), 32))) & 0xffffffffu);
  d.c = float(p * p / (z * z));
  d.inv_z = float(1.0 / z);
  const double two_pi = 6.283185307179586476925286766559;
  for (int k = 0; k < kMaxCorr; ++k) d.corr[k] = float(two_pi * K * binom(0.5, k + 2));
  for (int k = 0; k < 4; ++k) d.amp[k] = float(binom(-0.5, k + 1));
  d.wavelength = lam;
  d.pitch = p;
  d.z = z;
  d.k = two_pi / lam;
  return d;
}

DirectPlan plan_direct(const wcgh_layer* layers, int n_layers, double max_dx, double max_dy) {
  DirectPlan plan{3, true, 0.0};
  const double two_pi = 6.283185307179586476925286766559;
  const double s_max = max_dx * max_dx + max_dy * max_dy;
  int need = 3;
  bool poly = true;
  for (int l = 0; l < n_layers; ++l) {
    const double p = layers[l].pitch, z = layers[l].z, K = layers[l].z / layers[l].wavelength;
    const double u = s_max * p * p / (z * z);
    plan.u_max = std::max(plan.u_max, u);
    require(u < 0.5, "direct (fixed phase): geometry too oblique for the fp32 correction series "
                     "(u_max >= 0.5); use WCGH_PHASE_FP64");
    int nc = 0;
    for (nc = 1; nc <= kMaxCorr; ++nc) {
      // truncation after b_2..b_{nc+1}: next term bounds the tail for u < 1/2
      const double tail = two_pi * K * std::fabs(binom(0.5, nc + 2)) * std::pow(u, nc + 2) / (1.0 - u);
      if (tail <= 1e-7) break;
    }
    require(nc <= kMaxCorr, "direct (fixed phase): correction series does not converge to "
                            "1e-7 rad; use WCGH_PHASE_FP64");
    need = std::max(need, nc);
    // cubic (1+u)^(-1/2): relative tail below 2e-8
    if (std::fabs(binom(-0.5, 4)) * std::pow(u, 4) / (1.0 - u) > 2e-8) poly = false;
  }
  plan.n_corr = need <= 3 ? 3 : (need <= 5 ? 5 : 8);
  plan.poly_amp = poly;
  return plan;
}

int launch_direct(const wcgh_point* pts_dev, const int64_t* layer_begin_host, int n_layers,
                  const wcgh_layer* layers, int nh, int row0, int rows, int phase_mode,
                  double max_dx, double max_dy, float2* out_dev, DirectScratch& scratch,
                  cudaStream_t stream, cudaEvent_t ev_synth_end, double* updates_out) {
  require(n_layers >= 1 && n_layers <= kMaxLayers, "direct: 1..16 layers");
  require(rows >= 1 && row0 >= 0 && row0 + rows <= nh, "direct: row band outside the plane");
  const long long n_points = layer_begin_host[n_layers];
  if (updates_out) *updates_out = double(n_points) * double(rows) * double(nh);
  int launches = 0;
  if (n_points == 0) {
    WCGH_CUDA(cudaMemsetAsync(out_dev, 0, size_t(rows) * nh * sizeof(float2), stream));
    if (ev_synth_end) WCGH_CUDA(cudaEventRecord(ev_synth_end, stream));
    return 0;
  }
  DirectLayer h_layers[kMaxLayers];
  for (int l = 0; l < n_layers; ++l) h_layers[l] = make_direct_layer(layers[l]);
  WCGH_CUDA(cudaMemcpyToSymbolAsync(c_layers, h_layers, sizeof(DirectLayer) * n_layers, 0,
                                    cudaMemcpyHostToDevice, stream));
  // layer offsets live in a small device array appended to the scratch
  // Chunking depends on the point count only (determinism across row splits).
  const long long target = 64;
  long long chunk = (n_points + target - 1) / target;
  chunk = std::max<long long>(kBatch, ((chunk + kBatch - 1) / kBatch) * kBatch);
  const int n_chunks = int((n_points + chunk - 1) / chunk);

  const int P = nh >= 512 ? 16 : (nh >= 256 ? 8 : 4);
  const int tiles_x = (nh + 32 * P - 1) / (32 * P);
  const int tiles_y = (rows + 7) / 8;
  const size_t band = size_t(rows) * nh;
  const size_t stride = size_t(tiles_y) * 8 * nh;  // partial planes cover whole tiles
  const size_t lb_bytes = sizeof(long long) * (n_layers + 1);
  const size_t part_bytes = n_chunks > 1 ? stride * n_chunks * sizeof(float2) : 0;
  char* base = static_cast<char*>(scratch.partial.reserve(part_bytes + 256 + lb_bytes));
  long long* lb_dev = reinterpret_cast<long long*>(base + part_bytes + 256 - (part_bytes % 256));
  static_assert(sizeof(long long) == sizeof(int64_t), "int64");
  WCGH_CUDA(cudaMemcpyAsync(lb_dev, layer_begin_host, lb_bytes, cudaMemcpyHostToDevice, stream));

  float2* target_plane = n_chunks > 1 ? reinterpret_cast<float2*>(base) : out_dev;
  const size_t out_stride = n_chunks > 1 ? stride : 0;
  // With one chunk the kernel writes the band directly; rows beyond `rows`
  // are masked by the kernel (row < rows).
  dim3 grid(unsigned(tiles_x * tiles_y), unsigned(n_chunks));
  const int4* p4 = reinterpret_cast<const int4*>(pts_dev);
  if (phase_mode == WCGH_PHASE_FP64) {
    if (P == 16)
      k_direct_fp64<16><<<grid, kThreads, 0, stream>>>(p4, lb_dev, n_layers, chunk, n_points, nh, row0, rows, tiles_x, target_plane, out_stride);
    else if (P == 8)
      k_direct_fp64<8><<<grid, kThreads, 0, stream>>>(p4, lb_dev, n_layers, chunk, n_points, nh, row0, rows, tiles_x, target_plane, out_stride);
    else
      k_direct_fp64<4><<<grid, kThreads, 0, stream>>>(p4, lb_dev, n_layers, chunk, n_points, nh, row0, rows, tiles_x, target_plane, out_stride);
  } else {
    require(phase_mode == WCGH_PHASE_FIXED, "direct: unknown phase mode");
    const DirectPlan plan = plan_direct(layers, n_layers, max_dx, max_dy);
    if (P == 16)
      launch_fixed_nc<16>(plan, grid, stream, p4, lb_dev, n_layers, chunk, n_points, nh, row0, rows, tiles_x, target_plane, out_stride);
    else if (P == 8)
      launch_fixed_nc<8>(plan, grid, stream, p4, lb_dev, n_layers, chunk, n_points, nh, row0, rows, tiles_x, target_plane, out_stride);
    else
      launch_fixed_nc<4>(plan, grid, stream, p4, lb_dev, n_layers, chunk, n_points, nh, row0, rows, tiles_x, target_plane, out_stride);
  }
  WCGH_CHECK_LAUNCH();
  ++launches;
  if (ev_synth_end) WCGH_CUDA(cudaEventRecord(ev_synth_end, stream));
  if (n_chunks > 1) {
    // partial planes are laid out with a tile-rounded row count; reduce the band
    // row by row region: stride == band when rows % 8 == 0.
    if (stride == band) {
      k_reduce_chunks<<<unsigned((band + 255) / 256), 256, 0, stream>>>(target_plane, n_chunks, band, out_dev);
      WCGH_CHECK_LAUNCH();
      ++launches;
    } else {
      // rows not a multiple of 8: reduce the padded layout, then the band is its prefix
      k_reduce_chunks<<<unsigned((stride + 255) / 256), 256, 0, stream>>>(target_plane, n_chunks, stride, target_plane);
      WCGH_CHECK_LAUNCH();
      WCGH_CUDA(cudaMemcpyAsync(out_dev, target_plane, band * sizeof(float2), cudaMemcpyDeviceToDevice, stream));
      ++launches;
    }
  }
  return launches;
}

}  // namespace wcgh
