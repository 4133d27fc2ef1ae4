// Microbenchmark: packed FP32 (FFMA2 / FADD2 / FMUL2) throughput by operand
// pattern, to see whether the ~88-91% FMA-pipe ceiling of a pure FFMA2
// stream (tools/microbench_fmamix.cu) depends on where the operands come
// from (register pairs, a scalar broadcast register, a constant-bank
// operand, a uniform register).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbo tools/microbench_operands.cu && /tmp/mbo
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kIters = 4096;
constexpr int kAcc = 16;

__constant__ float c_w[4];

__device__ __forceinline__ float2 ffma2s(float w, float2 v, float2 a) {  // scalar broadcast
  float2 r;
  asm("{\n .reg .b64 pv, pw, pa, pr;\n mov.b64 pv, {%2, %3};\n mov.b64 pw, {%4, %4};\n"
      " mov.b64 pa, {%5, %6};\n fma.rn.f32x2 pr, pw, pv, pa;\n mov.b64 {%0, %1}, pr;\n}\n"
      : "=f"(r.x), "=f"(r.y)
      : "f"(v.x), "f"(v.y), "f"(w), "f"(a.x), "f"(a.y));
  return r;
}

// MODE 0: FFMA2 acc += w(scalar reg) * v(pair)        [K4's MAC]
// MODE 1: FFMA2 acc += u(pair) * v(pair)              [three register pairs]
// MODE 2: FFMA2 acc += w(constant bank) * v(pair)
// MODE 3: FFMA2 acc += w(uniform: REDUX) * v(pair)
// MODE 4: FADD2 acc += v(pair)
// MODE 5: FMUL2 acc = acc * v(pair)
// MODE 6: K3's run step (two chains): Z += w; u = g*i + v; t = w*u; w = w*u - t (8 packed ops)
template <int MODE>
__global__ void __launch_bounds__(256) k_bench(float* out, float seed, int off) {
  float2 acc[kAcc], v[4], u[4];
#pragma unroll
  for (int c = 0; c < kAcc; ++c) acc[c] = make_float2(seed * c, seed + c);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    v[c] = make_float2(seed * (threadIdx.x + c), seed - c);
    u[c] = make_float2(seed * (threadIdx.x - c), seed + 2 * c);
  }
  float w = seed * 0.5f;
  if (MODE == 3) w = __int_as_float(__reduce_or_sync(0xffffffffu, __float_as_int(w) + off));
  __syncthreads();
  for (int it = 0; it < kIters; ++it) {
    if constexpr (MODE == 6) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {  // two independent chains of 4 steps each per iteration
        float2& zr = acc[k * 8 + 0];
        float2& zi = acc[k * 8 + 1];
        float2& wr = acc[k * 8 + 2];
        float2& wi = acc[k * 8 + 3];
        const float2 vr = v[k], vi = v[k + 2], gr = u[k], gi = u[k + 2];
#pragma unroll
        for (int i = 1; i < 5; ++i) {
          zr = __fadd2_rn(zr, wr);
          zi = __fadd2_rn(zi, wi);
          const float2 fi = make_float2(float(i), float(i));
          const float2 ur = __ffma2_rn(gr, fi, vr), ui = __ffma2_rn(gi, fi, vi);
          const float2 t1 = __fmul2_rn(wi, ui), t2 = __fmul2_rn(wi, ur);
          const float2 nwr = __ffma2_rn(wr, ur, make_float2(-t1.x, -t1.y));
          wi = __ffma2_rn(wr, ui, t2);
          wr = nwr;
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < kAcc; ++c) {
        if constexpr (MODE == 0 || MODE == 3) {
          acc[c] = ffma2s(w, v[c & 3], acc[c]);
        } else if constexpr (MODE == 1) {
          acc[c] = __ffma2_rn(u[c & 3], v[c & 3], acc[c]);
        } else if constexpr (MODE == 2) {
          acc[c] = ffma2s(c_w[c & 3], v[c & 3], acc[c]);
        } else if constexpr (MODE == 4) {
          acc[c] = __fadd2_rn(acc[c], v[c & 3]);
        } else if constexpr (MODE == 5) {
          acc[c] = __fmul2_rn(acc[c], v[c & 3]);
        }
      }
    }
    if (MODE != 3) w += 1e-7f;
  }
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < kAcc; ++c) r += acc[c].x + acc[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(const char* name, double lane_ops_per_iter, int sms, int bps) {
  const int blocks = sms * bps;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * 256);
  k_bench<MODE><<<blocks, 256>>>(out, 1.2345f, 0);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int rep = 0; rep < 10; ++rep) k_bench<MODE><<<blocks, 256>>>(out, 1.2345f, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 10.0 * blocks * 256.0 * kIters * lane_ops_per_iter;
  const double rate = ops / (ms * 1e-3);
  printf("%-44s %d blk/SM: %.2f T lane-op/s = %.1f lane-op/clk/SM at 1965 MHz\n", name, bps,
         rate * 1e-12, rate / (sms * 1.965e9));
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const float hw[4] = {0.5f, 0.25f, 0.125f, 0.0625f};
  cudaMemcpyToSymbol(c_w, hw, sizeof(hw));
  for (int bps : {2, 4}) {
    run<0>("FFMA2 w(scalar reg) x v(pair) [K4 MAC]", 2.0 * kAcc, sms, bps);
    run<1>("FFMA2 u(pair) x v(pair)", 2.0 * kAcc, sms, bps);
    run<2>("FFMA2 w(constant bank) x v(pair)", 2.0 * kAcc, sms, bps);
    run<3>("FFMA2 w(uniform, REDUX) x v(pair)", 2.0 * kAcc, sms, bps);
    run<4>("FADD2 acc + v(pair)", 2.0 * kAcc, sms, bps);
    run<5>("FMUL2 acc * v(pair)", 2.0 * kAcc, sms, bps);
    run<6>("K3 run step (8 packed ops/step, 2 chains)", 2.0 * 4 * 8 * 2, sms, bps);
  }
  return 0;
}
