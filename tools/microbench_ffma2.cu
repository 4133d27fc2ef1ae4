// Microbenchmark: scalar FFMA vs packed FFMA2 (fma.rn.f32x2, sm_100a) issue
// and lane throughput per SM per clock -- pins the FP32 roofline of the LUT
// superposition kernel (K4), whose inner loop is acc += w * lut_sample
// (one complex-by-real MAC = 2 lane FMAs = 1 FFMA2 with a broadcast scalar).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb2 tools/microbench_ffma2.cu && /tmp/mb2
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kIters = 2048;
constexpr int kAcc = 16;

__device__ __forceinline__ float2 ffma2(float w, float2 v, float2 a) {
  float2 r;
  asm("{\n .reg .b64 pv, pw, pa, pr;\n mov.b64 pv, {%2, %3};\n mov.b64 pw, {%4, %4};\n"
      " mov.b64 pa, {%5, %6};\n fma.rn.f32x2 pr, pw, pv, pa;\n mov.b64 {%0, %1}, pr;\n}\n"
      : "=f"(r.x), "=f"(r.y)
      : "f"(v.x), "f"(v.y), "f"(w), "f"(a.x), "f"(a.y));
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_bench(float* out, long long* cycles, float seed) {
  float2 acc[kAcc], v[4];
#pragma unroll
  for (int c = 0; c < kAcc; ++c) acc[c] = make_float2(seed * c, seed + c);
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = make_float2(seed * (threadIdx.x + c), seed - c);
  float w = seed * 0.5f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kAcc; ++c) {
      if (MODE == 0) {
        acc[c].x = fmaf(w, v[c & 3].x, acc[c].x);
        acc[c].y = fmaf(w, v[c & 3].y, acc[c].y);
      } else {
        acc[c] = ffma2(w, v[c & 3], acc[c]);
      }
    }
    w += 1e-7f;
  }
  const long long t1 = clock64();
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < kAcc; ++c) r += acc[c].x + acc[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int sms, int bps) {
  const int blocks = sms * bps;
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * blocks * 256);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  k_bench<MODE><<<blocks, 256>>>(out, cyc, 1.2345f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_bench<MODE><<<blocks, 256>>>(out, cyc, 1.2345f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += double(h[i]);
  avg /= blocks;
  const double macs_per_sm = double(bps) * 256.0 * kIters * kAcc;  // complex-by-real MACs
  const double per_clk = macs_per_sm / avg;
  const double lane_fma = 2 * per_clk;
  const double wall = macs_per_sm * sms / (ms * 1e-3);
  printf("%-10s %d blk/SM: MAC/clk/SM %7.2f  lane-FMA/clk/SM %7.2f  (%.3f ms, %.3e MAC/s)\n", name,
         bps, per_clk, lane_fma, ms, wall);
  delete[] h;
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  for (int bps : {1, 2, 4}) {
    run<0>("ffma", sms, bps);
    run<1>("ffma2", sms, bps);
  }
  return 0;
}
