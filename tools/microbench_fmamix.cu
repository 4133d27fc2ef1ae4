// Microbenchmark: can scalar FFMA (fmalite) run beside packed FFMA2
// (fmaheavy only) to exceed 128 FP32 lane-FMAs/clk/SM, and does a
// predicated-off FFMA2 still occupy the fmaheavy pipe?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbm tools/microbench_fmamix.cu && /tmp/mbm
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

// MODE 0: all scalar FFMA; 1: all FFMA2; 2: NS of kAcc accumulators as two
// scalar FFMAs, the rest FFMA2; 3: FFMA2 under a runtime-false predicate
// for half the accumulators (counts only the executed half as work).
template <int MODE, int NS>
__global__ void __launch_bounds__(256) k_bench(float* out, long long* cycles, float seed, int off) {
  float2 acc[kAcc], v[4];
#pragma unroll
  for (int c = 0; c < kAcc; ++c) acc[c] = make_float2(seed * c, seed + c);
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = make_float2(seed * (threadIdx.x + c), seed - c);
  float w = seed * 0.5f, w0 = seed * float(off);  // w0 == 0 at run time (off = 0)
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kAcc; ++c) {
      if (MODE == 0 || (MODE == 2 && c < NS)) {
        acc[c].x = fmaf(w, v[c & 3].x, acc[c].x);
        acc[c].y = fmaf(w, v[c & 3].y, acc[c].y);
      } else if (MODE == 3 && (c & 1)) {
        if (w0 != 0.f) acc[c] = ffma2(w0, v[c & 3], acc[c]);
      } else {
        acc[c] = ffma2(w, v[c & 3], acc[c]);
      }
    }
    w += 1e-7f;
    w0 *= 1.0000001f;
  }
  const long long t1 = clock64();
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < kAcc; ++c) r += acc[c].x + acc[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE, int NS>
void run(const char* name, int sms, int bps) {
  const int blocks = sms * bps;
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * blocks * 256);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  k_bench<MODE, NS><<<blocks, 256>>>(out, cyc, 1.2345f, 0);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int rep = 0; rep < 5; ++rep) k_bench<MODE, NS><<<blocks, 256>>>(out, cyc, 1.2345f, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  long long* h = new long long[blocks];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += double(h[i]);
  avg /= blocks;
  const int active = MODE == 3 ? kAcc / 2 : kAcc;
  const double macs_per_sm = double(bps) * 256.0 * kIters * active;
  const double wall_lane = 2 * macs_per_sm * sms * 5 / (ms * 1e-3);  // lane FMAs/s
  printf("%-22s %d blk/SM: clock64 lane-FMA/clk/SM %7.2f | wall %.2f TFMA/s = %.1f lane-FMA/clk/SM at %d MHz\n",
         name, bps, 2 * macs_per_sm / avg, wall_lane * 1e-12, wall_lane / (sms * khz * 1e3), khz / 1000);
  delete[] h;
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bps : {2, 4}) {
    run<0, 0>("ffma (scalar)", sms, bps);
    run<1, 0>("ffma2", sms, bps);
    run<2, 2>("ffma2 + 2/16 scalar", sms, bps);
    run<2, 4>("ffma2 + 4/16 scalar", sms, bps);
    run<2, 6>("ffma2 + 6/16 scalar", sms, bps);
    run<2, 8>("ffma2 + 8/16 scalar", sms, bps);
    run<3, 0>("ffma2, half pred-off", sms, bps);
  }
  return 0;
}
