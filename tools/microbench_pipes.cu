// Microbenchmark: MUFU (XU) and FMA pipe throughput on the B200, to pin the
// roofline of the direct accumulation kernel (K3). Each thread runs an
// unrolled loop of independent chains; cycles are read with clock64 per
// CTA and throughput is reported per SM per clock.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_pipes.cu && /tmp/mb
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kIters = 4096;
constexpr int kChains = 8;

template <int MODE, int NFMA>
__global__ void __launch_bounds__(256) k_bench(float* out, long long* cycles, float seed) {
  float x[kChains], a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    x[c] = seed * (threadIdx.x + 1 + c);
    a[c] = 0.f;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      float s, co;
      if (MODE == 0) {  // sin + cos of the same argument
        __sincosf(x[c], &s, &co);
        a[c] += s * co;
      } else if (MODE == 1) {  // sin only
        s = __sinf(x[c]);
        a[c] += s;
      } else if (MODE == 2) {  // rsqrt only
        s = rsqrtf(x[c]);
        a[c] += s;
      } else if (MODE == 3) {  // ex2
        s = exp2f(x[c]);
        a[c] += s;
      } else {  // FFMA only
        s = x[c];
      }
      float t = s;
#pragma unroll
      for (int k = 0; k < NFMA; ++k) t = fmaf(t, 1.0001f, 0.5f);
      a[c] += t;
      x[c] += 1e-3f;
    }
  }
  const long long t1 = clock64();
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) r += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE, int NFMA>
void run(const char* name, int mufu_per_elem, int fma_per_elem, int sms, int blocks_per_sm) {
  const int blocks = sms * blocks_per_sm;
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * blocks * 256);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  k_bench<MODE, NFMA><<<blocks, 256>>>(out, cyc, 1.2345f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_bench<MODE, NFMA><<<blocks, 256>>>(out, cyc, 1.2345f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += double(h[i]);
  avg /= blocks;
  const double elems_per_sm = double(blocks_per_sm) * 256.0 * kIters * kChains;
  const double per_clk = elems_per_sm / avg;  // elements per SM per clock (co-resident blocks)
  const double ghz = (elems_per_sm * sms) / (per_clk * sms) / (ms * 1e-3) / 1e9;
  printf("%-28s elems/clk/SM %7.3f  mufu/clk/SM %6.2f  fma/clk/SM %7.2f  instr-est/clk/SM %6.2f  (%.3f ms, ~%.2f GHz)\n",
         name, per_clk, per_clk * mufu_per_elem, per_clk * fma_per_elem,
         per_clk * (mufu_per_elem + fma_per_elem + 2) / 32.0, ms, ghz);
  delete[] h;
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  for (int bps : {2, 4}) {
    printf("-- %d blocks/SM (%d warps/SM)\n", bps, bps * 8);
    run<0, 0>("sincos", 2, 1, sms, bps);
    run<1, 0>("sin", 1, 0, sms, bps);
    run<2, 0>("rsqrt", 1, 0, sms, bps);
    run<3, 0>("ex2", 1, 0, sms, bps);
    run<4, 16>("ffma x16", 0, 16, sms, bps);
    run<0, 4>("sincos + 4 ffma", 2, 5, sms, bps);
    run<0, 8>("sincos + 8 ffma", 2, 9, sms, bps);
    run<0, 12>("sincos + 12 ffma", 2, 13, sms, bps);
    run<0, 16>("sincos + 16 ffma", 2, 17, sms, bps);
  }
  return 0;
}
