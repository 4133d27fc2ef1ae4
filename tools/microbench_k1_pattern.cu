// K1 access-pattern microbenchmark: the u8 front end's memory traffic
// (8-byte row loads of an 8x8 cell from two uint8 images, 8 float4-pair row
// stores of fp32) with no compute, one thread per cell, vs a plain
// contiguous copy of the same bytes. Separates "access pattern" from
// "compute/latency" as the cause of k_analysis_u8's bandwidth.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/k1p tools/microbench_k1_pattern.cu && /tmp/k1p
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void __launch_bounds__(128, 4) k_cells(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                                  int n, float* __restrict__ out) {
  const int bx = blockIdx.x * 128 + threadIdx.x, by = blockIdx.y;
  if (bx >= n / 8) return;
  uint2 va[8], vb[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    va[r] = *reinterpret_cast<const uint2*>(a + size_t(8 * by + r) * n + 8 * bx);
    vb[r] = *reinterpret_cast<const uint2*>(b + size_t(8 * by + r) * n + 8 * bx);
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const unsigned x = va[r].x ^ vb[r].x, y = va[r].y ^ vb[r].y;
    float4* dst = reinterpret_cast<float4*>(out + size_t(8 * by + r) * n + 8 * bx);
    dst[0] = make_float4(float(x & 255), float(x >> 8 & 255), float(x >> 16 & 255), float(x >> 24));
    dst[1] = make_float4(float(y & 255), float(y >> 8 & 255), float(y >> 16 & 255), float(y >> 24));
  }
}

__global__ void k_linear(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, size_t count,
                         float* __restrict__ out) {
  const size_t i = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (i >= count) return;
  const unsigned x = *reinterpret_cast<const unsigned*>(a + i) ^ *reinterpret_cast<const unsigned*>(b + i);
  *reinterpret_cast<float4*>(out + i) =
      make_float4(float(x & 255), float(x >> 8 & 255), float(x >> 16 & 255), float(x >> 24));
}

int main() {
  const int n = 16384;
  const size_t n2 = size_t(n) * n;
  uint8_t *a, *b;
  float* out;
  cudaMalloc(&a, n2);
  cudaMalloc(&b, n2);
  cudaMalloc(&out, n2 * 4);
  cudaMemset(a, 1, n2);
  cudaMemset(b, 2, n2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = double(n2) * 6;
  for (int rep = 0; rep < 3; ++rep) {
    float ms = 0;
    cudaEventRecord(e0);
    k_cells<<<dim3((n / 8 + 127) / 128, n / 8), 128>>>(a, b, n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cell pattern : %.3f ms  %.0f GB/s\n", ms, bytes / (ms * 1e-3) / 1e9);
    cudaEventRecord(e0);
    k_linear<<<unsigned((n2 / 4 + 255) / 256), 256>>>(a, b, n2, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("linear       : %.3f ms  %.0f GB/s\n", ms, bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
