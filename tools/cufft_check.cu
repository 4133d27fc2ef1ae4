// Minimal cuFFT interop check (static vs shared cudart).
#include <cuda_runtime.h>
#include <cufft.h>
#include <cstdio>
int main() {
  const int L = 256;
  cufftComplex* d;
  cudaMalloc(&d, sizeof(cufftComplex) * L * L);
  cudaMemset(d, 0, sizeof(cufftComplex) * L * L);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cufftHandle p;
  printf("plan %d\n", (int)cufftPlan2d(&p, L, L, CUFFT_C2C));
  printf("setstream %d\n", (int)cufftSetStream(p, s));
  printf("exec %d\n", (int)cufftExecC2C(p, d, d, CUFFT_FORWARD));
  printf("sync %s\n", cudaGetErrorString(cudaStreamSynchronize(s)));
  printf("devsync %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
