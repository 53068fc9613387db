// FFMA vs DFMA vs F2F.F64.F32 throughput probe (one launch each, 148*8 CTAs x 256 thr)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ffma_k(float* o, int n) {
  float a = threadIdx.x, b = 1.0001f, c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  for (int i = 0; i < n; ++i) { c0 = fmaf(a, b, c0); c1 = fmaf(a, b, c1); c2 = fmaf(a, b, c2); c3 = fmaf(a, b, c3); }
  if (c0 + c1 + c2 + c3 == 1.2345f) o[0] = 1;
}
__global__ void dfma_k(double* o, int n) {
  double a = threadIdx.x, b = 1.0001, c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  for (int i = 0; i < n; ++i) { c0 = fma(a, b, c0); c1 = fma(a, b, c1); c2 = fma(a, b, c2); c3 = fma(a, b, c3); }
  if (c0 + c1 + c2 + c3 == 1.2345) o[0] = 1;
}
__global__ void f2f_k(double* o, int n) {
  float a = threadIdx.x; double c0 = 0, c1 = 0;
  for (int i = 0; i < n; ++i) { c0 += (double)(a + i); c1 += (double)(a - i); }
  if (c0 + c1 == 1.2345) o[0] = 1;
}
int main() {
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int n = 4096, blocks = 148 * 8, thr = 256;
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); ffma_k<<<blocks, thr>>>((float*)d, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA %.2f TFMA/s\n", (double)blocks * thr * n * 4 / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0); dfma_k<<<blocks, thr>>>(d, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA %.3f TFMA/s\n", (double)blocks * thr * n * 4 / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0); f2f_k<<<blocks, thr>>>(d, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("F2F+DADD %.3f T/s\n", (double)blocks * thr * n * 2 / (ms * 1e-3) / 1e12);
  }
  return 0;
}
