// Achievable HBM bandwidth of sorted random 256-B row gathers (K and V rows of
// selected tokens), vs contiguous streaming.  Rows: 16 seqs x 8 heads x 32768
// tokens x 256 B per tensor (1 GiB each).  Selection: every 10th token on
// average (sorted, random).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void gather_k(const uint4* __restrict__ K, const uint4* __restrict__ V, const int* __restrict__ idx,
                         int nsel, int unroll_rows, uint4* out) {
  // warp per group of rows; each half-warp loads one 256-B row (16 lanes x 16 B)
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int base = w * 16; base < nsel; base += nw * 16) {
    uint4 r[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      int i = base + q * 2 + (lane >> 4);
      int t = i < nsel ? idx[i] : 0;
      r[q] = __ldg(K + (size_t)t * 16 + (lane & 15));
      r[q + 8] = __ldg(V + (size_t)t * 16 + (lane & 15));
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) { acc.x ^= r[q].x; acc.y ^= r[q].y; acc.z ^= r[q].z; acc.w ^= r[q].w; }
  }
  if (acc.x == 0x12345678) out[0] = acc;
}
// K and V of a token interleaved: one 512-B row per token (full warp per row)
__global__ void gather_kv512(const uint4* __restrict__ KV, const int* __restrict__ idx, int nsel, uint4* out) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int base = w * 16; base < nsel; base += nw * 16) {
    uint4 r[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      int i = base + q;
      int t = i < nsel ? idx[i] : 0;
      r[q] = __ldg(KV + (size_t)t * 32 + lane);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) { acc.x ^= r[q].x; acc.y ^= r[q].y; acc.z ^= r[q].z; acc.w ^= r[q].w; }
  }
  if (acc.x == 0x12345678) out[0] = acc;
}
__global__ void stream_k(const uint4* __restrict__ K, size_t n, uint4* out) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (; i < n; i += st * 4) {
    uint4 a = K[i], b = i + st < n ? K[i + st] : a, c = i + 2 * st < n ? K[i + 2 * st] : a, d = i + 3 * st < n ? K[i + 3 * st] : a;
    acc.x ^= a.x ^ b.x ^ c.x ^ d.x;
  }
  if (acc.x == 0x12345678) out[0] = acc;
}
int main() {
  const size_t rows = 16ull * 8 * 32768;   // 4M rows of 256 B
  uint4 *K, *V, *o; int* idx;
  cudaMalloc(&K, rows * 256); cudaMalloc(&V, rows * 256); cudaMalloc(&o, 64);
  cudaMemset(K, 1, rows * 256); cudaMemset(V, 2, rows * 256);
  std::vector<int> h; srand(1);
  for (size_t r = 0; r < rows; ++r) if (rand() % 10 == 0) h.push_back((int)r);
  int nsel = (int)h.size();
  cudaMalloc(&idx, nsel * 4); cudaMemcpy(idx, h.data(), nsel * 4, cudaMemcpyHostToDevice);
  void* flush; cudaMalloc(&flush, 512 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(flush, rep, 512 << 20);
      cudaEventRecord(e0); gather_k<<<blocks, 256>>>(K, V, idx, nsel, 0, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("gather blocks=%d: %.1f GB/s (%d rows)\n", blocks, (double)nsel * 512 / (ms * 1e-3) / 1e9, nsel);
    }
  }
  for (int blocks : {148 * 8, 148 * 16}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(flush, rep, 512 << 20);
      cudaEventRecord(e0); gather_kv512<<<blocks, 256>>>(K, idx, nsel / 2, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("gather interleaved 512B blocks=%d: %.1f GB/s\n", blocks, (double)(nsel / 2) * 512 / (ms * 1e-3) / 1e9);
    }
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(flush, rep, 512 << 20);
    cudaEventRecord(e0); stream_k<<<148 * 8, 256>>>(K, rows * 16, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep == 2) printf("stream: %.1f GB/s\n", (double)rows * 256 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
