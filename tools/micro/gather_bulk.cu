// Sorted random 256-B K/V row gathers (the sparse decode's access pattern, 10%
// of 4M rows): 16-B cp.async per thread (the decode kernel's way) vs one TMA 1-D
// bulk copy (cp.async.bulk, 256 B) per row into shared memory.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_bulk gather_bulk.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// warp per 16 selected rows per iteration; 4 stages in flight per warp
constexpr int WPB = 4;   // warps per CTA; 4 stages x 8 KB per warp (128 KB dynamic smem)
typedef uint4 Buf[4][2][16][16];   // [stage][K/V][row][16-B chunk]
__global__ void __launch_bounds__(128) gather_cpasync(const uint4* K, const uint4* V, const int* idx, int nsel, int* out) {
  extern __shared__ __align__(128) Buf buf[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * WPB + warp, nw = gridDim.x * WPB;
  int acc = 0;
  int it = 0;
  for (int base = gw * 16; base < nsel; base += nw * 16, ++it) {
    const int st = it & 3;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = q * 2 + (lane >> 4), c = lane & 15;
      const int i = base + r;
      const int t = i < nsel ? idx[i] : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&buf[warp][st][0][r][c])), "l"(K + (size_t)t * 16 + c));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&buf[warp][st][1][r][c])), "l"(V + (size_t)t * 16 + c));
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 3;");
    acc += buf[warp][(it + 1) & 3][0][lane & 15][0].x;
  }
  asm volatile("cp.async.wait_group 0;");
  if (acc == 0x12345678) out[0] = acc;
}

__global__ void __launch_bounds__(128) gather_bulk(const uint4* K, const uint4* V, const int* idx, int nsel, int* out) {
  extern __shared__ __align__(128) Buf buf[];
  __shared__ __align__(8) unsigned long long bar[WPB][4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * WPB + warp, nw = gridDim.x * WPB;
  if (lane < 4) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[warp][lane])));
  __syncwarp();
  asm volatile("fence.mbarrier_init.release.cluster;");
  int acc = 0;
  int it = 0;
  unsigned phase[4] = {0, 0, 0, 0};
  for (int base = gw * 16; base < nsel; base += nw * 16, ++it) {
    const int st = it & 3;
    if (it >= 4) {   // stage reuse: wait for its previous fill
      unsigned p;
      do {
        asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q;}"
                     : "=r"(p) : "r"(smem_u32(&bar[warp][st])), "r"(phase[st]));
      } while (!p);
      phase[st] ^= 1;
      acc += buf[warp][st][0][lane & 15][0].x;
    }
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[warp][st])), "r"(16 * 2 * 256));
    __syncwarp();
    if (lane < 16) {   // lane r: the K and V rows of selected row r (two 256-B bulk copies)
      const int i = base + lane;
      const int t = i < nsel ? idx[i] : 0;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
                       smem_u32(&buf[warp][st][0][lane][0])), "l"(K + (size_t)t * 16), "r"(smem_u32(&bar[warp][st])) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
                       smem_u32(&buf[warp][st][1][lane][0])), "l"(V + (size_t)t * 16), "r"(smem_u32(&bar[warp][st])) : "memory");
    }
  }
  for (int s = 0; s < 4 && s < it; ++s) {   // drain
    const int st = (it + s) & 3;
    unsigned p;
    do {
      asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q;}"
                   : "=r"(p) : "r"(smem_u32(&bar[warp][st])), "r"(phase[st]));
    } while (!p);
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  const size_t rows = 16ull * 8 * 32768;   // 4M rows of 256 B per tensor
  uint4 *K, *V; int *idx, *o;
  cudaMalloc(&K, rows * 256); cudaMalloc(&V, rows * 256); cudaMalloc(&o, 64);
  cudaMemset(K, 1, rows * 256); cudaMemset(V, 2, rows * 256);
  std::vector<int> h; srand(1);
  for (size_t r = 0; r < rows; ++r) if (rand() % 10 == 0) h.push_back((int)r);
  const int nsel = (int)h.size();
  cudaMalloc(&idx, nsel * 4); cudaMemcpy(idx, h.data(), nsel * 4, cudaMemcpyHostToDevice);
  void* flush; cudaMalloc(&flush, 512 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const size_t sm = sizeof(Buf) * WPB;
  cudaFuncSetAttribute(gather_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(gather_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  printf("dynamic smem per CTA %zu B\n", sm);
  for (int kind = 0; kind < 2; ++kind) {
    for (int blocks : {148}) {
      float tot = 0.f;
      for (int rep = 0; rep < 6; ++rep) {
        cudaMemset(flush, rep, 512 << 20);
        cudaEventRecord(e0);
        if (kind == 0) gather_cpasync<<<blocks, 128, sm>>>(K, V, idx, nsel, o);
        else gather_bulk<<<blocks, 128, sm>>>(K, V, idx, nsel, o);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep >= 1) tot += ms;
      }
      const float ms = tot / 5;
      printf("%s blocks=%d: %.1f GB/s (%s)\n", kind ? "bulk 256B" : "cp.async 16B", blocks,
             (double)nsel * 512 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
