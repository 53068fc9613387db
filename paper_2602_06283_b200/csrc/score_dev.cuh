// cp.async / mbarrier / bulk-copy helpers and the score kernel's tile staging,
// shared by the score kernels (tables_score.cu) and the one-launch step (spread.cu).
#pragma once
#include "step_dev.cuh"

namespace sk {

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cpa16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Stage layout of one tile (32 keys) in a warp's ring: LP*32 bytes of codes in
// the global tile order (chunk ch of key lane at ch*32*CB + lane*CB), then 32
// fp32 value norms.  A lane copies exactly the bytes it later reads.
template <int LP>
struct TileStage {
  static constexpr int CB = LP < 16 ? LP : 16;
  static constexpr int NCH = LP / CB;
  static constexpr int CODE_BYTES = LP * 32;
  static constexpr int BYTES = CODE_BYTES + 128;
};

template <int LP>
__device__ __forceinline__ void issue_tile(uint32_t st, const uint8_t* tile_codes, const float* tile_vn,
                                           int lane) {
  constexpr int CB = TileStage<LP>::CB;
#pragma unroll
  for (int ch = 0; ch < TileStage<LP>::NCH; ++ch) {
    const uint32_t off = ch * (32 * CB) + lane * CB;
    if constexpr (CB == 16) cpa16(st + off, tile_codes + off);
    else cpa8(st + off, tile_codes + off);
  }
  cpa4(st + TileStage<LP>::CODE_BYTES + lane * 4, tile_vn + lane);
}

}  // namespace sk
