// Alg. 1 PrecomputeKeyHashes on the 5th-generation tensor
// cores: X[keys x (Lp*8)] = K_tile[keys x 128] . W^T[128 x (Lp*8)] with
// tcgen05.mma (kind::f16, bf16 inputs, fp32 accumulation in tensor memory),
// then sign -> bit i of table l (R-3, R-4) and a byte per (key, table) in the
// bank-rotated code layout.
//
// Persistent, warp-specialized CTA (one per SM), described at the kernel
// below; W (Lp tables x 8 rows, rows i >= P and tables l >= L zero) stays
// resident in shared memory in the canonical no-swizzle K-major core-matrix
// layout:
//   byte(row n, element d) = ((d / 8) * (NC / 8) + n / 8) * 128 + (n % 8) * 16 + (d % 8) * 2
// (core matrix = 8 rows x 16 B; SBO = 128 B between 8-row groups, LBO =
// NC/8 * 128 B between the two 8-element K chunks of one MMA).
// fp32 accumulation order differs from the CUDA-core path, so bits whose
// projection is within rounding of 0 may differ; both are checked against the
// fp64 oracle under the margin rule (tests/test_gpu_parity.py).
#include <cuda.h>

#include "internal.cuh"

namespace sk {

constexpr int kTcM = 128;                     // keys per tile (UMMA_M)
constexpr int kTcK = kD;                      // 128 = 8 k-steps of 16

__device__ __forceinline__ void tc_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "TCW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TCW_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase));
}
__device__ __forceinline__ void tc_cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}

// tcgen05 shared-memory matrix descriptor, no swizzle, K-major
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                          // version = 1 (sm_100)
  return d;                                        // base offset 0, layout SWIZZLE_NONE
}

// ----------------------------------------------------------------------------
// Warp-specialized, MMA overlapped with the epilogue.
//   warp 0 (1 lane): TMA producer -- 16 tensor-map box loads {8 elems, 128 rows}
//                    per 128-key tile land each K chunk directly in the
//                    core-matrix layout; 2-stage ring (full/empty mbarriers);
//   warp 1 (1 lane): MMA issuer -- per chunk of MMA_N output columns, 8 k-step
//                    tcgen05.mma into a TMEM slot (512 / MMA_N slots in a ring),
//                    tcgen05.commit -> slot full; after a tile, commit -> A stage empty;
//   warps 2..17:     epilogue -- warp w reads TMEM lanes 32 (w % 4) .. +31 and one
//                    quarter of the chunk's columns, sign-packs into a staging tile
//                    (double-buffered by tile), releases the slot; after a tile the
//                    16 warps copy the staging tile out with 16-byte stores.
// ----------------------------------------------------------------------------
#ifndef SK_EPI_WARPS
#define SK_EPI_WARPS 20
#endif
constexpr int kEpiWarps = SK_EPI_WARPS;   // a multiple of 4 (one group per TMEM lane quadrant)
constexpr int kTc2Threads = 64 + kEpiWarps * 32;   // producer warp, MMA warp, epilogue warps
constexpr int kColSplit = kEpiWarps / 4;            // epilogue warps per TMEM lane quadrant

__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* tm, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Sign packing (epilogue below): bit i = (x_i >= 0) is the inverted fp32 sign
// bit.  One funnel shift per column collects 32 sign bits (column c in bit
// 31 - c), __brev puts column c in bit c, so byte q is table q of the 32
// columns.  (An fp32 sum of exactly -0.0 -- all products -0 -- would read as
// negative here; it cannot occur unless all 128 products are negative zeros.)
template <int NC>
__global__ void __launch_bounds__(kTc2Threads, 1)
hash_keys_tc2_kernel(const __grid_constant__ CUtensorMap tmK, const uint16_t* __restrict__ W,
                     uint8_t* __restrict__ codes, int BH, int N_max, int L, int P, int n_begin,
                     int n_end) {
  constexpr int LP = NC / 8;
  constexpr int MMA_N = NC < 256 ? NC : 256;
  constexpr int NCHK = NC / MMA_N;                 // chunks per tile
  constexpr int NSLOT = 512 / MMA_N;               // TMEM chunk slots
  constexpr uint32_t W_BYTES = NC * kTcK * 2;
  constexpr uint32_t A_BYTES = kTcM * kTcK * 2;    // 32 KB
  constexpr int RS = LP / 4 + 1;                   // staging row stride (u32 words, odd: conflict-free)
  constexpr uint32_t STG_BYTES = kTcM * RS * 4;
  constexpr int CB = LP < 16 ? LP : 16;
  constexpr int NCH = LP / CB;
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(MMA_N >> 3) << 17) |
                             ((uint32_t)(kTcM >> 4) << 24);
  extern __shared__ __align__(1024) char smem[];
  char* sW = smem;
  char* sA = smem + W_BYTES;                       // 2 stages
  uint32_t* stage = reinterpret_cast<uint32_t*>(smem + W_BYTES + 2 * A_BYTES);   // 2 x [kTcM][RS] words
  __shared__ uint64_t full_A[2], empty_A[2], full_T[NSLOT], empty_T[NSLOT];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sW_u = smem_u32(sW), sA_u = smem_u32(sA);

  // ---- setup: W resident, barriers, TMEM ----------------------------------------
  for (int c = tid; c < NC * (kTcK / 8); c += kTc2Threads) {
    const int n = c / (kTcK / 8), kc = c % (kTcK / 8);
    const int l = n >> 3, i = n & 7;
    const bool v = l < L && i < P;
    const uint16_t* src = W + ((size_t)(v ? l : 0) * P + (v ? i : 0)) * kD + kc * 8;
    tc_cp16(sW_u + (uint32_t)((kc * (NC / 8) + (n >> 3)) * 128 + (n & 7) * 16), src, v);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) { tc_mbar_init(&full_A[i], 1); tc_mbar_init(&empty_A[i], 1); }
    for (int i = 0; i < NSLOT; ++i) { tc_mbar_init(&full_T[i], 1); tc_mbar_init(&empty_T[i], kEpiWarps); }
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // W visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  const int t_lo = n_begin / kTcM, t_hi = (n_end - 1) / kTcM;
  const int tiles_in_range = t_hi - t_lo + 1;
  const long long total = (long long)BH * tiles_in_range;

  if (warp == 0) {
    if (lane == 0) {                                             // ---- TMA producer
      int it = 0;
      for (long long t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        const int s = it & 1;
        tc_mbar_wait(&empty_A[s], ((it >> 1) & 1) ^ 1);
        const int bh = (int)(t / tiles_in_range), tile = t_lo + (int)(t % tiles_in_range);
        const int row0 = bh * N_max + tile * kTcM;
        mbar_arrive_expect(&full_A[s], A_BYTES);
#pragma unroll
        for (int kc = 0; kc < kTcK / 8; ++kc)
          tma_load_2d(sA_u + s * A_BYTES + kc * (kTcM / 8) * 128, &tmK, kc * 8, row0, &full_A[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {                                             // ---- MMA issuer
      int it = 0, c = 0;
      for (long long t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        const int s = it & 1;
        tc_mbar_wait(&full_A[s], (it >> 1) & 1);
        for (int h = 0; h < NCHK; ++h, ++c) {
          const int slot = c % NSLOT, use = c / NSLOT;
          tc_mbar_wait(&empty_T[slot], (use & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int ks = 0; ks < kTcK / 16; ++ks) {
            const uint64_t ad = umma_desc(sA_u + s * A_BYTES + ks * 2 * (kTcM / 8) * 128,
                                          (kTcM / 8) * 128, 128);
            const uint64_t bd = umma_desc(sW_u + ks * 2 * (NC / 8) * 128 + h * (MMA_N / 8) * 128,
                                          (NC / 8) * 128, 128);
            const uint32_t acc = ks > 0 ? 1u : 0u;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + slot * MMA_N),
                "l"(ad), "l"(bd), "r"(IDESC), "r"(acc));
          }
          umma_commit(&full_T[slot]);
        }
        umma_commit(&empty_A[s]);                                // A stage free after these MMAs
      }
    }
  } else {                                                       // ---- epilogue warps
    const int ew = warp - 2;
    const int qd = warp & 3;                                     // TMEM lane quadrant of this warp
    const int cpart = ew >> 2;                                   // which part of the chunk's columns
    const int r = qd * 32 + lane;                                // key row of this thread
    constexpr int MM = (LP < 32 ? LP : 32) - 1;
    constexpr int PART = MMA_N / kColSplit;                      // columns per warp and chunk
#if SK_EPI_WARPS == 16
    constexpr int GROUPS = PART >= 32 ? PART / 32 : 1;           // x32 loads per warp and chunk
#else
    constexpr int GROUPS = ((MMA_N >= 32 ? MMA_N / 32 : 1) + kColSplit - 1) / kColSplit;
#endif
    int it = 0, c = 0;
    for (long long t = blockIdx.x; t < total; t += gridDim.x, ++it) {
      const int bh = (int)(t / tiles_in_range), tile = t_lo + (int)(t % tiles_in_range);
      uint32_t* stg = stage + (it & 1) * (STG_BYTES / 4);
      for (int h = 0; h < NCHK; ++h, ++c) {
        const int slot = c % NSLOT, use = c / NSLOT;
        tc_mbar_wait(&full_T[slot], use & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
        for (int g = 0; g < GROUPS; ++g) {
#if SK_EPI_WARPS == 16
          const int col = PART >= 32 ? cpart * PART + g * 32 : cpart * 32;   // within the chunk
          if (col >= MMA_N) break;                               // narrow chunks: fewer busy warps
#else
          // 32-column groups of the whole tile dealt round-robin to the quadrant's
          // kColSplit warps: tile group gg = h * (MMA_N / 32) + col / 32
          constexpr int GPC = MMA_N >= 32 ? MMA_N / 32 : 1;     // groups per chunk
          int gg0 = h * GPC;
          gg0 += ((cpart - gg0) % kColSplit + kColSplit) % kColSplit;   // first tile group of mine in chunk h
          const int gg = gg0 + g * kColSplit;
          if (gg >= (h + 1) * GPC) break;
          const int col = (gg - h * GPC) * 32;
          if (col >= MMA_N) break;
#endif
          uint32_t v[32];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
              "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
                "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
                "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
              : "r"(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(slot * MMA_N + col)));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          // 32 sign bits with one funnel shift per column (column c lands in bit
          // 31 - c), inverted (bit = x >= 0) and bit-reversed: byte qq = the code
          // of table lb + qq (bit i = (x_i >= 0), i < P; padding tables >= L -> 0),
          // staged as one word in TABLE order (the copy-out applies the slot rotation)
          // four independent 8-column funnel-shift chains (dependency depth 8 + 2;
          // one 32-deep chain measured 0.452 vs 0.448 ms at the bench cache)
          uint32_t q0 = 0, q1 = 0, q2 = 0, q3 = 0;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            q0 = __funnelshift_l(v[c], q0, 1);
            q1 = __funnelshift_l(v[8 + c], q1, 1);
            q2 = __funnelshift_l(v[16 + c], q2, 1);
            q3 = __funnelshift_l(v[24 + c], q3, 1);
          }
          const uint32_t sg = __byte_perm(__byte_perm(q3, q2, 0x0040), __byte_perm(q1, q0, 0x0040), 0x5410);
          const int lb = (h * MMA_N + col) / 8;
          const uint32_t lmask = lb + 4 <= L ? 0xFFFFFFFFu : (lb >= L ? 0u : (0xFFFFFFFFu >> (8 * (lb + 4 - L))));
          stg[r * RS + (lb >> 2)] = __brev(~sg) & (((1u << P) - 1u) * 0x01010101u) & lmask;
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive1(&empty_T[slot]);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");   // staging tile complete
      uint8_t* cbase = codes + (size_t)bh * N_max * LP + (size_t)tile * kTcM * LP;
      for (int x = ew * 32 + lane; x < kTcM * NCH; x += kEpiWarps * 32) {
        const int ch = x / kTcM, rr = x % kTcM;
        const int jj = tile * kTcM + rr;
        if (jj < n_begin || jj >= n_end) continue;
        const int off = ((rr >> 5) * NCH + ch) * (32 * CB) + (rr & 31) * CB;
        // slot s of key jj holds table (s & ~MM) | ((s + jj) & MM): output word w =
        // 4 consecutive tables of the row's group, a funnel shift of 2 staged words
        const uint32_t* srow = stg + rr * RS;
        uint32_t o[CB / 4];
#pragma unroll
        for (int w = 0; w < CB / 4; ++w) {
          const int s0 = ch * CB + 4 * w;
          const int gb = (s0 & ~MM) >> 2;                        // group base (words)
          const int bq = (s0 + rr) & MM;                         // first table of the word (tile*128 = 0 mod 32)
          const uint32_t lo = srow[gb + (bq >> 2)], hi = srow[gb + (((bq >> 2) + 1) & (MM >> 2))];
          o[w] = __funnelshift_r(lo, hi, 8 * (bq & 3));
        }
        if constexpr (CB == 16) *reinterpret_cast<uint4*>(cbase + off) = make_uint4(o[0], o[1], o[2], o[3]);
        else *reinterpret_cast<uint2*>(cbase + off) = make_uint2(o[0], o[1]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

static socket_status launch_hash_keys_tc2(const socket_cfg& c, const void* K, const void* W,
                                          uint8_t* codes, int n_begin, int n_count, cudaStream_t st,
                                          bool* used) {
  *used = false;
  PFN_encodeTiled enc = get_encode();
  if (!enc) return SOCKET_OK;
  const int Lp = code_slots(c.L);
  const int NC = Lp * 8;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)kD, (cuuint64_t)c.B * c.H_kv * c.N_max};
  cuuint64_t strides[1] = {(cuuint64_t)kD * 2};
  cuuint32_t box[2] = {8, (cuuint32_t)kTcM};
  cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(K), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return SOCKET_OK;
  const int t_lo = n_begin / kTcM, t_hi = (n_begin + n_count - 1) / kTcM;
  const long long total = (long long)c.B * c.H_kv * (t_hi - t_lo + 1);
  const int grid = (int)(total < num_sms() ? total : num_sms());
  const size_t smem = (size_t)NC * kTcK * 2 + 2 * (size_t)kTcM * kTcK * 2 + 2 * (size_t)kTcM * (Lp / 4 + 1) * 4;
#define SK_TC2(NCV)                                                                                 \
  case NCV: {                                                                                       \
    cudaFuncSetAttribute(hash_keys_tc2_kernel<NCV>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                         (int)smem);                                                                \
    hash_keys_tc2_kernel<NCV><<<grid, kTc2Threads, smem, st>>>(tm, (const uint16_t*)W, codes,      \
                                                               c.B * c.H_kv, c.N_max, c.L, c.P,    \
                                                               n_begin, n_begin + n_count);        \
    break;                                                                                          \
  }
  switch (NC) {
    SK_TC2(64)
    SK_TC2(128)
    SK_TC2(256)
    SK_TC2(512)
    default:
      return SOCKET_OK;
  }
#undef SK_TC2
  *used = true;
  return check_launch("hash_keys_tc2_kernel");
}

socket_status launch_hash_keys_tc(const socket_cfg& c, const void* K, const void* W,
                                  uint8_t* codes, int n_begin, int n_count, cudaStream_t st,
                                  bool* used) {
  *used = false;
  if (c.P > 8) return SOCKET_OK;   // wide codes: CUDA-core path
  const int Lp = code_slots(c.L);
  const int NC = Lp * 8;
  if (NC > 512 || n_count < kTcM) return SOCKET_OK;    // CUDA-core path
  return launch_hash_keys_tc2(c, K, W, codes, n_begin, n_count, st, used);
}

}  // namespace sk
