// Alg. 2 SoftBucketProbs and Eq. 4 / Alg. 4 soft
// collision scoring (l.183-188, l.1485-1506).
//
// query_tables_kernel: per (b, selection row) builds T^(l)(r) for all tables:
//   u_{l,i} = tanh(W^(l)_i . q) / sqrt(d),  p(r) = prod_i sigma(2 u_i c_{r,i} / tau)
//   (exact product form of the corner softmax), summed over the group's query
//   heads in KV_SHARED mode.  It writes the plain [L][R] tables and/or the
//   score kernel's shared-memory image ("LUT"): panels of [256 rows][64 cols]
//   fp32 where column c holds table c (Lp >= 32) or table c mod Lp (Lp < 32).
//
// score_kernel: streams the tiled codes with 128-bit loads, lane = key j mod
// 32.  At slot step s lane l reads LUT column (s & 32) | ((s + l) & 31), so the
// 32 lanes hit 32 distinct banks (conflict-free).
#include "internal.cuh"

namespace sk {

constexpr int kTabThreads = 256;
constexpr int kTabPerCta = 4;     // tables per CTA
constexpr int kMaxHeads = 8;      // heads per selection row

// One CTA = (b, selection row) x 8 tables.  Steps (all latency-oriented):
//  1. stage q (NH heads) and W^(l) of the 8 tables in shared memory (16-B loads);
//  2. one thread per (head, table, bit): x = W_i . q in fp64 (bf16 products are
//     exact), u = tanh(x)/sqrt(d), factors sigma(+-2u/tau) in fp64;
//  3. half tables lo(r & 15) = prod_{i<4} f_i, hi(r >> 4) = prod_{i>=4} f_i in
//     fp64, rounded once to fp32;
//  4. T(r) = sum_h lo_h * hi_h; consecutive threads write consecutive table
//     columns of one LUT row (coalesced 32-byte segments).
__global__ void __launch_bounds__(kTabThreads)
query_tables_kernel(const uint16_t* __restrict__ q, const uint16_t* __restrict__ W,
                    float* __restrict__ plain, float* __restrict__ lut, int H_q, int H_sel,
                    int NH, int L, int P, int Lp, float tau) {
  __shared__ float qs[kMaxHeads][kD];
  __shared__ float wsm[kTabPerCta * 8][kD + 1];
  __shared__ double fx[kMaxHeads][kTabPerCta][8][2];        // sigma factors
  __shared__ float half_lo[kMaxHeads][16][kTabPerCta];
  __shared__ float half_hi[kMaxHeads][16][kTabPerCta];
  const int row = blockIdx.x;                // b * H_sel + r
  const int b = row / H_sel, r = row % H_sel;
  const int h0 = (NH == 1) ? r : r * NH;     // first query head of the row
  const int l0 = blockIdx.y * kTabPerCta;
  const int R = 1 << P;
  const int tid = threadIdx.x;
  // 1. staging
  for (int i = tid; i < NH * (kD / 8); i += kTabThreads) {
    const int h = i / (kD / 8), c = i % (kD / 8);
    const uint4 u = *reinterpret_cast<const uint4*>(q + ((size_t)b * H_q + h0 + h) * kD + c * 8);
    const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      qs[h][c * 8 + 2 * e] = bf16lo(w4[e]);
      qs[h][c * 8 + 2 * e + 1] = bf16hi(w4[e]);
    }
  }
  const int nrows_w = kTabPerCta * P;        // W rows of this CTA
  for (int i = tid; i < nrows_w * (kD / 8); i += kTabThreads) {
    const int wr = i / (kD / 8), c = i % (kD / 8);
    const int l = l0 + wr / P;
    uint4 u = make_uint4(0, 0, 0, 0);
    if (l < L) u = *reinterpret_cast<const uint4*>(W + ((size_t)l * P + wr % P) * kD + c * 8);
    const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      wsm[wr][c * 8 + 2 * e] = bf16lo(w4[e]);
      wsm[wr][c * 8 + 2 * e + 1] = bf16hi(w4[e]);
    }
  }
  __syncthreads();
  // 2. projections and logistic factors: every product of
  //    two bf16 values is exact in fp32; each half of the 128-term sum is
  //    accumulated with TwoSum compensation by one of two threads, and the
  //    halves are merged in fp64, so x is exact to ~2^-48.  u = tanh(x)/sqrt(d)
  //    and sigma(+-2u/tau) use the accurate fp32 functions (<= 2 ulp each), so a
  //    factor carries <= 3 ulp + 3 ulp * |a|; no fp64 transcendentals.
  const float inv_sqrt_d = 0.08838834764831845f;   // 1/sqrt(128), correctly rounded
  const int ndots = NH * nrows_w;
  for (int base = 0; base < 2 * ndots; base += kTabThreads) {   // uniform trip count
    const int di2 = base + tid;
    const bool act = di2 < 2 * ndots;
    const int di = act ? di2 >> 1 : 0, part = di2 & 1;            // two threads per dot
    const int wr = di % nrows_w, h = di / nrows_w;
    float s0 = 0.f, c0 = 0.f;
    const int t0 = part * (kD / 2);
#pragma unroll 8
    for (int t = t0; t < t0 + kD / 2; ++t) {
      const float p0 = wsm[wr][t] * qs[h][t];       // exact
      const float u0 = s0 + p0, b0 = u0 - s0;
      c0 += (s0 - (u0 - b0)) + (p0 - b0);
      s0 = u0;
    }
    const double mine = (double)s0 + (double)c0;
    const double other = __shfl_xor_sync(0xffffffffu, mine, 1);
    if (act && part == 0) {
      const float x = (float)(mine + other);
      const float uu = tanhf(x) * inv_sqrt_d;       // Alg. 2 l.217
      const float a = 2.0f * uu / tau;              // logit gap of bit i
      fx[h][wr / P][wr % P][1] = (double)(1.0f / (1.0f + expf(-a)));   // c_{r,i} = +1 (bit set)
      fx[h][wr / P][wr % P][0] = (double)(1.0f / (1.0f + expf(a)));    // c_{r,i} = -1
    }
  }
  __syncthreads();
  // 3. half tables (bits 0..3 and 4..P-1; an empty product is 1)
  for (int i = tid; i < NH * kTabPerCta * 32; i += kTabThreads) {
    const int e = i & 15, hi = (i >> 4) & 1, tl = (i >> 5) % kTabPerCta, h = i / (32 * kTabPerCta);
    double p = 1.0;
#pragma unroll
    for (int bit = 0; bit < 4; ++bit) {
      const int ib = hi * 4 + bit;
      if (ib < P) p *= fx[h][tl][ib][(e >> bit) & 1];
    }
    if (hi) half_hi[h][e][tl] = (float)p; else half_lo[h][e][tl] = (float)p;
  }
  __syncthreads();
  // 4. entries: thread -> (row rr, table tl) with tl fastest
  const int panels = Lp <= 64 ? 1 : (Lp + 63) / 64;
  float* lrow = lut ? lut + (size_t)row * panels * (256 * 64) : nullptr;
  for (int e = tid; e < 256 * kTabPerCta; e += kTabThreads) {
    const int tl = e % kTabPerCta, rr = e / kTabPerCta;
    const int l = l0 + tl;
    if (l >= Lp) continue;
    float T = 0.f;
    if (l < L && rr < R) {
      for (int h = 0; h < NH; ++h) T = fmaf(half_lo[h][rr & 15][tl], half_hi[h][rr >> 4][tl], T);
      if (plain) plain[((size_t)row * L + l) * R + rr] = T;
    }
    if (lrow) {
      if (Lp >= 32) {
        lrow[(size_t)(l >> 6) * (256 * 64) + rr * 64 + (l & 63)] = T;
      } else {
        for (int cc = l; cc < 32; cc += Lp) lrow[rr * 64 + cc] = T;
      }
    }
  }
}

socket_status launch_query_tables(const socket_cfg& c, const void* q, const void* W,
                                  float* plain, float* lut, cudaStream_t st) {
  const int H_sel = num_sel_rows(c);
  const int NH = c.group_mode == SOCKET_GROUP_PER_QHEAD ? 1 : c.H_q / c.H_kv;
  if (NH > kMaxHeads) return fail(SOCKET_EUNSUPPORTED, "more than 8 query heads per KV head");
  const int Lp = code_slots(c.L);
  dim3 grid(c.B * H_sel, (Lp + kTabPerCta - 1) / kTabPerCta);
  query_tables_kernel<<<grid, kTabThreads, 0, st>>>((const uint16_t*)q, (const uint16_t*)W, plain,
                                                    lut, c.H_q, H_sel, NH, c.L, c.P, Lp, c.tau);
  return check_launch("query_tables_kernel");
}

// ----------------------------------------------------------------------------
// score kernel
// ----------------------------------------------------------------------------
constexpr int kScoreThreads = 256;
constexpr int kScoreWarps = kScoreThreads / 32;

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes));
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

template <int LP>
struct CodeRegs {
  static constexpr int CB = LP < 16 ? LP : 16;
  static constexpr int NCH = LP / CB;
  static constexpr int NW = LP / 4;   // u32 words per key
  uint32_t w[NW];
};

template <int LP>
__device__ __forceinline__ void load_codes(CodeRegs<LP>& c, const uint8_t* tile_base, int lane) {
  constexpr int CB = CodeRegs<LP>::CB;
#pragma unroll
  for (int ch = 0; ch < CodeRegs<LP>::NCH; ++ch) {
    const uint8_t* p = tile_base + ch * (32 * CB) + lane * CB;
    if constexpr (CB == 16) {
      const uint4 v = ldg_nc_v4(p);
      c.w[ch * 4 + 0] = v.x; c.w[ch * 4 + 1] = v.y; c.w[ch * 4 + 2] = v.z; c.w[ch * 4 + 3] = v.w;
    } else {
      const uint2 v = ldg_nc_v2(p);
      c.w[ch * 2 + 0] = v.x; c.w[ch * 2 + 1] = v.y;
    }
  }
}

// sum over slots of LUT[code][column(s, lane)], two keys per lane sharing columns
template <int LP, int NK>
__device__ __forceinline__ void lookup_sum(const CodeRegs<LP> (&c)[NK], float (&acc)[NK],
                                           const char* lut, int lane) {
#pragma unroll
  for (int k = 0; k < NK; ++k) acc[k] = 0.f;
#pragma unroll
  for (int s = 0; s < LP; ++s) {
    // column within its 64-wide panel, times 4 bytes (fits in one byte)
    const uint32_t col4 = (uint32_t)(((s & 32) | ((s + lane) & 31)) << 2);
    constexpr int dummy = 0;
    (void)dummy;
    const uint32_t sel = 0x5504u | ((uint32_t)(s & 3) << 4);
    const char* panel = lut + (size_t)(s >> 6) * (256 * 64 * 4);
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const uint32_t addr = __byte_perm(c[k].w[s >> 2], col4, sel);  // code*256 + col*4
      acc[k] += *reinterpret_cast<const float*>(panel + addr);
    }
  }
}

template <int LP>
__global__ void __launch_bounds__(kScoreThreads, 2)
score_kernel(const float* __restrict__ lut_g, const uint8_t* __restrict__ codes,
             const float* __restrict__ vnorm, const int32_t* __restrict__ seq_lens,
             const uint8_t* __restrict__ mask, float* __restrict__ scores, int H_sel, int H_kv,
             int G_sel, int N_max, long long total_tiles) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t bar;
  constexpr int PANELS = LP <= 64 ? 1 : (LP + 63) / 64;
  constexpr uint32_t LUT_BYTES = PANELS * 256 * 64 * 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_per_row = N_max >> 5;
  const long long t_begin = total_tiles * blockIdx.x / gridDim.x;
  const long long t_end = total_tiles * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t phase = 0;
  long long t = t_begin;
  while (t < t_end) {
    const int row = (int)(t / tiles_per_row);
    const long long row_end = (long long)(row + 1) * tiles_per_row;
    const long long seg_end = row_end < t_end ? row_end : t_end;
    const int b = row / H_sel, r = row % H_sel;
    const int g = r / G_sel;                       // kv head of this selection row
    const int n = seq_lens[b];
    const int valid_tiles = (n + 31) >> 5;
    const int tile0 = (int)(t - (long long)row * tiles_per_row);
    const int tile1 = (int)(seg_end - (long long)row * tiles_per_row);
    const bool need_lut = tile0 < valid_tiles;
    if (need_lut && threadIdx.x == 0) {
      mbar_expect_tx(&bar, LUT_BYTES);
      const char* src = reinterpret_cast<const char*>(lut_g) + (size_t)row * LUT_BYTES;
      constexpr uint32_t kChunk = 32768;
#pragma unroll
      for (uint32_t off = 0; off < LUT_BYTES; off += kChunk) bulk_g2s(smem + off, src + off, kChunk, &bar);
    }
    const uint8_t* crow = codes + ((size_t)b * H_kv + g) * N_max * LP;
    const float* vrow = vnorm + ((size_t)b * H_kv + g) * N_max;
    const uint8_t* mrow = mask ? mask + (size_t)b * N_max : nullptr;
    float* srow = scores + (size_t)row * N_max;
    bool lut_ready = !need_lut;
    // each warp takes tile pairs (tt, tt + 8) with tt = tile0 + warp + 16 i; the
    // codes of the next pair are loaded while the current pair is looked up.
    auto load_pair = [&](CodeRegs<LP> (&c)[2], float (&vn)[2], int tt) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int ti = tt + u * kScoreWarps;
        if (ti < tile1 && ti < valid_tiles) {
          load_codes<LP>(c[u], crow + (size_t)ti * 32 * LP, lane);
          vn[u] = vrow[ti * 32 + lane];
        } else {
#pragma unroll
          for (int w = 0; w < CodeRegs<LP>::NW; ++w) c[u].w[w] = 0;
          vn[u] = 0.f;
        }
      }
    };
    auto finish_pair = [&](const CodeRegs<LP> (&c)[2], const float (&vn)[2], int tt) {
      const bool any_valid = tt < valid_tiles;
      float acc[2] = {0.f, 0.f};
      if (any_valid) {
        if (!lut_ready) { mbar_wait(&bar, phase); lut_ready = true; }
        lookup_sum<LP, 2>(c, acc, smem, lane);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int ti = tt + u * kScoreWarps;
        if (ti < tile1) {
          const int j = ti * 32 + lane;
          const bool ok = ti < valid_tiles && j < n && (!mrow || mrow[j]);
          srow[j] = ok ? vn[u] * acc[u] : -INFINITY;
        }
      }
    };
    CodeRegs<LP> ca[2], cb[2];
    float va[2], vb[2];
    int tt = tile0 + warp;
    if (tt < tile1) load_pair(ca, va, tt);
    while (tt < tile1) {
      const int t2 = tt + 2 * kScoreWarps;
      if (t2 < tile1) load_pair(cb, vb, t2);
      finish_pair(ca, va, tt);
      if (t2 >= tile1) break;
      const int t3 = t2 + 2 * kScoreWarps;
      if (t3 < tile1) load_pair(ca, va, t3);
      finish_pair(cb, vb, t2);
      tt = t3;
    }
    if (need_lut) {
      if (!lut_ready) mbar_wait(&bar, phase);
      phase ^= 1;
    }
    __syncthreads();   // everyone done with this LUT before it is overwritten
    t = seg_end;
  }
}

socket_status launch_score(const socket_cfg& c, const float* lut, const uint8_t* codes,
                           const float* vnorm, const int32_t* seq_lens, const uint8_t* mask,
                           float* scores, cudaStream_t st) {
  const int Lp = code_slots(c.L);
  const int H_sel = num_sel_rows(c);
  const int G_sel = c.group_mode == SOCKET_GROUP_PER_QHEAD ? c.H_q / c.H_kv : 1;
  const long long total_tiles = (long long)c.B * H_sel * (c.N_max / 32);
  const size_t smem = lut_bytes_per_row(c.L);
  long long grid = 2 * kNumSMs;
  if (grid > total_tiles) grid = total_tiles;
  if (grid < 1) return SOCKET_OK;
#define SK_SCORE_CASE(LPV)                                                                     \
  case LPV: {                                                                                  \
    auto kfn = score_kernel<LPV>;                                                              \
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
    kfn<<<(unsigned)grid, kScoreThreads, smem, st>>>(lut, codes, vnorm, seq_lens, mask, scores, \
                                                      H_sel, c.H_kv, G_sel, c.N_max,           \
                                                      total_tiles);                            \
    return check_launch("score_kernel");                                                       \
  }
  switch (Lp) {
    SK_SCORE_CASE(8)
    SK_SCORE_CASE(16)
    SK_SCORE_CASE(32)
    SK_SCORE_CASE(64)
    SK_SCORE_CASE(96)
    SK_SCORE_CASE(128)
    default:
      return fail(SOCKET_EUNSUPPORTED, "score: L > 128 not supported");
  }
#undef SK_SCORE_CASE
}

}  // namespace sk
