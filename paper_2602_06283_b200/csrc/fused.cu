// Fused small-batch decode step: one launch, one thread-
// block CLUSTER per selection row (b, kv head) in KV_SHARED mode, CS CTAs per
// cluster, CTA c owning the key slice [c S, (c+1) S):
//
//   A. tables (Alg. 2): CTA c projects q on the W rows of tables
//      [c tpc, (c+1) tpc) (fp64 tensor-core DMMA), builds their sigma factors,
//      half tables and LUT columns, and writes the columns into the LUT of
//      EVERY CTA of the cluster (distributed shared memory); with append, it
//      also hashes the newest key on those tables (Alg. 1) -> codes;
//   B. scores (Eq. 4 / Alg. 4): the CTA streams its slice's codes and norms,
//      scores = ||v|| * sum_l LUT, written to `scores` and kept in shared
//      memory as monotone keys (sink/window forced, invalid 0);
//   C. top-k (Alg. 3 l.244): topk_core over the cluster's shared-memory slices
//      (no score round trip); each CTA keeps its own selected rows;
//   D. sparse attention (Eq. 2, exact logits P:271): the CTA attends over its
//      selected rows (tensor-core MMA tiles, online softmax), and the cluster
//      merges the CS partial states by LSE through distributed shared memory.
//
// Same arithmetic as the multi-kernel path, stage by stage, except the split
// of the attention (per CTA slice here), so the outputs agree to fp32 rounding.
#include "mma_dev.cuh"
#include "score_dev.cuh"
#include "topk_dev.cuh"

namespace sk {

#ifdef SK_TRACE
static __device__ unsigned long long g_fused_trace[4096 * 8];
#define FU_STAMP(i)                                                                       \
  do {                                                                                    \
    if (threadIdx.x == 0) {                                                               \
      const int cta = blockIdx.y * gridDim.x + blockIdx.x;                                \
      if (cta < 4096) g_fused_trace[cta * 8 + (i)] = clock64();                           \
    }                                                                                     \
  } while (0)
extern "C" int socket_debug_fused_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_fused_trace, (size_t)n * sizeof(unsigned long long));
}
// this translation unit's copy of the top-k phase stamps (TK_TRACE in topk_dev.cuh)
extern "C" int socket_debug_fused_topk_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_topk_trace, (size_t)n * sizeof(unsigned long long));
}
#else
#define FU_STAMP(i) \
  do {              \
  } while (0)
#endif

constexpr int kFThreads = kTopkThreads;   // 512
constexpr int kFWarps = kFThreads / 32;
constexpr int kFScoreStages = 2;
constexpr int kFAttWarps = 8;
constexpr int kFAttStages = 2;
constexpr int kFLutBytes = 256 * 64 * 4;                                   // 64 KB
constexpr int kFRingBytes = kFWarps * kFScoreStages * TileStage<64>::BYTES; // 68 KB
constexpr int kFZone = kFLutBytes + kFRingBytes;                          // LUT + score ring
static_assert(kFZone >= kFAttWarps * kFAttStages * kTileBytes, "attention ring must fit the zone");
static_assert(128 * 8 * 8 + 128 * 72 * 4 + 8 * (8 * 2 * 16 + 2 * 16 * 16) * 4 <= kFRingBytes,
              "table staging must fit the ring zone");
constexpr int kFWs = 72;    // staged W row stride (floats): [t][w]
constexpr int kFQs = 8;     // staged q row stride (doubles): [t][h]

struct FusedArgs {
  const uint16_t* q;
  uint16_t* K;            // written at row seq_lens[b] - 1 when k_new is set
  uint16_t* V;
  const uint16_t* k_new;  // [B][H_kv][d] new rows, or null (already in the cache)
  const uint16_t* v_new;
  const uint16_t* W;
  uint8_t* codes;
  float* vnorm;
  const int32_t* seq_lens;
  const uint8_t* mask;
  float* scores;
  int32_t* idx;
  int32_t* cnt;
  uint16_t* out;
  float* lse;
  int H_q, H_kv, N_max, L, P, Lp, k, sink, window, do_append, hard;
  float tau, scale_log2;
  int S;     // keys per CTA slice (multiple of 128)
  int tpc;   // tables per CTA
};

size_t fused_smem_bytes(int S) { return (size_t)kFZone + (size_t)S * 4; }

template <int NH, int LP>
__global__ void __launch_bounds__(kFThreads, 1) fused_step_kernel(FusedArgs a) {
  extern __shared__ __align__(1024) char fsm[];
  __shared__ TopkShared TS;
  __shared__ float s_part[NH][kD + 2];          // this CTA's (m, l, o) per head (log2 units)
  __shared__ float s_ks[kD];
  __shared__ uint32_t s_bits[64];
  cg::cluster_group cluster = cg::this_cluster();
  const int c = (int)cluster.block_rank();
  const int CS = (int)cluster.num_blocks();
  const int row = blockIdx.y;                   // selection row = (b, kv head)
  const int b = row / a.H_kv, g = row % a.H_kv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P = a.P, L = a.L;
  const int n = a.seq_lens[b];
  float* lut = reinterpret_cast<float*>(fsm);
  uint32_t* keys = reinterpret_cast<uint32_t*>(fsm + kFZone);

  FU_STAMP(0);
  // cluster barrier phase 1 of 2: every CTA of the cluster must be running before
  // the LUT columns are pushed into its shared memory (waited for just before
  // the push, so the table work below hides it)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  // ===== A. tables of my tables + append of the newest key ========================
  const int l0 = c * a.tpc;
  const int ntab = max(0, min(a.tpc, LP - l0));           // my tables (incl. padding ones)
  const int nw = max(0, min(a.tpc, L - l0)) * P;          // my valid W rows
  {
    double* qs = reinterpret_cast<double*>(fsm + kFLutBytes);              // [t][kFQs]
    float* ws = reinterpret_cast<float*>(fsm + kFLutBytes + kD * kFQs * 8);  // [t][kFWs]
    float* s_fx = ws + kD * kFWs;                       // sigma factors [h][bit][c][table]
    float* s_half = s_fx + NH * 8 * 2 * 16;             // half tables [h][hi][entry][table]
    const int h0 = g * NH;
    {   // q: 8 (padded) vectors x 16 uint4; W: 64 rows x 16 uint4 -- all loads first
      uint4 vw[2], vq;
      const int m = tid & 7, cq = (tid >> 3) & 15;
      vq = make_uint4(0, 0, 0, 0);
      if (tid < 128 && m < NH) vq = __ldg(reinterpret_cast<const uint4*>(a.q + ((size_t)b * a.H_q + h0 + m) * kD) + cq);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = tid + u * kFThreads, w = e & 63, cw = e >> 6;
        vw[u] = make_uint4(0, 0, 0, 0);
        if (w < nw) vw[u] = __ldg(reinterpret_cast<const uint4*>(a.W + (size_t)(l0 * P + w) * kD) + cw);
      }
      if (tid < 128) {
        const uint32_t w4[4] = {vq.x, vq.y, vq.z, vq.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) qs[(cq * 8 + e) * kFQs + m] = (double)((e & 1) ? bf16hi(w4[e >> 1]) : bf16lo(w4[e >> 1]));
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = tid + u * kFThreads, w = e & 63, cw = e >> 6;
        const uint32_t w4[4] = {vw[u].x, vw[u].y, vw[u].z, vw[u].w};
#pragma unroll
        for (int e2 = 0; e2 < 8; ++e2) ws[(cw * 8 + e2) * kFWs + w] = (e2 & 1) ? bf16hi(w4[e2 >> 1]) : bf16lo(w4[e2 >> 1]);
      }
    }
    const bool app = a.do_append && n > 0 && n <= a.N_max;   // outgrown cache: no write
    if (app && tid < kD) {
      const size_t crow = (((size_t)b * a.H_kv + g) * a.N_max + n - 1) * kD;
      if (a.k_new) {   // the new rows come from k_new / v_new; CTA 0 stores them in the cache
        const size_t nrow = ((size_t)b * a.H_kv + g) * kD;
        const uint16_t kv = a.k_new[nrow + tid];
        s_ks[tid] = bf16lo((uint32_t)kv);
        if (c == 0) {
          a.K[crow + tid] = kv;
          a.V[crow + tid] = a.v_new[nrow + tid];
        }
      } else {
        s_ks[tid] = bf16lo((uint32_t)a.K[crow + tid]);
      }
    }
    __syncthreads();
    FU_STAMP(1);
    // x[h][w] = q_h . W_w in fp64 on the tensor cores: warp w owns W rows
    // 8 (w & 7) .. + 7 over the K half w >> 3; x = (K half 0) + (K half 1) -- the
    // same decomposition as the chained prologue's tables tiles, so the LUTs agree
    // bit for bit
    {
      const int nt8 = warp & 7, kh = warp >> 3;
      double d0 = 0.0, d1 = 0.0;
      const int kr = lane & 3, col = lane >> 2;
      if (nt8 * 8 < nw) {
#pragma unroll 8
        for (int k0 = kh * (kD / 2); k0 < (kh + 1) * (kD / 2); k0 += 4) {
          const double av = qs[(k0 + kr) * kFQs + col];
          const double bv = (double)ws[(k0 + kr) * kFWs + nt8 * 8 + col];
          dmma_8x8x4(d0, d1, av, bv);
        }
      }
      __syncthreads();                                   // qs dead: partials go there
      double* xp = qs;                                   // [kh][h 8][w 64]
      if (nt8 * 8 < nw) {
        xp[(kh * 8 + col) * 64 + nt8 * 8 + 2 * (lane & 3)] = d0;
        xp[(kh * 8 + col) * 64 + nt8 * 8 + 2 * (lane & 3) + 1] = d1;
      }
      __syncthreads();
      const float inv_sqrt_d = 0.08838834764831845f;
      if (kh == 0 && nt8 * 8 < nw) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int h = lane >> 2, w = nt8 * 8 + 2 * (lane & 3) + i;
          if (h < NH && w < nw) {
            const double x = xp[h * 64 + w] + xp[(8 + h) * 64 + w];
            const int tl = w / P, bit = w - tl * P;
            float fp, fm;
            if (a.hard) {
              fp = x >= 0.0 ? 1.f : 0.f;
              fm = 1.f - fp;
            } else {
              const float uu = tanhf((float)x) * inv_sqrt_d;            // Alg. 2 l.217
              const float av = 2.0f * uu / a.tau;
              fp = 1.0f / (1.0f + expf(-av));
              fm = 1.0f / (1.0f + expf(av));
            }
            s_fx[((h * 8 + bit) * 2 + 1) * 16 + tl] = fp;
            s_fx[((h * 8 + bit) * 2 + 0) * 16 + tl] = fm;
          }
        }
      }
    }
    // append: the newest key's bits on my tables, fp32 t-ascending (SIMT prefill order)
    if (app && tid < 64) {
      bool bit = false;
      if (tid < nw) {
        float x = 0.f;
#pragma unroll 16
        for (int t = 0; t < kD; ++t) x = fmaf(ws[t * kFWs + tid], s_ks[t], x);
        bit = x >= 0.f;                                                  // sign(0) = +1 (R-3)
      }
      s_bits[tid] = bit ? 1u : 0u;
    }
    __syncthreads();
    // half tables (fp64 products, rounded once): one (h, table, half) per thread
    if (tid < NH * 16 * 2) {
      const int hi = tid & 1, tl = (tid >> 1) & 15, h = tid >> 5;
      if (tl < ntab) {
        double f[4][2];
#pragma unroll
        for (int bit = 0; bit < 4; ++bit) {
          const int ib = hi * 4 + bit;
          const bool ok = ib < P && (l0 + tl) < L;
          f[bit][0] = ok ? (double)s_fx[((h * 8 + ib) * 2 + 0) * 16 + tl] : 1.0;
          f[bit][1] = ok ? (double)s_fx[((h * 8 + ib) * 2 + 1) * 16 + tl] : 1.0;
        }
        double p01[4], p012[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) p01[e] = f[0][e & 1] * f[1][e >> 1];
#pragma unroll
        for (int e = 0; e < 8; ++e) p012[e] = p01[e & 3] * f[2][e >> 2];
#pragma unroll
        for (int e = 0; e < 16; ++e) s_half[((h * 2 + hi) * 16 + e) * 16 + tl] = (float)(p012[e & 7] * f[3][e >> 3]);
      }
    }
    if (app && tid < ntab) {   // code byte of my table tid (padding tables write 0)
      const int l = l0 + tid;
      uint32_t code = 0;
      if (l < L)
        for (int i = 0; i < P; ++i) code |= s_bits[tid * P + i] << i;   // row i -> bit i (R-4)
      const int j = n - 1;
      const int M = (LP < 32 ? LP : 32) - 1;
      const int s = (l & ~M) | ((l - j) & M);
      a.codes[((size_t)b * a.H_kv + g) * a.N_max * LP + code_off(j, s, LP)] = (uint8_t)code;
    }
    if (app && c == 0 && warp == 0) {   // ||v_j|| of the newest key (vnorm_kernel's order)
      const uint2 u = a.v_new ? *reinterpret_cast<const uint2*>(a.v_new + ((size_t)b * a.H_kv + g) * kD + lane * 4)
                              : *reinterpret_cast<const uint2*>(a.V + (((size_t)b * a.H_kv + g) * a.N_max + n - 1) * kD + lane * 4);
      float va = bf16lo(u.x), vb = bf16hi(u.x), vc = bf16lo(u.y), vd = bf16hi(u.y);
      float sq = fmaf(va, va, fmaf(vb, vb, fmaf(vc, vc, vd * vd)));
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
      if (lane == 0) a.vnorm[((size_t)b * a.H_kv + g) * a.N_max + n - 1] = sqrtf(sq);
    }
    __syncthreads();
    FU_STAMP(2);
    // LUT columns of my tables -> every CTA of the cluster.  Column of table l:
    // l (LP >= 32), or l, l + LP, ... < 32 (LP < 32, replicated)
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");   // every CTA is running
    const int R = 1 << P;
    if (LP >= 32 && (a.tpc & 3) == 0) {
      // task = (LUT row rr, 4-table group): one float4 per destination CTA
      const int ng = a.tpc >> 2;
      for (int e = tid; e < 256 * ng; e += kFThreads) {
        const int gq = e % ng, rr = e / ng;
        const int tl = gq * 4, l = l0 + tl;
        if (l >= LP) continue;
        float4 T = make_float4(0.f, 0.f, 0.f, 0.f);
        if (rr < R) {
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const float4 lo = *reinterpret_cast<const float4*>(s_half + ((h * 2 + 0) * 16 + (rr & 15)) * 16 + tl);
            const float4 hv = *reinterpret_cast<const float4*>(s_half + ((h * 2 + 1) * 16 + (rr >> 4)) * 16 + tl);
            T.x = fmaf(lo.x, hv.x, T.x);
            T.y = fmaf(lo.y, hv.y, T.y);
            T.z = fmaf(lo.z, hv.z, T.z);
            T.w = fmaf(lo.w, hv.w, T.w);
          }
          if (l + 0 >= L) T.x = 0.f;
          if (l + 1 >= L) T.y = 0.f;
          if (l + 2 >= L) T.z = 0.f;
          if (l + 3 >= L) T.w = 0.f;
        }
        for (int r = 0; r < CS; ++r)
          *reinterpret_cast<float4*>(cluster.map_shared_rank(lut, r) + rr * 64 + l) = T;
      }
    } else {
      for (int e = tid; e < 256 * 16; e += kFThreads) {
        const int tl = e & 15, rr = e >> 4;
        if (tl >= ntab) continue;
        const int l = l0 + tl;
        float T = 0.f;
        if (l < L && rr < R) {
#pragma unroll
          for (int h = 0; h < NH; ++h) T = fmaf(s_half[((h * 2 + 0) * 16 + (rr & 15)) * 16 + tl], s_half[((h * 2 + 1) * 16 + (rr >> 4)) * 16 + tl], T);
        }
        for (int r = 0; r < CS; ++r) {
          float* rl = cluster.map_shared_rank(lut, r);
          if (LP >= 32) rl[rr * 64 + l] = T;
          else for (int cc = l; cc < 32; cc += LP) rl[rr * 64 + cc] = T;
        }
      }
    }
    __threadfence();   // the appended code / norm before the cluster barrier (release)
  }
  FU_STAMP(3);
  cluster.sync();
  FU_STAMP(4);

  // ===== B. scores of my slice ======================================================
  const int base = c * a.S;
  int len = n - base;
  len = len < 0 ? 0 : (len > a.S ? a.S : len);
  uint32_t nvalid = 0, nforced = 0, kmin = 0xFFFFFFFFu, kmax = 0u;
  {
    using TSt = TileStage<LP>;
    const uint32_t ring = smem_u32(fsm + kFLutBytes) + (uint32_t)warp * (kFScoreStages * TSt::BYTES);
    const char* ringp = fsm + kFLutBytes + warp * (kFScoreStages * TSt::BYTES);
    uint32_t pk[16];
#pragma unroll
    for (int m = 0; m < 16; ++m)
      pk[m] = (uint32_t)(((2 * m + lane) & 31) << 2) | ((uint32_t)(((2 * m + 1 + lane) & 31) << 2) << 8);
    const uint8_t* crow = a.codes + ((size_t)b * a.H_kv + g) * a.N_max * LP;
    const float* vrow = a.vnorm + ((size_t)b * a.H_kv + g) * a.N_max;
    const uint8_t* mrow = a.mask ? a.mask + (size_t)b * a.N_max : nullptr;
    float* srow = a.scores + (size_t)row * a.N_max;
    const int tiles = a.S >> 5;
    const int vt = (len + 31) >> 5;                    // tiles holding valid keys
    const int my = warp < vt ? (vt - warp + kFWarps - 1) / kFWarps : 0;
    const int t0 = base >> 5;
    if (my > 0) issue_tile<LP>(ring, crow + (size_t)(t0 + warp) * 32 * LP, vrow + (t0 + warp) * 32, lane);
    cpa_commit();
    for (int i = 0; i < my; ++i) {
      if (i + 1 < my) {
        const int ti = t0 + warp + (i + 1) * kFWarps;
        issue_tile<LP>(ring + ((i + 1) & 1) * TSt::BYTES, crow + (size_t)ti * 32 * LP, vrow + ti * 32, lane);
      }
      cpa_commit();
      cpa_wait<1>();
      const char* st = ringp + (i & 1) * TSt::BYTES;
      uint32_t w[LP / 4];
#pragma unroll
      for (int ch = 0; ch < TSt::NCH; ++ch) {
        if constexpr (TSt::CB == 16) {
          const uint4 v = *reinterpret_cast<const uint4*>(st + ch * 512 + lane * 16);
          w[ch * 4 + 0] = v.x; w[ch * 4 + 1] = v.y; w[ch * 4 + 2] = v.z; w[ch * 4 + 3] = v.w;
        } else {
          const uint2 v = *reinterpret_cast<const uint2*>(st + ch * 256 + lane * 8);
          w[ch * 2 + 0] = v.x; w[ch * 2 + 1] = v.y;
        }
      }
      const float vn = *reinterpret_cast<const float*>(st + TSt::CODE_BYTES + lane * 4);
      uint64_t acc = 0ull;
#pragma unroll
      for (int s2 = 0; s2 < LP; s2 += 2) {
        float v[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int ss = s2 + u, sl = ss & 31;
          const uint32_t sel = (uint32_t)(4 + (sl & 1)) | ((uint32_t)(ss & 3) << 4) | 0x7600u;
          const uint32_t addr = __byte_perm(w[ss >> 2], pk[sl >> 1], sel);
          v[u] = *reinterpret_cast<const float*>(fsm + ((ss & 32) ? 128 : 0) + addr);
        }
        const uint64_t pv = (uint64_t)__float_as_uint(v[0]) | ((uint64_t)__float_as_uint(v[1]) << 32);
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(pv));
      }
      const float score = vn * (__uint_as_float((uint32_t)acc) + __uint_as_float((uint32_t)(acc >> 32)));
      const int li = (warp + i * kFWarps) * 32 + lane;   // slice-local index
      const int j = base + li;
      const bool ok = li < len && (!mrow || mrow[j]);
      srow[j] = ok ? score : -INFINITY;
      uint32_t key = 0u;
      if (ok) key = (j < a.sink || j >= n - a.window) ? 0xFFFFFFFFu : f2key(score);
      keys[li] = key;
      nvalid += key != 0u;
      nforced += key == 0xFFFFFFFFu;
      if (key != 0u && key != 0xFFFFFFFFu) { kmin = min(kmin, key); kmax = max(kmax, key); }
    }
    cpa_wait<0>();
    // tiles past seq_len: -inf scores, invalid keys
    for (int ti = vt + warp; ti < tiles; ti += kFWarps) {
      const int li = ti * 32 + lane;
      srow[base + li] = -INFINITY;
      keys[li] = 0u;
    }
  }
  __syncthreads();

  FU_STAMP(5);
  // ===== C. exact top-k over the cluster =============================================
  TopkArgs ta = {};
  ta.op = 0;
  ta.index_base = 0;
  ta.scores = a.scores;
  ta.seq_lens = a.seq_lens;
  ta.rows = (int)gridDim.y;
  ta.H_sel = a.H_kv;
  ta.N_max = a.N_max;
  ta.k = a.k;
  ta.sink = a.sink;
  ta.window = a.window;
  ta.per = a.S;
  ta.idx = a.idx;
  ta.cnt = a.cnt;
  ta.sel_scores = nullptr;
  int32_t* sel = reinterpret_cast<int32_t*>(fsm);   // LUT region (dead)
  int sel_lo = 0, sel_cnt = 0;
  topk_core(ta, keys, TS, row, n, base, len, nvalid, nforced, kmin, kmax, sel, &sel_lo, &sel_cnt);
  __syncthreads();
  int32_t* list = reinterpret_cast<int32_t*>(keys);  // keys are dead: move the list out of the ring zone
  for (int i = tid; i < sel_cnt; i += kFThreads) list[i] = sel[i];
  __syncthreads();

  FU_STAMP(6);
  // ===== D. attention over my selected rows + cluster LSE merge =====================
  {
    const int gid = lane >> 2, tig = lane & 3;
    const int h0 = g * NH;
    uint32_t qb[8][2];
    {
      const bool hv = gid < NH;
      const uint32_t* qrow = reinterpret_cast<const uint32_t*>(a.q + ((size_t)b * a.H_q + h0 + (hv ? gid : 0)) * kD);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        qb[ks][0] = hv ? qrow[ks * 8 + tig] : 0u;
        qb[ks][1] = hv ? qrow[ks * 8 + 4 + tig] : 0u;
      }
    }
    float o[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) { o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f; }
    float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;
    const uint16_t* Kb = a.K + ((size_t)b * a.H_kv + g) * a.N_max * kD;
    const uint16_t* Vb = a.V + ((size_t)b * a.H_kv + g) * a.N_max * kD;
    const int ntiles = (sel_cnt + kTileRows - 1) / kTileRows;
    if (warp < kFAttWarps) {
      const uint32_t ring0 = smem_u32(fsm) + (uint32_t)warp * (kFAttStages * kTileBytes);
      auto issue = [&](int t, int stage) {
        const int row0 = t * kTileRows;
        const uint32_t kbuf = ring0 + stage * kTileBytes, vbuf = kbuf + kTileRows * 256;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int cc = (it * 32 + lane) & 15, rr = (it * 32 + lane) >> 4;
          const int i = row0 + rr;
          const bool v = i < sel_cnt;
          const int tok = v ? list[i] : 0;
          cp16(kbuf + swz(rr, cc), Kb + (size_t)tok * kD + cc * 8, v);
          cp16(vbuf + swz(rr, cc), Vb + (size_t)tok * kD + cc * 8, v);
        }
      };
      int my = 0;
      for (int t = warp; t < ntiles; t += kFAttWarps) ++my;
      if (my > 0) issue(warp, 0);
      cp_commit();
      for (int jt = 0; jt < my; ++jt) {
        const int t = warp + jt * kFAttWarps;
        if (jt + 1 < my) issue(warp + (jt + 1) * kFAttWarps, (jt + 1) & 1);
        cp_commit();
        cp_wait<1>();
        __syncwarp();
        const uint32_t kbuf = ring0 + (jt & 1) * kTileBytes, vbuf = kbuf + kTileRows * 256;
        float s[4] = {0.f, 0.f, 0.f, 0.f};
        {
          const int rr = (lane & 7) + ((lane >> 3) & 1) * 8;
          const int cc = lane >> 4;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4(kbuf + swz(rr, ks * 2 + cc), a0, a1, a2, a3);
            mma_bf16(s, a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
          }
        }
        const int row0 = t * kTileRows;
        const bool v0 = row0 + gid < sel_cnt, v1 = row0 + gid + 8 < sel_cnt;
        const float z0 = v0 ? s[0] * a.scale_log2 : -INFINITY;
        const float z1 = v0 ? s[1] * a.scale_log2 : -INFINITY;
        const float z2 = v1 ? s[2] * a.scale_log2 : -INFINITY;
        const float z3 = v1 ? s[3] * a.scale_log2 : -INFINITY;
        float tA = fmaxf(z0, z2), tB = fmaxf(z1, z3);
#pragma unroll
        for (int off = 4; off <= 16; off <<= 1) {
          tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, off));
          tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, off));
        }
        const float nA = fmaxf(mA, tA), nB = fmaxf(mB, tB);
        const float alA = (nA == -INFINITY) ? 1.f : exp2f(mA - nA);
        const float alB = (nB == -INFINITY) ? 1.f : exp2f(mB - nB);
        const float p0 = (nA == -INFINITY) ? 0.f : exp2f(z0 - nA);
        const float p1 = (nB == -INFINITY) ? 0.f : exp2f(z1 - nB);
        const float p2 = (nA == -INFINITY) ? 0.f : exp2f(z2 - nA);
        const float p3 = (nB == -INFINITY) ? 0.f : exp2f(z3 - nB);
        const uint32_t P01 = pack_bf16(p0, p1), P23 = pack_bf16(p2, p3);
        float sA = bf16lo(P01) + bf16lo(P23), sB = bf16hi(P01) + bf16hi(P23);
#pragma unroll
        for (int off = 4; off <= 16; off <<= 1) {
          sA += __shfl_xor_sync(0xffffffffu, sA, off);
          sB += __shfl_xor_sync(0xffffffffu, sB, off);
        }
        lA = lA * alA + sA;
        lB = lB * alB + sB;
        mA = nA;
        mB = nB;
        const uint32_t pb0 = movm_t(P01), pb1 = movm_t(P23);
        {
          const int mi = lane >> 3;
          const int rr = (lane & 7) + (mi >> 1) * 8;
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4_t(vbuf + swz(rr, mt * 2 + (mi & 1)), a0, a1, a2, a3);
            o[mt][0] *= alA; o[mt][1] *= alB; o[mt][2] *= alA; o[mt][3] *= alB;
            mma_bf16(o[mt], a0, a1, a2, a3, pb0, pb1);
          }
        }
        __syncwarp();
      }
      cp_wait<0>();
    }
    __syncthreads();
    // merge the attention warps' states (ring region reused)
    float* sm_o = reinterpret_cast<float*>(fsm);                    // [warps][8][128]
    float* sm_m = sm_o + kFAttWarps * 8 * kD;
    float* sm_l = sm_m + kFAttWarps * 8;
    if (warp < kFAttWarps) {
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        const int d0 = mt * 16 + gid;
        sm_o[(warp * 8 + 2 * tig) * kD + d0] = o[mt][0];
        sm_o[(warp * 8 + 2 * tig + 1) * kD + d0] = o[mt][1];
        sm_o[(warp * 8 + 2 * tig) * kD + d0 + 8] = o[mt][2];
        sm_o[(warp * 8 + 2 * tig + 1) * kD + d0 + 8] = o[mt][3];
      }
      if (gid == 0) {
        sm_m[warp * 8 + 2 * tig] = mA; sm_m[warp * 8 + 2 * tig + 1] = mB;
        sm_l[warp * 8 + 2 * tig] = lA; sm_l[warp * 8 + 2 * tig + 1] = lB;
      }
    }
    __syncthreads();
    for (int x = tid; x < NH * kD; x += kFThreads) {
      const int h = x / kD, e = x % kD;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kFAttWarps; ++w) M = fmaxf(M, sm_m[w * 8 + h]);
      float Ls = 0.f, O = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int w = 0; w < kFAttWarps; ++w) {
          const float wt = exp2f(sm_m[w * 8 + h] - M);
          Ls = fmaf(wt, sm_l[w * 8 + h], Ls);
          O = fmaf(wt, sm_o[(w * 8 + h) * kD + e], O);
        }
      }
      s_part[h][2 + e] = O;
      if (e == 0) { s_part[h][0] = M; s_part[h][1] = Ls; }
    }
    cluster.sync();
    // cluster LSE merge: CTA c merges heads h = c, c + CS, ... over the CS partials
    constexpr float kLn2 = 0.6931471805599453f;
    for (int h = c; h < NH; h += CS) {
      for (int e = tid; e < kD + 1; e += kFThreads) {
        float M = -INFINITY;
        for (int r = 0; r < CS; ++r) M = fmaxf(M, cluster.map_shared_rank(&s_part[0][0], r)[h * (kD + 2)]);
        float Ls = 0.f, O = 0.f;
        if (M != -INFINITY) {
          for (int r = 0; r < CS; ++r) {
            const float* pr = cluster.map_shared_rank(&s_part[0][0], r) + h * (kD + 2);
            const float wt = exp2f(pr[0] - M);
            Ls = fmaf(wt, pr[1], Ls);
            if (e < kD) O = fmaf(wt, pr[2 + e], O);
          }
        }
        const size_t oh = (size_t)b * a.H_q + h0 + h;
        if (e < kD) a.out[oh * kD + e] = (uint16_t)f2bf_bits(Ls > 0.f ? O / Ls : 0.f);
        else if (a.lse) a.lse[oh] = Ls > 0.f ? (M + log2f(Ls)) * kLn2 : -INFINITY;
      }
    }
    cluster.sync();   // keep s_part alive until every CTA has read it
  }
  FU_STAMP(7);
}

// Host: pick the cluster size and check that the whole grid is co-resident
// (one wave); returns false when the fused path does not apply.
static bool fused_geometry(const socket_cfg& c, int& CS, int& S) {
  if (c.group_mode != SOCKET_GROUP_KV_SHARED || c.P > 8) return false;
  const int Lp = code_slots(c.L);
  if (Lp > 64) return false;
  const int NH = c.H_q / c.H_kv;
  if (NH != 1 && NH != 2 && NH != 4 && NH != 8) return false;
  const int rows = c.B * c.H_kv;
  // measured (tools/fused_check.py): one launch wins while the grid is at most
  // 8 clusters of 8 (B = 1 at 8 KV heads: 39 vs 48 us at 32K); beyond that the
  // multi-kernel path spreads each stage over all 148 SMs and is faster
  if (rows > 8) return false;
  for (int cs : {8, 4}) {   // clusters of 16 do not all fit one wave
    if (c.N_max % (cs * 128) != 0) continue;
    const int s = c.N_max / cs;
    // keys of a slice <= 32 KB: with the LUT + score ring (132 KB) and the static
    // top-k state (34 KB) the CTA uses ~200 KB of shared memory
    if (s > 8192 || rows * cs > num_sms()) continue;
    if ((Lp + cs - 1) / cs * c.P > 64) continue;   // <= 64 W rows per CTA (staging, 8 DMMA warps)
    CS = cs;
    S = s;
    return true;
  }
  return false;
}

bool fused_step_applies(const socket_cfg& c) {
  int CS, S;
  if (c.flags & SOCKET_FLAG_CHAINED_STEP) return false;
  return fused_geometry(c, CS, S);
}

socket_status launch_fused_step(const socket_cfg& c, const void* q, void* K, void* V,
                                const void* W, uint8_t* codes, float* vnorm, const int32_t* seq_lens,
                                const uint8_t* mask, int do_append, const void* k_new,
                                const void* v_new, int k, int sink, int window,
                                float* scores, int32_t* idx, int32_t* cnt, void* out, float* lse,
                                cudaStream_t st) {
  int CS, S;
  if (!fused_geometry(c, CS, S)) return fail(SOCKET_EUNSUPPORTED, "fused step: shape not supported");
  const int Lp = code_slots(c.L);
  FusedArgs a;
  a.q = (const uint16_t*)q;
  a.K = (uint16_t*)K;
  a.V = (uint16_t*)V;
  a.k_new = (const uint16_t*)k_new;
  a.v_new = (const uint16_t*)v_new;
  a.W = (const uint16_t*)W;
  a.codes = codes;
  a.vnorm = vnorm;
  a.seq_lens = seq_lens;
  a.mask = mask;
  a.scores = scores;
  a.idx = idx;
  a.cnt = cnt;
  a.out = (uint16_t*)out;
  a.lse = lse;
  a.H_q = c.H_q;
  a.H_kv = c.H_kv;
  a.N_max = c.N_max;
  a.L = c.L;
  a.P = c.P;
  a.Lp = Lp;
  a.k = k;
  a.sink = sink;
  a.window = window;
  a.do_append = do_append;
  a.hard = c.scoring == SOCKET_SCORING_HARD;
  a.tau = c.tau;
  a.scale_log2 = c.sm_scale * kLog2eM;
  a.S = S;
  a.tpc = (Lp + CS - 1) / CS;
  const size_t sm = fused_smem_bytes(S);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, c.B * c.H_kv, 1);
  cfg.blockDim = dim3(kFThreads, 1, 1);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int NH = c.H_q / c.H_kv;
  cudaError_t e = cudaSuccess;
#define SK_FUSED(N, LPV)                                                                          \
  if (NH == N && Lp == LPV) {                                                                     \
    auto kfn = fused_step_kernel<N, LPV>;                                                         \
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) \
      return fail(SOCKET_ECUDA, "fused step: shared memory request rejected");                   \
    if (CS > 8) cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);    \
    e = cudaLaunchKernelEx(&cfg, kfn, a);                                                         \
  } else
  SK_FUSED(1, 8) SK_FUSED(1, 16) SK_FUSED(1, 32) SK_FUSED(1, 64)
  SK_FUSED(2, 8) SK_FUSED(2, 16) SK_FUSED(2, 32) SK_FUSED(2, 64)
  SK_FUSED(4, 8) SK_FUSED(4, 16) SK_FUSED(4, 32) SK_FUSED(4, 64)
  SK_FUSED(8, 8) SK_FUSED(8, 16) SK_FUSED(8, 32) SK_FUSED(8, 64)
  { return fail(SOCKET_EUNSUPPORTED, "fused step: heads / tables not instantiated"); }
#undef SK_FUSED
  if (e != cudaSuccess) return fail(SOCKET_ECUDA, std::string("fused step launch: ") + cudaGetErrorString(e));
  return check_launch("fused_step_kernel");
}

}  // namespace sk
