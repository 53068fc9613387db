// Row-spread one-launch decode step (small batch): one
// cooperative launch of at most one CTA per SM; selection row (b, kv head) r
// (KV_SHARED) is spread over C CTAs, CTA c owning the key slice [c S, (c+1) S).
// The CTAs of a row meet at a few row barriers in global memory (L2):
//
//   0. every warp starts streaming its slice's code tiles into its cp.async
//      ring, and every CTA reads its slice's value norms (bounds below);
//   A. tables (Alg. 2): CTA c projects q on the W rows of tables
//      [c tpc, (c+1) tpc) (fp64 tensor-core DMMA), builds their sigma factors,
//      half tables and LUT columns and writes the columns into the row's LUT
//      image in global memory; with append it also hashes the newest key on
//      those tables (Alg. 1), and the CTA owning the newest key stores
//      its K/V rows and its value norm;
//      -- row barrier 1 --
//   B. every CTA loads the whole LUT image; the score range of the row is
//      bounded from the LUT (sum over tables of the min / max entry) and the
//      row's norm range, and scores (Eq. 4 / Alg. 4) of the slice are binned on
//      that range (2048 bins, monotone in the score) as they are computed;
//      bins are added into the row histogram (red.global.add);
//      -- row barrier 2 --
//   C. top-k (Alg. 3 l.244): the row histogram locates the bin of rank k; its
//      keys (typically tens per row) are published per CTA; refinement levels
//      (more barriers) only when that bin holds more than 2048 keys;
//      -- row barrier 3 --
//      every CTA resolves the exact threshold T and tie quota from the
//      published candidates, and knows the output position of its own keys;
//   D. sparse attention (Eq. 2, exact logits P:271) over the CTA's selected
//      rows (tensor-core MMA tiles, online softmax); partial states go to
//      global memory and the last CTA of the row (ticket) merges them by LSE.
//
// Selection, scores and codes are the same as the multi-kernel path's (same
// arithmetic, exact top-k); outputs agree to fp32 rounding (the attention is
// split per CTA slice).  The workspace's row control words must be zero before
// the first launch; every launch leaves them zero.  The final LSE merge is
// spread over the row's CTAs after a 4th row barrier (CTA order, deterministic).
#include <algorithm>

#include "mma_dev.cuh"
#include "score_dev.cuh"

namespace sk {

#ifdef SK_TRACE
static __device__ unsigned long long g_spread_trace[4096 * 32];
#define SP_STAMP(i)                                                                       \
  do {                                                                                    \
    if (threadIdx.x == 0) {                                                               \
      const int cta = blockIdx.y * gridDim.x + blockIdx.x;                                \
      if (cta < 4096) g_spread_trace[cta * 32 + (i)] = clock64();                         \
      if (((i) == 0 || (i) == 10) && cta < 4096) {                                        \
        unsigned long long gt;                                                            \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));                            \
        g_spread_trace[cta * 32 + ((i) == 0 ? 23 : 24)] = gt;                             \
      }                                                                                   \
    }                                                                                     \
  } while (0)
extern "C" int socket_debug_spread_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_spread_trace, (size_t)n * sizeof(unsigned long long));
}
#else
#define SP_STAMP(i) \
  do {              \
  } while (0)
#endif

constexpr int kSpThreads = 512;
constexpr int kSpWarps = kSpThreads / 32;
constexpr int kSpBins = 2048;
constexpr int kSpHistWords = kSpBins + 64;    // + [2048] #valid, [2049] #forced (level 0)
constexpr int kSpLevels = 4;                  // histogram levels: the last one is always one key wide
constexpr int kSpCandCap = 2048;              // row-wide candidates resolved in shared memory
constexpr int kSpAttWarps = 8;                // attention warps (two 16-row stages each)
constexpr int kSpLutBytes = 256 * 64 * 4;     // 64 KB LUT image
constexpr int kSpFWs = 72;                    // staged W row stride (floats)
constexpr int kSpFQs = 8;                     // staged q row stride (doubles)
constexpr int kSpTpp = 8;                     // tables per projection pass (<= 64 W rows)

__host__ __device__ constexpr int sp_ring_bytes(int LP, int nst) {
  return kSpWarps * nst * (LP * 32 + 128);
}
constexpr int kSpAttRing = kSpAttWarps * 2 * kTileBytes;   // 128 KB
// dynamic shared memory: a zone holding [LUT 64 KB | code rings] during A-B and
// [attention list | resolve scratch 16 KB | attention ring] during C-D, then the
// slice's keys
__host__ __device__ inline int sp_scr_off(int S) { return (S * 4 + 1023) & ~1023; }
__host__ __device__ inline int sp_att_off(int S) { return sp_scr_off(S) + 16384; }
__host__ __device__ inline int sp_zone(int LP, int S, int nst) {
  const int z0 = kSpLutBytes + sp_ring_bytes(LP, nst), z1 = sp_att_off(S) + kSpAttRing;
  return z0 > z1 ? z0 : z1;
}

// global-memory workspace of one selection row (u32 words)
struct SpLayout {
  int C, NH;
  __host__ __device__ size_t ctrl() const { return 0; }                                   // bar, ticket
  __host__ __device__ size_t hist() const { return 16; }                                  // [levels][kSpHistWords]
  __host__ __device__ size_t stat() const { return hist() + (size_t)kSpLevels * kSpHistWords; }  // [C][4] f32
  __host__ __device__ size_t info() const { return stat() + (size_t)C * 4; }             // [C][4] u32
  __host__ __device__ size_t lut() const { return (info() + (size_t)C * 4 + 63) & ~(size_t)63; }  // [256][64] f32
  __host__ __device__ size_t tmm() const { return lut() + 256 * 64; }                    // [64][2] f32 table min / max
  __host__ __device__ size_t cand() const { return tmm() + 128; }                         // [C][kSpCandCap] uint2
  __host__ __device__ size_t part() const { return cand() + (size_t)C * kSpCandCap * 2; } // [C][NH][kD+2] f32
  __host__ __device__ size_t words() const { return (part() + (size_t)C * NH * (kD + 2) + 63) & ~(size_t)63; }
};

struct SpreadArgs {
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
  uint32_t* ws;           // rows x row_words
  size_t row_words;
  int H_q, H_kv, N_max, L, P, k, sink, window, do_append, hard;
  float tau, scale_log2;
  int S;     // keys per CTA slice (multiple of 32)
  int tpc;   // tables per CTA
  int zone;  // sp_zone(LP, S, nst)
  int nst;   // code ring stages per warp (3 or 4)
};

// ---- row barrier in global memory ------------------------------------------------
__device__ __forceinline__ void sp_arrive(uint32_t* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
  }
}
__device__ __forceinline__ uint64_t sp_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// spin until the row's counter reaches target; a counter that never gets there
// (a workspace whose control words were not zeroed) traps after 2 s instead of
// hanging the device
__device__ __forceinline__ void sp_wait(uint32_t* bar, uint32_t target) {
  if (threadIdx.x == 0) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    if (v < target) {
      const uint64_t t0 = sp_now();
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        if (v < target && sp_now() - t0 > 2000000000ull) __trap();
      } while (v < target);
    }
  }
  __syncthreads();
}
__device__ __forceinline__ void sp_red_add(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// block-wide: bin of rank `need` (1-based, counted from the top) of a
// kSpBins-bin histogram in shared memory; returns (bin, rank inside the bin,
// keys in the bin) through s_dec.  Thread t owns bins 2047 - 4t .. 2044 - 4t.
__device__ __forceinline__ void sp_locate(const uint32_t* h, uint32_t need, uint32_t* s_w, uint32_t* s_dec) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t c4[4], tot = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) { c4[e] = h[kSpBins - 1 - (4 * tid + e)]; tot += c4[e]; }
  uint32_t inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  uint32_t wpre = 0;
#pragma unroll
  for (int w = 0; w < kSpWarps; ++w) wpre += (w < warp) ? s_w[w] : 0u;
  const uint32_t excl = wpre + inc - tot;
  if (excl < need && excl + tot >= need) {
    uint32_t run = excl;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (run < need && run + c4[e] >= need) {
        s_dec[0] = (uint32_t)(kSpBins - 1 - (4 * tid + e));
        s_dec[1] = need - run;
        s_dec[2] = c4[e];
      }
      run += c4[e];
    }
  }
  __syncthreads();
}

// Block-wide ascending selection over a slice's keys: key in [lo, hi] and
// (key > T, or key == T among the first eqq keys == T of the slice, eqq > 0 only
// when T is in [lo, hi]).  Writes slice-local indices to list[list0 + rank]
// (list != null) and base + index to orow[pos0 + rank] (orow != null); returns
// the count (every thread).
__device__ __forceinline__ int sp_select(const uint32_t* keys, int slen, uint32_t lo, uint32_t hi, uint32_t T,
                                         uint32_t eqq, int32_t* list, int list0, int32_t* orow, uint32_t pos0,
                                         int base, uint32_t* s_w, uint32_t* s_w2) {
  constexpr unsigned kFull = 0xffffffffu;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // warp w owns a contiguous chunk of whole 128-key rows; lane l holds keys
  // 4 l .. 4 l + 3 of a row (one 16-B load).  Counts are packed (gt | eq << 16;
  // a chunk holds far fewer than 65536 keys).
  const int per = ((slen + kSpWarps - 1) / kSpWarps + 127) & ~127;
  const int c0 = warp * per, c1 = min(slen, c0 + per);
  auto load4 = [&](int li, uint32_t (&k)[4]) {
    if (li + 3 < c1) {
      const uint4 v = *reinterpret_cast<const uint4*>(keys + li);
      k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) k[e] = li + e < c1 ? keys[li + e] : 0u;
    }
  };
  auto flags = [&](uint32_t key) -> uint32_t {   // 1: > T inside [lo, hi]; 0x10000: == T
    return (key > T && key >= lo && key <= hi) ? 1u : ((key != 0u && key == T) ? 0x10000u : 0u);
  };
  uint32_t cnt = 0;
  for (int i0 = c0; i0 < c1; i0 += 128) {
    uint32_t k[4];
    load4(i0 + 4 * lane, k);
#pragma unroll
    for (int e = 0; e < 4; ++e) cnt += flags(k[e]);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
  __syncthreads();   // previous readers of s_w / s_w2
  if (lane == 0) { s_w[warp] = cnt & 0xFFFFu; s_w2[warp] = cnt >> 16; }
  __syncthreads();
  uint32_t gb = 0, eb = 0, gt = 0, et = 0;
#pragma unroll
  for (int w = 0; w < kSpWarps; ++w) {
    const uint32_t xg = s_w[w], xe = s_w2[w];
    gb += (w < warp) ? xg : 0u;
    eb += (w < warp) ? xe : 0u;
    gt += xg;
    et += xe;
  }
  for (int i0 = c0; i0 < c1; i0 += 128) {
    const int li = i0 + 4 * lane;
    uint32_t k[4], f[4], mine = 0;
    load4(li, k);
#pragma unroll
    for (int e = 0; e < 4; ++e) { f[e] = flags(k[e]); mine += f[e]; }
    uint32_t inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    const uint32_t ex = inc - mine;
    uint32_t g = gb + (ex & 0xFFFFu), ev = eb + (ex >> 16);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool isgt = f[e] == 1u, iseq = f[e] == 0x10000u;
      if (isgt || (iseq && ev < eqq)) {
        const uint32_t p = g + min(ev, eqq);
        if (list) list[list0 + p] = li + e;
        if (orow) orow[pos0 + p] = base + li + e;
      }
      g += isgt ? 1u : 0u;
      ev += iseq ? 1u : 0u;
    }
    const uint32_t tot = __shfl_sync(kFull, inc, 31);
    gb += tot & 0xFFFFu;
    eb += tot >> 16;
  }
  __syncthreads();   // the list is read by other warps next
  return (int)(gt + min(et, eqq));
}

template <int NH, int LP>
__global__ void __launch_bounds__(kSpThreads, 1) spread_step_kernel(SpreadArgs a) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(16) uint32_t s_hist[kSpBins];
  __shared__ uint32_t s_w[kSpWarps], s_w2[kSpWarps];
  __shared__ uint32_t s_dec[8];
  __shared__ float s_red[2 * kSpWarps];
  __shared__ float s_ks[kD];
  __shared__ uint32_t s_bits[64];
  __shared__ uint32_t s_cgt[160], s_ceq[160];   // per row CTA: candidates > T / == T (C <= 148)
  __shared__ float s_bound[4];
  __shared__ uint32_t s_tmm[2 * kSpTpp];
  __shared__ uint4 s_q[NH * 16];                // q of the row's heads (bf16)        // this pass's tables: min / max entry (float bits, >= 0)
  constexpr uint32_t kFull = 0xffffffffu;
  using TSt = TileStage<LP>;
  const int c = blockIdx.x, C = gridDim.x, row = blockIdx.y;
  const int b = row / a.H_kv, g = row % a.H_kv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P = a.P, L = a.L;
  const int n_raw = a.seq_lens[b];
  const int n = n_raw < 0 ? 0 : (n_raw > a.N_max ? a.N_max : n_raw);
  const bool app = a.do_append && n_raw > 0 && n_raw <= a.N_max;   // outgrown cache: no write (R-27)
  const int jn = n - 1;                                            // the newest key (if app)
  const SpLayout lay{C, NH};
  uint32_t* rw = a.ws + (size_t)row * a.row_words;
  uint32_t* bar = rw + lay.ctrl();
  uint32_t* gh = rw + lay.hist();
  float* glut = reinterpret_cast<float*>(rw + lay.lut());
  float* lut = reinterpret_cast<float*>(smem);
  char* ringz = smem + kSpLutBytes;
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem + a.zone);
  const int base = c * a.S;
  const int slen = max(0, min(a.S, a.N_max - base));               // keys of my slice
  const int len = max(0, min(slen, n - base));                     // valid prefix (mask aside)
  const bool own_new = app && jn >= base && jn < base + slen;
  const size_t kvrow = (size_t)b * a.H_kv + g;
  const uint8_t* crow = a.codes + kvrow * a.N_max * LP;
  const float* vrow = a.vnorm + kvrow * a.N_max;
  uint32_t nb = 0;   // row barriers passed
  SP_STAMP(0);

  // ===== 0. loads the table phase needs first (ahead of the code stream in the
  //          memory queues), then the code prefetch ===============================
  const int h0 = g * NH;
  const int ltab0 = c * a.tpc;
  const int ltab1 = min(LP, ltab0 + a.tpc);
  uint4 pre_w[2], pre_q = make_uint4(0, 0, 0, 0);
  {
    const int m = tid & 7, cq = (tid >> 3) & 15;
    const int nw0 = ltab0 < ltab1 ? max(0, min(min(kSpTpp, ltab1 - ltab0), L - ltab0)) * P : 0;
    if (tid < 128 && m < NH && nw0 > 0) pre_q = *(reinterpret_cast<const uint4*>(a.q + ((size_t)b * a.H_q + h0 + m) * kD) + cq);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = tid + u * kSpThreads, w = e & 63, cw = e >> 6;
      pre_w[u] = make_uint4(0, 0, 0, 0);
      if (w < nw0) pre_w[u] = __ldg(reinterpret_cast<const uint4*>(a.W + (size_t)(ltab0 * P + w) * kD) + cw);
    }
  }
  float4 v4[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j4 = base + 4 * (tid + u * kSpThreads);
    v4[u] = j4 < base + len ? __ldcg(reinterpret_cast<const float4*>(vrow + j4)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  uint16_t pre_k = 0;
  if (app && n > 0 && tid < kD)
    pre_k = a.k_new ? a.k_new[kvrow * kD + tid] : a.K[(kvrow * a.N_max + jn) * kD + tid];
  const int vt = (len + 31) >> 5;                                  // tiles holding valid keys
  const int my = warp < vt ? (vt - warp + kSpWarps - 1) / kSpWarps : 0;
  const int t0 = base >> 5;
  const int lt = own_new ? (jn - base) >> 5 : -1;                  // slice tile of the new key
  const int nst = a.nst;
  const int i_late = (lt >= 0 && (lt % kSpWarps) == warp && lt / kSpWarps < nst) ? lt / kSpWarps : -1;
  const uint32_t ring = smem_u32(ringz) + (uint32_t)warp * (nst * TSt::BYTES);
  const char* ringp = ringz + warp * (nst * TSt::BYTES);
  auto prefetch = [&]() {
    for (int s = 0; s < nst; ++s) {
      if (s < my && s != i_late) {
        const int ti = t0 + warp + s * kSpWarps;
        issue_tile<LP>(ring + s * TSt::BYTES, crow + (size_t)ti * 32 * LP, vrow + ti * 32, lane);
      }
      cpa_commit();
    }
  };
  // CTAs that build tables start the code stream once their table inputs have
  // arrived (the stream would otherwise queue ahead of them in the memory system)
  const bool has_tables = ltab0 < ltab1;
  if (!has_tables) prefetch();
  // q of my heads for the attention phase
  if (tid < NH * 16) s_q[tid] = *(reinterpret_cast<const uint4*>(a.q + ((size_t)b * a.H_q + h0) * kD) + tid);
  // zero my share of the row histograms (used after barrier 1)
  for (int i = c * kSpThreads + tid; i < kSpLevels * kSpHistWords; i += C * kSpThreads) gh[i] = 0u;

  // ===== A. tables of my tables (+ append bits), norm bounds of my slice ==========
  float nmin = INFINITY, nmax = 0.f;
  {   // float4 loads (the first four issued above; slices start at multiples of 32 keys)
    for (int j4 = base + 4 * (tid + 4 * kSpThreads); j4 < base + len; j4 += 4 * kSpThreads) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(vrow + j4));
      const float e4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (j4 + e < base + len && !(app && j4 + e == jn)) { nmin = fminf(nmin, e4[e]); nmax = fmaxf(nmax, e4[e]); }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j4 = base + 4 * (tid + u * kSpThreads);
      const float e4[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
      for (int e = 0; e < 4; ++e)   // (the new key's norm is computed below)
        if (j4 + e < base + len && !(app && j4 + e == jn)) { nmin = fminf(nmin, e4[e]); nmax = fmaxf(nmax, e4[e]); }
    }
  }
  if (app && n > 0) {
    if (tid < kD) {
      const size_t crowkv = (kvrow * a.N_max + jn) * kD;
      s_ks[tid] = bf16lo((uint32_t)pre_k);
      if (a.k_new && own_new) {
        a.K[crowkv + tid] = pre_k;
        a.V[crowkv + tid] = a.v_new[kvrow * kD + tid];
      }
    }
    if (own_new && warp == 0) {   // ||v_j|| of the newest key (vnorm_kernel's order)
      const uint2 u = a.v_new ? *reinterpret_cast<const uint2*>(a.v_new + kvrow * kD + lane * 4)
                              : *reinterpret_cast<const uint2*>(a.V + (kvrow * a.N_max + jn) * kD + lane * 4);
      float va = bf16lo(u.x), vb = bf16hi(u.x), vc = bf16lo(u.y), vd = bf16hi(u.y);
      float sq = fmaf(va, va, fmaf(vb, vb, fmaf(vc, vc, vd * vd)));
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) sq += __shfl_xor_sync(kFull, sq, o);
      const float nv = sqrtf(sq);
      if (lane == 0) a.vnorm[kvrow * a.N_max + jn] = nv;
      nmin = fminf(nmin, nv);
      nmax = fmaxf(nmax, nv);
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    nmin = fminf(nmin, __shfl_xor_sync(kFull, nmin, o));
    nmax = fmaxf(nmax, __shfl_xor_sync(kFull, nmax, o));
  }
  if (lane == 0) { s_red[warp] = nmin; s_red[kSpWarps + warp] = nmax; }

  const int R = 1 << P;
  for (int l0 = ltab0; l0 < ltab1; l0 += kSpTpp) {
    const int ntab = min(kSpTpp, ltab1 - l0);                  // tables of this pass (incl. padding)
    const int nw = max(0, min(ntab, L - l0)) * P;              // valid W rows of this pass
    double* qs = reinterpret_cast<double*>(smem);                                 // [t][kSpFQs]
    float* wsm = reinterpret_cast<float*>(smem + kD * kSpFQs * 8);               // [t][kSpFWs]
    float* s_fx = wsm + kD * kSpFWs;                       // sigma factors [h][bit][sign][table 8]
    float* s_half = s_fx + NH * 8 * 2 * kSpTpp;            // half tables [h][hi][entry 16][table 8]
    __syncthreads();                                       // previous pass done with the staging
    {   // q: 8 (padded) vectors x 16 uint4; W: 64 rows x 16 uint4 -- all loads first
      uint4 vw[2] = {pre_w[0], pre_w[1]}, vq = pre_q;   // first pass: loaded at kernel start
      const int m = tid & 7, cq = (tid >> 3) & 15;
      if (l0 != ltab0) {
        vq = make_uint4(0, 0, 0, 0);
        if (tid < 128 && m < NH) vq = *(reinterpret_cast<const uint4*>(a.q + ((size_t)b * a.H_q + h0 + m) * kD) + cq);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int e = tid + u * kSpThreads, w = e & 63, cw = e >> 6;
          vw[u] = make_uint4(0, 0, 0, 0);
          if (w < nw) vw[u] = __ldg(reinterpret_cast<const uint4*>(a.W + (size_t)(l0 * P + w) * kD) + cw);
        }
      }
      if (tid < 128) {
        const uint32_t w4[4] = {vq.x, vq.y, vq.z, vq.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) qs[(cq * 8 + e) * kSpFQs + m] = (double)((e & 1) ? bf16hi(w4[e >> 1]) : bf16lo(w4[e >> 1]));
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = tid + u * kSpThreads, w = e & 63, cw = e >> 6;
        const uint32_t w4[4] = {vw[u].x, vw[u].y, vw[u].z, vw[u].w};
#pragma unroll
        for (int e2 = 0; e2 < 8; ++e2) wsm[(cw * 8 + e2) * kSpFWs + w] = (e2 & 1) ? bf16hi(w4[e2 >> 1]) : bf16lo(w4[e2 >> 1]);
      }
    }
    __syncthreads();
    if (l0 == ltab0) prefetch();
    SP_STAMP(11);
    // x[h][w] = q_h . W_w in fp64 on the tensor cores: warp w owns W rows
    // 8 (w & 7) .. + 7 over the K half w >> 3; x = (K half 0) + (K half 1) -- the
    // chained prologue's decomposition, so the LUTs agree bit for bit
    {
      const int nt8 = warp & 7, kh = warp >> 3;
      double d0 = 0.0, d1 = 0.0;
      const int kr = lane & 3, col = lane >> 2;
      // the newest key's bits (fp32, t ascending: the SIMT prefill's order) on warps
      // 14-15, concurrently with the DMMA, when those warps have no DMMA rows
      const bool early_app = app && nw <= 48;
      if (early_app && warp >= 14) {
        const int w = tid - 448;
        bool bit = false;
        if (w < nw) {
          float x = 0.f;
#pragma unroll 32
          for (int t = 0; t < kD; ++t) x = fmaf(wsm[t * kSpFWs + w], s_ks[t], x);
          bit = x >= 0.f;                                                // sign(0) = +1 (R-3)
        }
        s_bits[w] = bit ? 1u : 0u;
      }
      if (nt8 * 8 < nw) {
#pragma unroll 8
        for (int k0 = kh * (kD / 2); k0 < (kh + 1) * (kD / 2); k0 += 4) {
          const double av = qs[(k0 + kr) * kSpFQs + col];
          const double bv = (double)wsm[(k0 + kr) * kSpFWs + nt8 * 8 + col];
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
            s_fx[((h * 8 + bit) * 2 + 1) * kSpTpp + tl] = fp;
            s_fx[((h * 8 + bit) * 2 + 0) * kSpTpp + tl] = fm;
          }
        }
      }
    }
    // append (when not done above): the newest key's bits on these tables
    if (app && nw > 48 && tid < 64) {
      bool bit = false;
      if (tid < nw) {
        float x = 0.f;
#pragma unroll 16
        for (int t = 0; t < kD; ++t) x = fmaf(wsm[t * kSpFWs + tid], s_ks[t], x);
        bit = x >= 0.f;                                                  // sign(0) = +1 (R-3)
      }
      s_bits[tid] = bit ? 1u : 0u;
    }
    __syncthreads();
    SP_STAMP(16);
    // half tables (fp64 products, rounded once): one (h, table, half) per thread
    if (tid < NH * kSpTpp * 2) {
      const int hi = tid & 1, tl = (tid >> 1) & (kSpTpp - 1), h = tid >> 4;
      if (tl < ntab) {
        double f[4][2];
#pragma unroll
        for (int bit = 0; bit < 4; ++bit) {
          const int ib = hi * 4 + bit;
          const bool ok = ib < P && (l0 + tl) < L;
          f[bit][0] = ok ? (double)s_fx[((h * 8 + ib) * 2 + 0) * kSpTpp + tl] : 1.0;
          f[bit][1] = ok ? (double)s_fx[((h * 8 + ib) * 2 + 1) * kSpTpp + tl] : 1.0;
        }
        double p01[4], p012[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) p01[e] = f[0][e & 1] * f[1][e >> 1];
#pragma unroll
        for (int e = 0; e < 8; ++e) p012[e] = p01[e & 3] * f[2][e >> 2];
#pragma unroll
        for (int e = 0; e < 16; ++e) s_half[((h * 2 + hi) * 16 + e) * kSpTpp + tl] = (float)(p012[e & 7] * f[3][e >> 3]);
      }
    }
    SP_STAMP(17);
    if (tid < kSpTpp) { s_tmm[tid] = 0x7F800000u; s_tmm[kSpTpp + tid] = 0u; }
    if (app && tid < ntab) {   // code byte of table l0 + tid (padding tables write 0)
      const int l = l0 + tid;
      uint32_t code = 0;
      if (l < L)
        for (int i = 0; i < P; ++i) code |= s_bits[tid * P + i] << i;   // row i -> bit i (R-4)
      const int M = (LP < 32 ? LP : 32) - 1;
      const int s = (l & ~M) | ((l - jn) & M);
      a.codes[kvrow * a.N_max * LP + code_off(jn, s, LP)] = (uint8_t)code;
    }
    __syncthreads();
    // LUT columns of these tables -> the row's LUT image in global memory.  Column
    // of table l: l (LP >= 32), or l, l + LP, ... < 32 (LP < 32, replicated)
    if (LP >= 32 && (ntab & 3) == 0) {
      const int ng = ntab >> 2;                               // 1 or 2 (kSpTpp = 8)
      float4 mn4 = make_float4(INFINITY, INFINITY, INFINITY, INFINITY), mx4 = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int e = tid; e < 256 * ng; e += kSpThreads) {
        const int gq = e % ng, rr = e / ng;
        const int tl = gq * 4, l = l0 + tl;
        float4 T = make_float4(0.f, 0.f, 0.f, 0.f);
        if (rr < R) {
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const float4 lo = *reinterpret_cast<const float4*>(s_half + ((h * 2 + 0) * 16 + (rr & 15)) * kSpTpp + tl);
            const float4 hv = *reinterpret_cast<const float4*>(s_half + ((h * 2 + 1) * 16 + (rr >> 4)) * kSpTpp + tl);
            T.x = fmaf(lo.x, hv.x, T.x);
            T.y = fmaf(lo.y, hv.y, T.y);
            T.z = fmaf(lo.z, hv.z, T.z);
            T.w = fmaf(lo.w, hv.w, T.w);
          }
          if (l + 0 >= L) T.x = 0.f;
          if (l + 1 >= L) T.y = 0.f;
          if (l + 2 >= L) T.z = 0.f;
          if (l + 3 >= L) T.w = 0.f;
          mn4.x = fminf(mn4.x, T.x); mn4.y = fminf(mn4.y, T.y); mn4.z = fminf(mn4.z, T.z); mn4.w = fminf(mn4.w, T.w);
          mx4.x = fmaxf(mx4.x, T.x); mx4.y = fmaxf(mx4.y, T.y); mx4.z = fmaxf(mx4.z, T.z); mx4.w = fmaxf(mx4.w, T.w);
        }
        *reinterpret_cast<float4*>(glut + rr * 64 + l) = T;
      }
      // lanes with the same table group (gq = tid % ng, ng in {1, 2}): xor offsets >= ng
      for (int o = 16; o >= ng; o >>= 1) {
        mn4.x = fminf(mn4.x, __shfl_xor_sync(kFull, mn4.x, o)); mx4.x = fmaxf(mx4.x, __shfl_xor_sync(kFull, mx4.x, o));
        mn4.y = fminf(mn4.y, __shfl_xor_sync(kFull, mn4.y, o)); mx4.y = fmaxf(mx4.y, __shfl_xor_sync(kFull, mx4.y, o));
        mn4.z = fminf(mn4.z, __shfl_xor_sync(kFull, mn4.z, o)); mx4.z = fmaxf(mx4.z, __shfl_xor_sync(kFull, mx4.z, o));
        mn4.w = fminf(mn4.w, __shfl_xor_sync(kFull, mn4.w, o)); mx4.w = fmaxf(mx4.w, __shfl_xor_sync(kFull, mx4.w, o));
      }
      if (lane < ng) {   // entries are >= 0: float order = bit order
        const int tl = lane * 4;
        const float m4[4] = {mn4.x, mn4.y, mn4.z, mn4.w}, x4[4] = {mx4.x, mx4.y, mx4.z, mx4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          atomicMin(&s_tmm[tl + u], __float_as_uint(m4[u]));
          atomicMax(&s_tmm[kSpTpp + tl + u], __float_as_uint(x4[u]));
        }
      }
    } else {
      float mn1 = INFINITY, mx1 = 0.f;                       // table tid & 7 (fixed per thread)
      for (int e = tid; e < 256 * kSpTpp; e += kSpThreads) {
        const int tl = e & (kSpTpp - 1), rr = e / kSpTpp;
        if (tl >= ntab) continue;
        const int l = l0 + tl;
        float T = 0.f;
        if (l < L && rr < R) {
#pragma unroll
          for (int h = 0; h < NH; ++h)
            T = fmaf(s_half[((h * 2 + 0) * 16 + (rr & 15)) * kSpTpp + tl], s_half[((h * 2 + 1) * 16 + (rr >> 4)) * kSpTpp + tl], T);
        }
        if (rr < R) { mn1 = fminf(mn1, T); mx1 = fmaxf(mx1, T); }
        if (LP >= 32) glut[rr * 64 + l] = T;
        else for (int cc = l; cc < 32; cc += LP) glut[rr * 64 + cc] = T;
      }
#pragma unroll
      for (int o = 16; o >= kSpTpp; o >>= 1) {
        mn1 = fminf(mn1, __shfl_xor_sync(kFull, mn1, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(kFull, mx1, o));
      }
      if (lane < kSpTpp && lane < ntab) {
        atomicMin(&s_tmm[lane], __float_as_uint(mn1));
        atomicMax(&s_tmm[kSpTpp + lane], __float_as_uint(mx1));
      }
    }
    __syncthreads();
    SP_STAMP(18);
    if (tid < ntab) {
      float* tmm = reinterpret_cast<float*>(rw + lay.tmm());
      tmm[2 * (l0 + tid)] = __uint_as_float(s_tmm[tid]);
      tmm[2 * (l0 + tid) + 1] = __uint_as_float(s_tmm[kSpTpp + tid]);
    }
  }
  __syncthreads();
  if (tid == 0) {   // my norm bounds -> the row
    float mn = INFINITY, mx = 0.f;
#pragma unroll
    for (int w = 0; w < kSpWarps; ++w) { mn = fminf(mn, s_red[w]); mx = fmaxf(mx, s_red[kSpWarps + w]); }
    float4* st = reinterpret_cast<float4*>(rw + lay.stat()) + c;
    *st = make_float4(mn, mx, 0.f, 0.f);
  }
  SP_STAMP(1);
  sp_arrive(bar);
  sp_wait(bar, (++nb) * C);
  SP_STAMP(2);

  // ===== B. LUT, score range, scores + level-0 histogram ==========================
  if (i_late >= 0) {   // the new key's tile (its code bytes and norm written before the barrier)
    const int ti = t0 + lt;
    issue_tile<LP>(ring + i_late * TSt::BYTES, crow + (size_t)ti * 32 * LP, vrow + ti * 32, lane);
    cpa_commit();
  }
  float2 tmm2 = make_float2(0.f, 0.f), tmm3 = make_float2(0.f, 0.f);
  float4 st4 = make_float4(INFINITY, 0.f, 0.f, 0.f);
  {   // LUT image, per-table min / max and the CTAs' norm ranges: one round trip
    if (warp == 0) {
      const float2* tmm = reinterpret_cast<const float2*>(rw + lay.tmm());
      if (lane < LP) tmm2 = __ldcg(tmm + lane);
      if (lane + 32 < LP) tmm3 = __ldcg(tmm + lane + 32);
    }
    if (warp >= 1 && warp <= 5 && tid - 32 < C) st4 = __ldcg(reinterpret_cast<const float4*>(rw + lay.stat()) + (tid - 32));
    const uint4* src = reinterpret_cast<const uint4*>(glut);
    uint4* dst = reinterpret_cast<uint4*>(lut);
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + tid + u * kSpThreads);
#pragma unroll
    for (int u = 0; u < 8; ++u) dst[tid + u * kSpThreads] = v[u];
  }
  for (int i = tid; i < kSpBins; i += kSpThreads) s_hist[i] = 0u;
  {   // row norm range: warps 1..5 hold the CTAs' (min, max) (C <= 160)
    float mn = st4.x, mx = st4.y;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(kFull, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
    }
    if (lane == 0 && warp >= 1 && warp <= 5) { s_red[warp] = mn; s_red[kSpWarps + warp] = mx; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w <= 5; ++w) { mn = fminf(mn, s_red[w]); mx = fmaxf(mx, s_red[kSpWarps + w]); }
      s_bound[0] = mn;
      s_bound[1] = mx;
    }
    __syncthreads();
  }
  if (warp == 0) {   // LUT range: sum over the tables of their min / max entry
    float smn = tmm2.x + tmm3.x, smx = tmm2.y + tmm3.y;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      smn += __shfl_xor_sync(kFull, smn, o);
      smx += __shfl_xor_sync(kFull, smx, o);
    }
    if (lane == 0) {
      // generous margins: the bins only have to be monotone in the score; keys
      // outside [lo, hi] fall into the edge bins (still exact)
      const float lo = fmaxf(0.f, smn * s_bound[0] * 0.999f);
      const float hi = smx * s_bound[1] * 1.001f;
      const uint32_t klo = f2key(lo), khi = f2key(fmaxf(hi, lo));
      const uint32_t span = khi - klo;
      s_dec[4] = klo;
      s_dec[5] = span < (uint32_t)kSpBins ? 0u : (uint32_t)((32 - __clz(span)) - 11);
    }
  }
  __syncthreads();
  const uint32_t klo0 = s_dec[4], sh0 = s_dec[5];
  SP_STAMP(3);
  uint32_t nvalid = 0, nforced = 0;
  {
    uint32_t pk[16];
#pragma unroll
    for (int m = 0; m < 16; ++m)
      pk[m] = (uint32_t)(((2 * m + lane) & 31) << 2) | ((uint32_t)(((2 * m + 1 + lane) & 31) << 2) << 8);
    const uint8_t* mrow = a.mask ? a.mask + (size_t)b * a.N_max : nullptr;
    float* srow = a.scores + (size_t)row * a.N_max;
    for (int i = 0; i < my; ++i) {
      if (i == i_late) cpa_wait<0>();
      else if (nst == 4) cpa_wait<3>();
      else cpa_wait<2>();
      const char* st = ringp + (i % nst) * TSt::BYTES;
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
          v[u] = *reinterpret_cast<const float*>(smem + ((ss & 32) ? 128 : 0) + addr);
        }
        const uint64_t pv = (uint64_t)__float_as_uint(v[0]) | ((uint64_t)__float_as_uint(v[1]) << 32);
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(pv));
      }
      // the next tile into the stage just read (its lanes' own bytes)
      if (i + nst < my) {
        const int ti = t0 + warp + (i + nst) * kSpWarps;
        issue_tile<LP>(ring + (i % nst) * TSt::BYTES, crow + (size_t)ti * 32 * LP, vrow + ti * 32, lane);
      }
      cpa_commit();
      const float score = vn * (__uint_as_float((uint32_t)acc) + __uint_as_float((uint32_t)(acc >> 32)));
      const int li = (warp + i * kSpWarps) * 32 + lane;   // slice-local index
      const int j = base + li;
      const bool ok = li < len && (!mrow || mrow[j]);
      srow[j] = ok ? score : -INFINITY;
      uint32_t key = 0u;
      if (ok) key = (j < a.sink || j >= n - a.window) ? 0xFFFFFFFFu : f2key(score);
      keys[li] = key;
      nvalid += key != 0u;
      nforced += key == 0xFFFFFFFFu;
      if (key != 0u && key != 0xFFFFFFFFu) {
        const uint32_t d = key > klo0 ? key - klo0 : 0u;
        atomicAdd(&s_hist[min((uint32_t)(kSpBins - 1), d >> sh0)], 1u);
      }
    }
    cpa_wait<0>();
    // keys past the valid prefix: -inf scores, invalid keys
    for (int li = vt * 32 + tid; li < slen; li += kSpThreads) {
      srow[base + li] = -INFINITY;
      keys[li] = 0u;
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    nvalid += __shfl_xor_sync(kFull, nvalid, o);
    nforced += __shfl_xor_sync(kFull, nforced, o);
  }
  if (lane == 0) { s_w[warp] = nvalid; s_w2[warp] = nforced; }
  __syncthreads();
  uint32_t my_valid = 0, my_forced = 0;
#pragma unroll
  for (int w = 0; w < kSpWarps; ++w) { my_valid += s_w[w]; my_forced += s_w2[w]; }
  // publish: level-0 bins, my counts (per CTA and row totals)
  for (int i = tid; i < kSpBins; i += kSpThreads) {
    const uint32_t v = s_hist[i];
    if (v) sp_red_add(gh + i, v);
  }
  if (tid == 0) {
    if (my_valid) sp_red_add(gh + kSpBins, my_valid);
    if (my_forced) sp_red_add(gh + kSpBins + 1, my_forced);
    uint4* inf = reinterpret_cast<uint4*>(rw + lay.info()) + c;
    *inf = make_uint4(my_valid, my_forced, 0u, 0u);
  }
  SP_STAMP(4);
  sp_arrive(bar);
  sp_wait(bar, (++nb) * C);
  SP_STAMP(5);

  // ===== C. exact top-k over the row ===============================================
  {
    const uint4* src = reinterpret_cast<const uint4*>(gh);
    if (tid < kSpBins / 4) reinterpret_cast<uint4*>(s_hist)[tid] = __ldcg(src + tid);
    if (tid == 0) { s_dec[6] = __ldcg(gh + kSpBins); s_dec[7] = __ldcg(gh + kSpBins + 1); }
  }
  __syncthreads();
  const uint32_t tvalid = s_dec[6], tforced = s_dec[7];
  const uint32_t k_eff = min((uint32_t)a.k, tvalid);
  // selection: keys > T, plus the first `quota` keys == T (row index order)
  uint32_t T = 0u, quota = 0u;
  // phase C / D shared memory: [L: the attention list | resolve scratch | attention ring]
  int32_t* slist = reinterpret_cast<int32_t*>(smem);
  char* scr = smem + sp_scr_off(a.S);
  uint4* s_info = reinterpret_cast<uint4*>(scr);                        // [C]
  uint32_t* s_off = reinterpret_cast<uint32_t*>(scr + 160 * 16);        // [C + 1]
  uint32_t* s_cand = reinterpret_cast<uint32_t*>(scr + 4096);           // [kSpCandCap]
  const uint16_t* Kb = a.K + kvrow * a.N_max * kD;
  const uint16_t* Vb = a.V + kvrow * a.N_max * kD;
  const uint32_t att_ring = smem_u32(smem + sp_att_off(a.S)) + (uint32_t)warp * (2 * kTileBytes);
  int n_list = 0;           // valid entries of slist for the gathers
  bool list = false;        // the final bin is wider than one key value
  // K / V rows of slist[16 t, 16 t + 16) into stage st of this warp's ring
  // (cp.async, zero-filled past n_list)
  auto att_issue = [&](int t, int st) {
    const int row0 = t * kTileRows;
    const uint32_t kbuf = att_ring + st * kTileBytes, vbuf = kbuf + kTileRows * 256;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int cc = (it * 32 + lane) & 15, rr = (it * 32 + lane) >> 4;
      const int i = row0 + rr;
      const bool v = i < n_list;
      const int tok = v ? base + slist[i] : 0;
      cp16(kbuf + swz(rr, cc), Kb + (size_t)tok * kD + cc * 8, v);
      cp16(vbuf + swz(rr, cc), Vb + (size_t)tok * kD + cc * 8, v);
    }
  };
  int mode;   // 0: all valid keys; 1: forced keys only; 2: threshold from candidates
  uint32_t blo = 0, bhi = 0;   // final bracket (mode 2)
  if (k_eff == tvalid) {
    mode = 0;
  } else if (k_eff <= tforced) {
    mode = 1;
    T = 0xFFFFFFFFu;
    quota = k_eff;
  } else {
    mode = 2;
    uint32_t need = k_eff - tforced;      // rank among regular keys
    // level 0 bracket: bins over [klo0, ...) with clamped edges
    unsigned long long lo = klo0;
    uint32_t sh = sh0;
    sp_locate(s_hist, need, s_w, s_dec);
    uint32_t bs = s_dec[0], nd = s_dec[1], cb = s_dec[2];
    // key range of bin bs (edge bins extend to the regular key range [1, 0xFFFFFFFE])
    auto bin_range = [&](uint32_t bin, bool clamped, uint32_t& r0, uint32_t& r1) {
      unsigned long long x0 = lo + ((unsigned long long)bin << sh);
      unsigned long long x1 = lo + ((unsigned long long)(bin + 1) << sh) - 1ull;
      if (clamped && bin == 0) x0 = 1ull;
      if (clamped && bin == kSpBins - 1) x1 = 0xFFFFFFFEull;
      r0 = (uint32_t)min(x0, 0xFFFFFFFEull);
      r1 = (uint32_t)min(x1, 0xFFFFFFFEull);
    };
    bin_range(bs, true, blo, bhi);
    int level = 0;
    while (cb > (uint32_t)kSpCandCap && blo != bhi && level + 1 < kSpLevels) {
      // refinement: 2048 bins over [blo, bhi], keys inside only
      ++level;
      lo = blo;
      const uint32_t span = bhi - blo;
      sh = span < (uint32_t)kSpBins ? 0u : (uint32_t)((32 - __clz(span)) - 11);
      for (int i = tid; i < kSpBins; i += kSpThreads) s_hist[i] = 0u;
      __syncthreads();
      for (int li = tid; li < slen; li += kSpThreads) {
        const uint32_t key = keys[li];
        if (key >= blo && key <= bhi && key != 0xFFFFFFFFu) atomicAdd(&s_hist[(key - blo) >> sh], 1u);
      }
      __syncthreads();
      uint32_t* ghl = gh + (size_t)level * kSpHistWords;
      for (int i = tid; i < kSpBins; i += kSpThreads) {
        const uint32_t v = s_hist[i];
        if (v) sp_red_add(ghl + i, v);
      }
      sp_arrive(bar);
      sp_wait(bar, (++nb) * C);
      if (tid < kSpBins / 4) reinterpret_cast<uint4*>(s_hist)[tid] = __ldcg(reinterpret_cast<const uint4*>(ghl) + tid);
      __syncthreads();
      need = nd;
      sp_locate(s_hist, need, s_w, s_dec);
      bs = s_dec[0];
      nd = s_dec[1];
      cb = s_dec[2];
      bin_range(bs, false, blo, bhi);
    }
    // candidates: my keys in [blo, bhi] and my keys above bhi (forced included)
    uint32_t ab = 0;
    if (tid == 0) { s_dec[3] = 0u; }
    __syncthreads();
    list = blo != bhi;
    uint2* gc = reinterpret_cast<uint2*>(rw + lay.cand()) + (size_t)c * kSpCandCap;
    for (int li = tid; li < slen; li += kSpThreads) {
      const uint32_t key = keys[li];
      ab += (key != 0u && key > bhi) ? 1u : 0u;
      if (key >= blo && key <= bhi && key != 0u && key != 0xFFFFFFFFu) {
        const uint32_t sl = atomicAdd(&s_dec[3], 1u);
        if (list && sl < (uint32_t)kSpCandCap) gc[sl] = make_uint2(key, (uint32_t)li);
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ab += __shfl_xor_sync(kFull, ab, o);
    if (lane == 0) s_w[warp] = ab;
    __syncthreads();
    if (tid == 0) {
      uint32_t tot = 0;
#pragma unroll
      for (int w = 0; w < kSpWarps; ++w) tot += s_w[w];
      uint4* inf = reinterpret_cast<uint4*>(rw + lay.info()) + c;
      *inf = make_uint4(my_valid, my_forced, tot, s_dec[3]);
    }
    SP_STAMP(6);
    sp_arrive(bar);
    sp_wait(bar, (++nb) * C);
    SP_STAMP(7);
    // every CTA's (valid, forced, above, #candidates) and the candidates
    // themselves (rank-major) into shared memory, one L2 round trip each
    if (tid < C) s_info[tid] = __ldcg(reinterpret_cast<const uint4*>(rw + lay.info()) + tid);
    __syncthreads();
    if (warp == 0) {
      uint32_t run = 0;
      for (int r0 = 0; r0 < C; r0 += 32) {
        const int r = r0 + lane;
        const uint32_t nc = r < C ? s_info[r].w : 0u;
        uint32_t inc = nc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, inc, o);
          if (lane >= o) inc += y;
        }
        if (r < C) s_off[r] = run + inc - nc;
        run += __shfl_sync(kFull, inc, 31);
      }
      if (lane == 0) s_off[C] = run;
    }
    __syncthreads();
    const uint32_t Ct = list ? s_off[C] : 0u;   // candidates in the final bin (row-wide) <= kSpCandCap
    // candidate i belongs to the CTA r with s_off[r] <= i < s_off[r + 1]
    auto owner = [&](uint32_t i) {
      int lo2 = 0, hi2 = C - 1;
      while (lo2 < hi2) {
        const int mid = (lo2 + hi2 + 1) >> 1;
        if (s_off[mid] <= i) lo2 = mid; else hi2 = mid - 1;
      }
      return lo2;
    };
    for (uint32_t i = tid; i < Ct; i += kSpThreads) {
      const int r = owner(i);
      s_cand[i] = __ldcg(reinterpret_cast<const uint2*>(rw + lay.cand()) + (size_t)r * kSpCandCap + (i - s_off[r])).x;
    }
    __syncthreads();
    SP_STAMP(19);
#ifdef SK_TRACE
    if (tid == 0) g_spread_trace[(blockIdx.y * gridDim.x + blockIdx.x) * 32 + 21] = Ct;
#endif
    if (list) {
      // T = the nd-th largest candidate: rank counting (small) or a 4-digit radix
      if (Ct <= 256u) {
        for (int i = tid; i < (int)Ct; i += kSpThreads) {
          const uint32_t me = s_cand[i];
          uint32_t gt = 0, eq = 0;
          int j2 = 0;
          for (; j2 + 4 <= (int)Ct; j2 += 4) {   // 16-B broadcast loads (s_cand is 16-B aligned)
            const uint4 v = *reinterpret_cast<const uint4*>(&s_cand[j2]);
            gt += (v.x > me) + (v.y > me) + (v.z > me) + (v.w > me);
            eq += (v.x == me) + (v.y == me) + (v.z == me) + (v.w == me);
          }
          for (; j2 < (int)Ct; ++j2) { const uint32_t x = s_cand[j2]; gt += x > me; eq += x == me; }
          if (gt < nd && gt + eq >= nd) { s_dec[0] = me; s_dec[1] = gt; }
        }
        __syncthreads();
        T = s_dec[0];
        quota = nd - s_dec[1];
      } else {
        uint32_t prefix = 0, k_rem = nd;
        for (int pass = 0; pass < 4; ++pass) {
          const int shift = 24 - 8 * pass;
          const uint32_t hmask = pass == 0 ? 0u : (0xFFFFFFFFu << (shift + 8));
          for (int i = tid; i < 256; i += kSpThreads) s_hist[i] = 0u;
          __syncthreads();
          for (int i = tid; i < (int)Ct; i += kSpThreads) {
            const uint32_t x = s_cand[i];
            if ((x & hmask) == (prefix & hmask)) atomicAdd(&s_hist[(x >> shift) & 255u], 1u);
          }
          __syncthreads();
          if (warp == 0) {
            uint32_t c8[8], tot = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) { c8[q] = s_hist[255 - (lane * 8 + q)]; tot += c8[q]; }
            uint32_t inc = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(kFull, inc, o);
              if (lane >= o) inc += y;
            }
            const uint32_t excl = inc - tot;
            const unsigned hb = __ballot_sync(kFull, excl < k_rem && inc >= k_rem);
            if (lane == __ffs(hb) - 1) {
              uint32_t run = excl;
              for (int q = 0; q < 8; ++q) {
                if (run + c8[q] >= k_rem) { s_dec[0] = 255 - (lane * 8 + q); s_dec[1] = k_rem - run; break; }
                run += c8[q];
              }
            }
          }
          __syncthreads();
          prefix |= s_dec[0] << shift;
          k_rem = s_dec[1];
          __syncthreads();
        }
        T = prefix;
        quota = k_rem;
      }
      SP_STAMP(20);
      // candidates > T / == T per CTA
      for (int r = tid; r < C; r += kSpThreads) { s_cgt[r] = 0u; s_ceq[r] = 0u; }
      __syncthreads();
      for (uint32_t i = tid; i < Ct; i += kSpThreads) {
        const uint32_t x = s_cand[i];
        if (x >= T) {
          const int r = owner(i);
          atomicAdd(x > T ? &s_cgt[r] : &s_ceq[r], 1u);
        }
      }
    } else {
      T = blo;       // the final bin is one key value: every key in it ties at T
      quota = nd;
    }
  }
  __syncthreads();

  // ---- per-CTA selected counts -> my output offset ---------------------------------
  // sel(r) = above(r) + gt(r) + min(eq(r), quota left); above(r) counts keys > the
  // final bin (mode 2), or all valid keys (mode 0), or 0 (mode 1)
  if (mode != 2) {
    if (tid < C) s_info[tid] = __ldcg(reinterpret_cast<const uint4*>(rw + lay.info()) + tid);
    __syncthreads();
  }
  if (warp == 0) {
    const bool lst = mode == 2 && blo != bhi;
    uint32_t gsel_before = 0, my_sel = 0, my_eqq = 0;
    uint32_t run_sel = 0, run_eq = 0;
    for (int r0 = 0; r0 < C; r0 += 32) {
      const int r = r0 + lane;
      uint32_t above = 0, gt = 0, eq = 0;
      if (r < C) {
        const uint4 inf = s_info[r];
        if (mode == 0) above = inf.x;
        else if (mode == 1) eq = inf.y;
        else {
          above = inf.z;
          if (lst) { gt = s_cgt[r]; eq = s_ceq[r]; }
          else eq = inf.w;
        }
      }
      // eq quota: the first `quota` keys == T in (rank, index) order
      uint32_t einc = eq;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, einc, o);
        if (lane >= o) einc += y;
      }
      const uint32_t ebefore = run_eq + einc - eq;
      const uint32_t eqq = quota > ebefore ? min(eq, quota - ebefore) : 0u;
      const uint32_t sel = above + gt + eqq;
      uint32_t sinc = sel;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, sinc, o);
        if (lane >= o) sinc += y;
      }
      if (r == c) { gsel_before = run_sel + sinc - sel; my_sel = sel; my_eqq = eqq; }
      run_eq += __shfl_sync(kFull, einc, 31);
      run_sel += __shfl_sync(kFull, sinc, 31);
    }
    gsel_before = __reduce_add_sync(kFull, gsel_before);   // set by one lane of one round only
    my_sel = __reduce_add_sync(kFull, my_sel);
    my_eqq = __reduce_add_sync(kFull, my_eqq);
    if (lane == 0) { s_dec[0] = gsel_before; s_dec[1] = my_sel; s_dec[2] = my_eqq; }
  }
  __syncthreads();
  const uint32_t pos0 = s_dec[0], nsel = s_dec[1], my_eqq = s_dec[2];
  SP_STAMP(8);

  // ---- my selection: the attention list and the idx output (one pass) -------------
  int32_t* orow = a.idx + (size_t)row * a.k;
  sp_select(keys, slen, 1u, 0xFFFFFFFFu, T, my_eqq, slist, 0, orow, pos0, base, s_w, s_w2);
  if (c == 0) {
    for (int p = (int)k_eff + tid; p < a.k; p += kSpThreads) orow[p] = -1;
    if (tid == 0) a.cnt[row] = (int)k_eff;
  }
  __syncthreads();
  n_list = (int)nsel;
  SP_STAMP(9);

  // ===== D. attention over my selected rows (L[0, nsel)), partial state to the row ==
  float* gpart = reinterpret_cast<float*>(rw + lay.part());
  {
    const int gid = lane >> 2, tig = lane & 3;
    float o[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) { o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f; }
    float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;
    const int ntiles = ((int)nsel + kTileRows - 1) / kTileRows;
    if (warp < kSpAttWarps) {
      uint32_t qb[8][2];
      {
        const bool hv = gid < NH;
        const uint32_t* qrow = reinterpret_cast<const uint32_t*>(s_q) + (hv ? gid : 0) * (kD / 2);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          qb[ks][0] = hv ? qrow[ks * 8 + tig] : 0u;
          qb[ks][1] = hv ? qrow[ks * 8 + 4 + tig] : 0u;
        }
      }
      int myt = 0;
      for (int t = warp; t < ntiles; t += kSpAttWarps) ++myt;
      if (myt > 0) att_issue(warp, 0);
      cp_commit();
      for (int j = 0; j < myt; ++j) {
        const int t = warp + j * kSpAttWarps;
        if (j + 1 < myt) att_issue(t + kSpAttWarps, (j + 1) & 1);
        cp_commit();
        cp_wait<1>();
        __syncwarp();
        const uint32_t kbuf = att_ring + (j & 1) * kTileBytes, vbuf = kbuf + kTileRows * 256;
        const int sel_cnt = (int)nsel;
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
          tA = fmaxf(tA, __shfl_xor_sync(kFull, tA, off));
          tB = fmaxf(tB, __shfl_xor_sync(kFull, tB, off));
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
          sA += __shfl_xor_sync(kFull, sA, off);
          sB += __shfl_xor_sync(kFull, sB, off);
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
    SP_STAMP(12);
    // merge the warps' states (attention ring reused) -> my partial in global
    float* sm_o = reinterpret_cast<float*>(smem + sp_att_off(a.S)); // [warps][8][128]
    float* sm_m = sm_o + kSpAttWarps * 8 * kD;
    float* sm_l = sm_m + kSpAttWarps * 8;
    if (warp < kSpAttWarps) {
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
    float* mypart = gpart + (size_t)c * NH * (kD + 2);
    for (int x = tid; x < NH * (kD + 2); x += kSpThreads) {
      const int h = x / (kD + 2), e = x % (kD + 2);
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kSpAttWarps; ++w) M = fmaxf(M, sm_m[w * 8 + h]);
      float val = M;
      if (e > 0) {
        float acc = 0.f;
        if (M != -INFINITY) {
#pragma unroll
          for (int w = 0; w < kSpAttWarps; ++w) {
            const float wt = exp2f(sm_m[w * 8 + h] - M);
            acc = fmaf(wt, e == 1 ? sm_l[w * 8 + h] : sm_o[(w * 8 + h) * kD + e - 2], acc);
          }
        }
        val = acc;
      }
      __stcg(mypart + x, val);
    }
  }
  // ---- LSE merge of the row's C partials, spread over the CTAs -------------------------
  // after a row barrier CTA c merges output elements [c per, (c + 1) per) of the
  // row's NH (kD + 1) (o and lse), each over the C partials in CTA order
  // (deterministic); the exit ticket's last CTA resets the row's counters
  SP_STAMP(13);
  sp_arrive(bar);
  sp_wait(bar, (++nb) * C);
  SP_STAMP(14);
  {
    constexpr float kLn2 = 0.6931471805599453f;
    const int tot_el = NH * (kD + 1);
    const int per = (tot_el + C - 1) / C;
    for (int x = c * per + tid; x < min(tot_el, (c + 1) * per); x += kSpThreads) {
      const int h = x / (kD + 1), e = x % (kD + 1);
      const float* ph = gpart + (size_t)h * (kD + 2);
      constexpr int kB = 8;   // partials in flight per thread
      float M = -INFINITY;
      for (int r0 = 0; r0 < C; r0 += kB) {
        float mv[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) mv[u] = r0 + u < C ? __ldcg(ph + (size_t)(r0 + u) * NH * (kD + 2)) : -INFINITY;
#pragma unroll
        for (int u = 0; u < kB; ++u) M = fmaxf(M, mv[u]);
      }
      float Ls = 0.f, O = 0.f;
      if (M != -INFINITY) {
        for (int r0 = 0; r0 < C; r0 += kB) {
          float mv[kB], lv[kB], ov[kB];
#pragma unroll
          for (int u = 0; u < kB; ++u) {
            const float* pr = ph + (size_t)(r0 + u) * NH * (kD + 2);
            const bool v = r0 + u < C;
            mv[u] = v ? __ldcg(pr) : -INFINITY;
            lv[u] = v ? __ldcg(pr + 1) : 0.f;
            ov[u] = v && e < kD ? __ldcg(pr + 2 + e) : 0.f;
          }
#pragma unroll
          for (int u = 0; u < kB; ++u) {
            const float wt = mv[u] == -INFINITY ? 0.f : exp2f(mv[u] - M);
            Ls = fmaf(wt, lv[u], Ls);
            O = fmaf(wt, ov[u], O);
          }
        }
      }
      const size_t oh = (size_t)b * a.H_q + h0 + h;
      if (e < kD) a.out[oh * kD + e] = (uint16_t)f2bf_bits(Ls > 0.f ? O / Ls : 0.f);
      else if (a.lse) a.lse[oh] = Ls > 0.f ? (M + log2f(Ls)) * kLn2 : -INFINITY;
    }
  }
  __syncthreads();
  if (tid == 0) {   // exit ticket: every CTA of the row is past its last barrier wait
    if (atomicAdd(bar + 1, 1u) == (uint32_t)(C - 1)) { bar[0] = 0u; bar[1] = 0u; }
  }
  SP_STAMP(10);
}

// ---------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------
size_t spread_smem_bytes(int LP, int S, int nst) { return (size_t)sp_zone(LP, S, nst) + (size_t)S * 4; }
constexpr size_t kSpStaticSmem = 14 * 1024;   // s_hist + small arrays (ptxas: <= 13.3 KB)
static int spread_stages(int LP, int S) {
  return spread_smem_bytes(LP, S, 4) + kSpStaticSmem <= 232448 ? 4 : 3;
}

// geometry: C CTAs per selection row over all SMs (one wave, cooperative); false
// when the row-spread step does not apply
bool spread_geometry(const socket_cfg& c, int& C, int& S) {
  if (c.group_mode != SOCKET_GROUP_KV_SHARED || c.P > 8) return false;
  const int Lp = code_slots(c.L);
  if (Lp > 64) return false;
  const int NH = c.H_q / c.H_kv;
  if (NH != 1 && NH != 2 && NH != 4 && NH != 8) return false;
  const long long rows = (long long)c.B * c.H_kv;
  const int sms = num_sms();
  if (rows < 1 || rows * 2 > sms || rows > 65535) return false;
  int cper = (int)(sms / rows);
  const int tiles = c.N_max / 32;
  cper = std::min(cper, tiles);
  S = (tiles + cper - 1) / cper * 32;
  C = (c.N_max + S - 1) / S;
  if (C > 160) return false;                                   // per-CTA count arrays
  // shared memory: zone + keys + static state
  if (spread_smem_bytes(Lp, S, 3) + kSpStaticSmem > 232448) return false;
  return true;
}

size_t spread_workspace_bytes(const socket_cfg& c) {
  int C, S;
  if (!spread_geometry(c, C, S)) return 0;
  const SpLayout lay{C, c.H_q / c.H_kv};
  return (size_t)c.B * c.H_kv * lay.words() * 4;
}

socket_status launch_spread_step(const socket_cfg& c, const void* q, void* K, void* V,
                                 const void* W, uint8_t* codes, float* vnorm, const int32_t* seq_lens,
                                 const uint8_t* mask, int do_append, const void* k_new,
                                 const void* v_new, int k, int sink, int window,
                                 float* scores, int32_t* idx, int32_t* cnt, void* out, float* lse,
                                 void* ws, cudaStream_t st) {
  int C, S;
  if (!spread_geometry(c, C, S)) return fail(SOCKET_EUNSUPPORTED, "spread step: shape not supported");
  const int Lp = code_slots(c.L);
  const int NH = c.H_q / c.H_kv;
  SpreadArgs a;
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
  a.ws = static_cast<uint32_t*>(ws);
  a.row_words = SpLayout{C, NH}.words();
  a.H_q = c.H_q;
  a.H_kv = c.H_kv;
  a.N_max = c.N_max;
  a.L = c.L;
  a.P = c.P;
  a.k = k;
  a.sink = sink;
  a.window = window;
  a.do_append = do_append;
  a.hard = c.scoring == SOCKET_SCORING_HARD;
  a.tau = c.tau;
  a.scale_log2 = c.sm_scale * kLog2eM;
  a.S = S;
  // tables per CTA, a multiple of 4: the LUT columns are written as float4 groups
  // starting at table c * tpc (C = 6 once gave 11 -> misaligned 16-B stores)
  a.tpc = ((Lp + C - 1) / C + 3) & ~3;
  a.nst = spread_stages(Lp, S);
  a.zone = sp_zone(Lp, S, a.nst);
  const size_t sm = spread_smem_bytes(Lp, S, a.nst);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, c.B * c.H_kv, 1);
  cfg.blockDim = dim3(kSpThreads, 1, 1);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // every CTA co-resident (row barriers)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;   // (measured: no launch-latency cost over a plain launch)
  cudaError_t e = cudaSuccess;
#define SK_SPREAD(N, LPV)                                                                         \
  if (NH == N && Lp == LPV) {                                                                     \
    auto kfn = spread_step_kernel<N, LPV>;                                                        \
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) \
      return fail(SOCKET_ECUDA, "spread step: shared memory request rejected");                  \
    e = cudaLaunchKernelEx(&cfg, kfn, a);                                                         \
  } else
  SK_SPREAD(1, 8) SK_SPREAD(1, 16) SK_SPREAD(1, 32) SK_SPREAD(1, 64)
  SK_SPREAD(2, 8) SK_SPREAD(2, 16) SK_SPREAD(2, 32) SK_SPREAD(2, 64)
  SK_SPREAD(4, 8) SK_SPREAD(4, 16) SK_SPREAD(4, 32) SK_SPREAD(4, 64)
  SK_SPREAD(8, 8) SK_SPREAD(8, 16) SK_SPREAD(8, 32) SK_SPREAD(8, 64)
  { return fail(SOCKET_EUNSUPPORTED, "spread step: heads / tables not instantiated"); }
#undef SK_SPREAD
  if (e != cudaSuccess) return fail(SOCKET_ECUDA, std::string("spread step launch: ") + cudaGetErrorString(e));
  return check_launch("spread_step_kernel");
}

}  // namespace sk
