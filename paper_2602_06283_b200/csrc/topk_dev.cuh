// Device side of the exact cluster top-k (Alg. 3 l.244, PAPER.md; sink/window
// P:686), used by topk_cluster_kernel and the sequence-shard protocol kernels
// (topk.cu).  Not part of the ABI.
#pragma once
#include <cooperative_groups.h>
#include <cstdlib>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace sk {

constexpr int kTopkThreads = 512;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kBins = 2048;
constexpr int kCandCap = 2048;
constexpr int kMaxCluster = 16;   // CTAs per cluster (non-portable maximum)

#ifdef SK_TRACE
// phase stamps (clock64 of thread 0 of every CTA), read by tools/trace_topk.py
static __device__ unsigned long long g_topk_trace[4096 * 16];   // per translation unit
#define TK_TRACE(i)                                                                          \
  do {                                                                                       \
    if (threadIdx.x == 0) {                                                                  \
      const int cta = blockIdx.y * gridDim.x + blockIdx.x;                                   \
      if (cta < 4096) g_topk_trace[cta * 16 + (i)] = clock64();                              \
    }                                                                                        \
  } while (0)
#else
#define TK_TRACE(i) \
  do {              \
  } while (0)
#endif

struct TopkArgs {
  // scores [rows][N_max] of keys at global positions index_base + j; the row
  // length is seq_lens[b] (total), the local valid count local_len(...)
  const float* scores;
  const int32_t* seq_lens;
  int rows, H_sel, N_max, k, sink, window;
  long long index_base;
  int per;                 // slice length per CTA (multiple of 128)
  uint32_t* gkeys;         // nullptr: slices in shared memory; else [rows][csize][per] global
  int32_t* idx;
  int32_t* cnt;
  float* sel_scores;
  // sequence-shard protocol: op 0 = select (socket_topk),
  // 1 = digest, 2 = window message, 3 = emit with a resolved threshold
  int op;
  int Q;                   // op 1: digest pairs per row
  uint32_t* digest;        // op 1 out: [rows][Q][2] (edge key, #keys >= edge)
  const uint32_t* state;   // op 2, 3 in: [rows][kStateWords]
  uint32_t* msg;           // op 2 out: [rows][kMsgWords]
};

// per-row state of the shard resolve (see shard_topk.cu)
constexpr int kStateWords = 8;   // lo, hi (0 = 2^32), k_eff, resolved, T, quota, need, -
constexpr int kMsgHdr = 8;       // lo, hi, above, wc, mode (0 keys, 1 histogram), sh, -, -
constexpr int kMsgCap = kBins;   // keys or histogram bins per message
constexpr int kMsgWords = kMsgHdr + kMsgCap;

__device__ __forceinline__ float load_elem(const TopkArgs& a, int row, int e) {
  return a.scores[(size_t)row * a.N_max + e];
}

// monotone key of local key e of a row with total length n_glob (invalid = 0,
// forced sink / local-window key = 0xFFFFFFFF; positions are global)
__device__ __forceinline__ uint32_t make_key(float s, int e, int n_glob, long long index_base, int sink,
                                             int window) {
  if (s == -INFINITY) return 0u;
  const long long pos = index_base + e;
  if (pos < sink || pos >= (long long)n_glob - window) return 0xFFFFFFFFu;
  return f2key(s);
}

// exclusive scan over the warps of one value per warp
__device__ __forceinline__ int block_excl_scan_warps(int v, int* sh, int warp, int lane, int& total) {
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  int pre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kTopkWarps; ++w) {
    const int x = sh[w];
    pre += (w < warp) ? x : 0;
    tot += x;
  }
  total = tot;
  return pre;
}

struct __align__(16) TopkShared {
  uint32_t hist[kBins];          // local histogram (radix fallback: two 256-bin buffers)
  uint32_t cand[kCandCap];       // local candidates: keys of the target bin
  uint32_t cidx[kCandCap];       // their slice-local indices
  uint32_t gcand[kCandCap];      // candidates gathered from the cluster, rank-major
  uint32_t rhist[256];           // local radix histogram for candidate resolve
  int scan[kTopkWarps];
  int scan2[kTopkWarps];
  uint32_t wab[kTopkWarps];      // per warp: keys strictly above the target bin (forced included)
  uint32_t wgt[kTopkWarps];      // per warp: local candidates > T
  uint32_t weq[kTopkWarps];      // per warp: local candidates == T
  uint32_t roff[17];             // gathered-candidate offset of every rank
  uint32_t rab[16];              // above-bin count of every rank
  uint32_t glob[4];              // cluster totals: nvalid, nforced, kmin, kmax
  uint32_t coarse[64];           // local histogram folded into 64 coarse bins (read remotely)
  uint32_t acc[2];               // lower ranks' candidates > T / == T
  alignas(16) uint32_t stat[8];  // nvalid, nforced, kmin, kmax, ncand, above, gt, eq (read remotely)
  uint32_t dec[4];
  // written by the other CTAs (pushed before a cluster barrier, never read remotely):
  uint4 sall[kMaxCluster];       // every rank's (nvalid, nforced, kmin, kmax)
  uint2 call[kMaxCluster];       // every rank's (#candidates, #keys above the target bin)
  uint32_t gall[kCandCap];       // every rank's candidates, rank r at [r * cap, r * cap + count)
};

__device__ __forceinline__ void topk_emit(const TopkArgs& a, uint32_t* keys, TopkShared& S, int row, int base,
                                          int len, uint32_t T, uint32_t quota, uint32_t k_out, bool counted,
                                          int32_t* sel_local, int* sel_lo, int* sel_cnt);

// Local exact select over a small candidate array: the `need`-th largest key
// (1-based) and how many candidates are strictly greater.
__device__ __forceinline__ void local_select(const uint32_t* c, int C, uint32_t need, TopkShared& S, int tid,
                             int warp, int lane, uint32_t& T, uint32_t& above) {
  uint32_t prefix = 0, k_rem = need;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    const uint32_t hmask = pass == 0 ? 0u : (0xFFFFFFFFu << (shift + 8));
    for (int i = tid; i < 256; i += kTopkThreads) S.rhist[i] = 0;
    __syncthreads();
    for (int i = tid; i < ((C + 31) & ~31); i += kTopkThreads) {
      const bool m = i < C && (c[i] & hmask) == (prefix & hmask);
      const uint32_t bin = m ? ((c[i] >> shift) & 255u) : 256u;
      const uint32_t peers = __match_any_sync(0xffffffffu, bin);
      if (m && lane == __ffs(peers) - 1) atomicAdd(&S.rhist[bin], (uint32_t)__popc(peers));
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t c8[8], tot = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) { c8[q] = S.rhist[255 - (lane * 8 + q)]; tot += c8[q]; }
      uint32_t inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const uint32_t excl = inc - tot;
      const unsigned hb = __ballot_sync(0xffffffffu, excl < k_rem && inc >= k_rem);
      if (lane == __ffs(hb) - 1) {
        uint32_t run = excl;
        for (int q = 0; q < 8; ++q) {
          if (run + c8[q] >= k_rem) { S.dec[0] = 255 - (lane * 8 + q); S.dec[1] = k_rem - run; break; }
          run += c8[q];
        }
      }
    }
    __syncthreads();
    prefix |= S.dec[0] << shift;
    k_rem = S.dec[1];
  }
  T = prefix;
  above = need - k_rem;
}

// Everything after the slice load: cluster statistics, the exact threshold T
// and tie quota, and the stable emit of idx / cnt (see the file header of
// topk.cu).  keys[] holds this CTA's slice (base, len) as monotone u32 keys
// (len rounded up to 128 with 0 = invalid), and (nvalid, nforced, kmin, kmax)
// are this thread's statistics of its loaded keys (kmin over regular keys,
// 0xFFFFFFFF if none).  If sel_local != NULL, the CTA's selected keys (global
// indices, ascending) are also written to sel_local[0 .. *sel_cnt), i.e. the
// CTA's contiguous share idx[row][*sel_lo .. *sel_lo + *sel_cnt).
__device__ __forceinline__ void topk_core(const TopkArgs& a, uint32_t* keys, TopkShared& S, int row,
                                       int n, int base, int len, uint32_t nvalid, uint32_t nforced,
                                       uint32_t kmin, uint32_t kmax, int32_t* sel_local,
                                       int* sel_lo, int* sel_cnt) {
  constexpr unsigned kFull = 0xffffffffu;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int csize = (int)cluster.num_blocks();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int len32 = (len + 31) & ~31;
  const int len128 = (len + 127) & ~127;
  const int nr = len128 >> 7;
  const int rpw = max(1, (nr + kTopkWarps - 1) / kTopkWarps);
  const int r0 = warp * rpw, r1 = min(nr, r0 + rpw);
  (void)n;
  if (tid < 8) S.stat[tid] = (tid == 2) ? 0xFFFFFFFFu : 0u;   // kmin starts at +max
  if (tid < kTopkWarps) { S.wgt[tid] = 0; S.weq[tid] = 0; }
  if (tid < 2) S.acc[tid] = 0;
  for (int i = tid; i < kBins; i += kTopkThreads) S.hist[i] = 0;
  __syncthreads();
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    nvalid += __shfl_xor_sync(kFull, nvalid, o);
    nforced += __shfl_xor_sync(kFull, nforced, o);
    kmin = min(kmin, __shfl_xor_sync(kFull, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(kFull, kmax, o));
  }
  if (lane == 0) {
    atomicAdd(&S.stat[0], nvalid);
    atomicAdd(&S.stat[1], nforced);
    atomicMin(&S.stat[2], kmin);
    atomicMax(&S.stat[3], kmax);
  }
  __syncthreads();
  // push my statistics to every rank (remote stores complete at the barrier;
  // the caller has made sure every CTA of the cluster is running)
  if (tid < csize)
    *cluster.map_shared_rank(&S.sall[crank], tid) = *reinterpret_cast<const uint4*>(S.stat);
  TK_TRACE(2);
  cluster.sync();
  // ---- 1. cluster totals from the pushed statistics (local reads) --------------
  if (warp == 0) {
    uint32_t v0 = 0, v1 = 0, v2 = 0xFFFFFFFFu, v3 = 0;
    if (lane < csize) {
      const uint4 rs = S.sall[lane];
      v0 = rs.x; v1 = rs.y; v2 = rs.z; v3 = rs.w;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      v0 += __shfl_xor_sync(kFull, v0, o);
      v1 += __shfl_xor_sync(kFull, v1, o);
      v2 = min(v2, __shfl_xor_sync(kFull, v2, o));
      v3 = max(v3, __shfl_xor_sync(kFull, v3, o));
    }
    if (lane == 0) { S.glob[0] = v0; S.glob[1] = v1; S.glob[2] = v2; S.glob[3] = v3; }
  }
  __syncthreads();
  const uint32_t tvalid = S.glob[0], tforced = S.glob[1], gmin = S.glob[2], gmax = S.glob[3];
  const uint32_t k_eff = min((uint32_t)a.k, tvalid);
  TK_TRACE(3);

  // ---- find T and quota --------------------------------------------------------
  uint32_t T = 0, quota = 0;            // select keys > T, plus `quota` keys == T
  bool done = false;
  if (k_eff == tvalid) {
    done = true;                         // everything valid is selected
  } else if (k_eff <= tforced) {
    T = 0xFFFFFFFFu;                     // only forced keys (they all tie at the max key)
    quota = k_eff;
    done = true;
  }
  const uint32_t need = k_eff - tforced;  // rank among regular keys (>= 1 when !done)
  bool fallback = false, counted = false;
  if (!done) {
    // 2. adaptive histogram over [gmin, gmax]
    // bin = (key - gmin) >> sh with the smallest sh that maps [gmin, gmax] into
    // kBins bins: monotone and exact (no division)
    const uint32_t span = gmax - gmin;
    const int sh = span < (uint32_t)kBins ? 0 : (32 - __clz(span)) - 11;
    for (int i = tid * 4; i < len128; i += kTopkThreads * 4) {
      const uint4 kv = *reinterpret_cast<const uint4*>(keys + i);
      const uint32_t k4[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (k4[e] != 0u && k4[e] != 0xFFFFFFFFu) atomicAdd(&S.hist[(k4[e] - gmin) >> sh], 1u);
    }
    // coarse histogram: 64 bins of 32 fine bins each (thread t folds bins 4t..4t+3,
    // 8 lanes per coarse bin)
    __syncthreads();
    {
      const uint4 h = *reinterpret_cast<const uint4*>(&S.hist[tid * 4]);
      uint32_t cs4 = h.x + h.y + h.z + h.w;
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) cs4 += __shfl_xor_sync(kFull, cs4, o);
      if ((lane & 7) == 0) S.coarse[tid >> 3] = cs4;
    }
    TK_TRACE(4);
    cluster.sync();
    TK_TRACE(5);
    // cluster sums, coarse then fine (DSMEM: csize x (64 + 32) words per CTA), each
    // followed by a descending suffix scan that locates the bin of rank `need`
    if (warp == 0) {
      uint32_t c0 = 0, c1 = 0;                 // coarse bins 63 - 2 lane, 62 - 2 lane
      {   // all ranks' loads in flight at once (a DSMEM load is ~200 cycles)
        uint32_t v0[kMaxCluster], v1[kMaxCluster];
#pragma unroll
        for (int r = 0; r < kMaxCluster; ++r) {
          const uint32_t* rc = cluster.map_shared_rank(S.coarse, r < csize ? r : 0);
          v0[r] = rc[63 - 2 * lane];
          v1[r] = rc[62 - 2 * lane];
        }
#pragma unroll
        for (int r = 0; r < kMaxCluster; ++r)
          if (r < csize) { c0 += v0[r]; c1 += v1[r]; }
      }
      const uint32_t tot = c0 + c1;
      uint32_t inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
      }
      const uint32_t excl = inc - tot;         // keys in coarse bins above mine
      const unsigned hit = __ballot_sync(kFull, excl < need && inc >= need);
      const int hl = __ffs(hit) - 1;
      const uint32_t ex_h = __shfl_sync(kFull, excl, hl), c0_h = __shfl_sync(kFull, c0, hl);
      const bool first = ex_h + c0_h >= need;
      const int cb = first ? 63 - 2 * hl : 62 - 2 * hl;
      const uint32_t need_c = need - (first ? ex_h : ex_h + c0_h);   // rank inside coarse bin cb
      // fine bins of cb: lane l holds bin cb*32 + 31 - l (descending)
      const int fb = cb * 32 + 31 - lane;
      uint32_t f = 0;
      {
        uint32_t v[kMaxCluster];
#pragma unroll
        for (int r = 0; r < kMaxCluster; ++r) v[r] = cluster.map_shared_rank(S.hist, r < csize ? r : 0)[fb];
#pragma unroll
        for (int r = 0; r < kMaxCluster; ++r) f += r < csize ? v[r] : 0u;
      }
      uint32_t finc = f;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, finc, o);
        if (lane >= o) finc += y;
      }
      const uint32_t fex = finc - f;
      if (fex < need_c && finc >= need_c) { S.dec[0] = (uint32_t)fb; S.dec[1] = need_c - fex; S.dec[2] = f; }
    }
    __syncthreads();
    const uint32_t bstar = S.dec[0], need2 = S.dec[1], C = S.dec[2];
    TK_TRACE(6);
    if (C <= (uint32_t)kCandCap) {
      // 3. candidate pass: keys of bin bstar -> S.cand (+ slice index); per warp the
      //    number of keys strictly above the bin (all of them are > T, forced included)
      // a lane scans 4 consecutive keys per 128-key round (same rounds per warp
      // as the emit pass, so the per-warp counts line up)
      uint32_t ab = 0;
      for (int r = r0; r < r1; ++r) {
        const int i0 = r * 128 + lane * 4;
        const uint4 kv = *reinterpret_cast<const uint4*>(keys + i0);
        const uint32_t k4[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t key = k4[e];
          const bool reg = key != 0u && key != 0xFFFFFFFFu;
          const uint32_t bin = (key - gmin) >> sh;
          ab += (key == 0xFFFFFFFFu || (reg && bin > bstar)) ? 1u : 0u;
          if (reg && bin == bstar) {              // rare: ~C / len of the keys
            const uint32_t sl = atomicAdd(&S.stat[4], 1u);
            S.cand[sl] = key;
            S.cidx[sl] = (uint32_t)(i0 + e);
          }
        }
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) ab += __shfl_xor_sync(kFull, ab, o);
      if (lane == 0) { S.wab[warp] = ab; atomicAdd(&S.stat[5], ab); }
      __syncthreads();
      // push (count, above) and -- when they fit my share of the buffer -- my
      // candidates to every rank, so that after the barrier all reads are local
      const int cap = kCandCap / csize;
      {
        const uint32_t nloc = S.stat[4], abv = S.stat[5];
        const int npush = 1 + (nloc <= (uint32_t)cap ? (int)nloc : 0);
        for (int e = tid; e < csize * npush; e += kTopkThreads) {
          const int r = e % csize, i = e / csize;
          if (i == 0) *cluster.map_shared_rank(&S.call[crank], r) = make_uint2(nloc, abv);
          else cluster.map_shared_rank(S.gall, r)[crank * cap + i - 1] = S.cand[i - 1];
        }
      }
      TK_TRACE(7);
      cluster.sync();
      TK_TRACE(8);
      // every rank's candidate count and above-bin count (local), rank-major offsets
      if (warp == 0) {
        uint32_t nc = 0, rab = 0;
        if (lane < csize) {
          const uint2 rs = S.call[lane];
          nc = rs.x;
          rab = rs.y;
        }
        uint32_t inc = nc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, inc, o);
          if (lane >= o) inc += y;
        }
        if (lane < csize) { S.roff[lane + 1] = inc; S.rab[lane] = rab; }
        if (lane == 0) S.roff[0] = 0;
        const unsigned over = __ballot_sync(kFull, lane < csize && nc > (uint32_t)cap);
        if (lane == 0) S.dec[3] = over;
      }
      __syncthreads();
      const bool pushed = S.dec[3] == 0u;   // else some rank had more than `cap`: read remotely
      for (int i = tid; i < (int)C; i += kTopkThreads) {
        int r = 0;
        while (r + 1 < csize && S.roff[r + 1] <= (uint32_t)i) ++r;
        S.gcand[i] = pushed ? S.gall[r * cap + i - (int)S.roff[r]]
                            : cluster.map_shared_rank(S.cand, r)[i - (int)S.roff[r]];
      }
      __syncthreads();
      // T = the need2-th largest candidate, above = candidates > T
      uint32_t above;
      if (C <= 192u) {
        // rank counting (O(C^2), small C): candidate i is T iff #greater < need2 <= #greater + #equal
        for (int i = tid; i < (int)C; i += kTopkThreads) {
          const uint32_t me = S.gcand[i];
          uint32_t gt = 0, eq = 0;
          int j = 0;
          for (; j + 4 <= (int)C; j += 4) {
            const uint4 v = *reinterpret_cast<const uint4*>(&S.gcand[j]);
            gt += (v.x > me) + (v.y > me) + (v.z > me) + (v.w > me);
            eq += (v.x == me) + (v.y == me) + (v.z == me) + (v.w == me);
          }
          for (; j < (int)C; ++j) { gt += S.gcand[j] > me; eq += S.gcand[j] == me; }
          if (gt < need2 && gt + eq >= need2) { S.dec[0] = me; S.dec[1] = gt; }   // ties write equal values
        }
        __syncthreads();
        T = S.dec[0];
        above = S.dec[1];
      } else {
        local_select(S.gcand, (int)C, need2, S, tid, warp, lane, T, above);
      }
      quota = need2 - above;
      TK_TRACE(9);
      // keys > T / == T before this CTA and per warp, from the candidate lists alone
      uint32_t gtb = 0, eqb = 0;
      for (int i = tid; i < (int)S.roff[crank]; i += kTopkThreads) {
        const uint32_t cv = S.gcand[i];
        gtb += cv > T;
        eqb += cv == T;
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        gtb += __shfl_xor_sync(kFull, gtb, o);
        eqb += __shfl_xor_sync(kFull, eqb, o);
      }
      if (lane == 0 && (gtb | eqb)) { atomicAdd(&S.acc[0], gtb); atomicAdd(&S.acc[1], eqb); }
      const int nloc = (int)S.stat[4];
      for (int i = tid; i < nloc; i += kTopkThreads) {
        const uint32_t cv = S.cand[i];
        const int w = (int)(S.cidx[i] >> 7) / rpw;
        if (cv > T) atomicAdd(&S.wgt[w], 1u);
        else if (cv == T) atomicAdd(&S.weq[w], 1u);
      }
      __syncthreads();
      counted = true;
    } else {
      fallback = true;
    }
  }
  if (fallback) {
    // 4-pass MSB radix select over the cluster (8-bit digits), regular keys only
    uint32_t prefix = 0, k_rem = need;
    uint32_t* h2 = S.hist;                  // two 256-bin buffers: hist[0..255], hist[256..511]
    cluster.sync();                          // everyone finished reading the 2048-bin histograms
    for (int i = tid; i < 512; i += kTopkThreads) h2[i] = 0;
    __syncthreads();
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      uint32_t* hb = h2 + (pass & 1) * 256;
      const uint32_t hmask = pass == 0 ? 0u : (0xFFFFFFFFu << (shift + 8));
      for (int i = tid; i < len32; i += kTopkThreads) {
        const uint32_t key = keys[i];
        const bool m = key != 0u && key != 0xFFFFFFFFu && (key & hmask) == (prefix & hmask);
        const uint32_t bin = m ? ((key >> shift) & 255u) : 256u;
        const uint32_t peers = __match_any_sync(kFull, bin);
        if (m && lane == __ffs(peers) - 1) atomicAdd(&hb[bin], (uint32_t)__popc(peers));
      }
      cluster.sync();
      if (warp == 0) {
        uint32_t c8[8], tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int bin = 255 - (lane * 8 + q);
          uint32_t s = 0, v[kMaxCluster];
#pragma unroll
          for (int c = 0; c < kMaxCluster; ++c) v[c] = *cluster.map_shared_rank(&hb[bin], c < csize ? c : 0);
#pragma unroll
          for (int c = 0; c < kMaxCluster; ++c) s += c < csize ? v[c] : 0u;
          c8[q] = s;
          tot += s;
        }
        uint32_t inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, inc, o);
          if (lane >= o) inc += y;
        }
        const uint32_t excl = inc - tot;
        const unsigned hbits = __ballot_sync(kFull, excl < k_rem && inc >= k_rem);
        if (lane == __ffs(hbits) - 1) {
          uint32_t run = excl;
          for (int q = 0; q < 8; ++q) {
            if (run + c8[q] >= k_rem) { S.dec[0] = 255 - (lane * 8 + q); S.dec[1] = k_rem - run; break; }
            run += c8[q];
          }
        }
      }
      // clear the other buffer (its last remote readers finished before this sync)
      for (int i = tid; i < 256; i += kTopkThreads) h2[((pass + 1) & 1) * 256 + i] = 0;
      __syncthreads();
      prefix |= S.dec[0] << shift;
      k_rem = S.dec[1];
    }
    T = prefix;
    quota = k_rem;
  }

  // ---- stable compaction ------------------------------------------------------
  TK_TRACE(10);
  topk_emit(a, keys, S, row, base, len, T, quota, k_eff, counted, sel_local, sel_lo, sel_cnt);
}

// Stable compaction of a row's selection: keys > T plus the first `quota` keys
// == T in index order, written in ascending index order.  Output position of a
// selected key = gt_rank + min(eq_rank, quota), where gt_rank / eq_rank count
// keys > T / == T at smaller indices (row-global).  If `counted`, the per-warp
// counts come from topk_core's candidate pass (S.wab / S.wgt / S.weq / S.rab /
// S.acc); otherwise a count pass computes them.  k_out = the row's total count
// (written to cnt by CTA 0).  Ends with a cluster barrier.
__device__ __forceinline__ void topk_emit(const TopkArgs& a, uint32_t* keys, TopkShared& S, int row, int base,
                                          int len, uint32_t T, uint32_t quota, uint32_t k_out, bool counted,
                                          int32_t* sel_local, int* sel_lo, int* sel_cnt) {
  constexpr unsigned kFull = 0xffffffffu;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int len128 = (len + 127) & ~127;
  const int nr = len128 >> 7;
  const int rpw = max(1, (nr + kTopkWarps - 1) / kTopkWarps);
  const int r0 = warp * rpw, r1 = min(nr, r0 + rpw);
  int gbase, ebase;   // row-global ranks of this warp's first key
  uint32_t cta_gb = 0, cta_eb = 0, cta_gt = 0, cta_eq = 0;   // this CTA's share (sel_local)
  if (counted) {
    uint32_t gb = S.acc[0], eb = S.acc[1];
    for (int r = 0; r < crank; ++r) gb += S.rab[r];
    uint32_t gw = 0, ew = 0;
    for (int w = 0; w < warp; ++w) { gw += S.wab[w] + S.wgt[w]; ew += S.weq[w]; }
    gbase = (int)(gb + gw);
    ebase = (int)(eb + ew);
    cta_gb = gb;
    cta_eb = eb;
    for (int w = 0; w < kTopkWarps; ++w) { cta_gt += S.wab[w] + S.wgt[w]; cta_eq += S.weq[w]; }
  } else {
    // count pass: keys > T / == T per warp, then per CTA, then cluster prefix
    uint32_t g = 0, e = 0;
    for (int r = r0; r < r1; ++r) {
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const uint32_t key = keys[r * 128 + x * 32 + lane];
        g += __popc(__ballot_sync(kFull, key > T));
        e += __popc(__ballot_sync(kFull, key != 0u && key == T));
      }
    }
    if (lane == 0) { S.scan[warp] = (int)g; S.scan2[warp] = (int)e; }
    __syncthreads();
    uint32_t gw = 0, ew = 0, gtot = 0, etot = 0;
#pragma unroll
    for (int w = 0; w < kTopkWarps; ++w) {
      const uint32_t xg = (uint32_t)S.scan[w], xe = (uint32_t)S.scan2[w];
      gw += w < warp ? xg : 0u; ew += w < warp ? xe : 0u;
      gtot += xg; etot += xe;
    }
    if (tid == 0) { S.stat[6] = gtot; S.stat[7] = etot; }
    cluster.sync();
    uint32_t gb = 0, eb = 0;
    {
      uint32_t vg[kMaxCluster], ve[kMaxCluster];
#pragma unroll
      for (int r = 0; r < kMaxCluster; ++r) {
        const uint32_t* rs = cluster.map_shared_rank(S.stat, r < crank ? r : 0);
        vg[r] = rs[6];
        ve[r] = rs[7];
      }
#pragma unroll
      for (int r = 0; r < kMaxCluster; ++r)
        if (r < crank) { gb += vg[r]; eb += ve[r]; }
    }
    gbase = (int)(gb + gw);
    ebase = (int)(eb + ew);
    cta_gb = gb;
    cta_eb = eb;
    cta_gt = gtot;
    cta_eq = etot;
  }
  TK_TRACE(11);
  const int sel0 = (int)cta_gb + min((int)cta_eb, (int)quota);
  if (sel_lo) {
    *sel_lo = sel0;
    *sel_cnt = (int)(cta_gb + cta_gt) + min((int)(cta_eb + cta_eq), (int)quota) - sel0;
  }
  int32_t* orow = a.idx + (size_t)row * a.k;
  float* srow = a.sel_scores ? a.sel_scores + (size_t)row * a.k : nullptr;
  const int q = (int)quota;
  for (int r = r0; r < r1; ++r) {
    // lane owns keys 4 lane .. 4 lane + 3 of the round (index order within the
    // round = lane-major); ties at T (rare) take the per-32 ballot path below
    const int i0 = r * 128 + lane * 4;
    const uint4 kv = *reinterpret_cast<const uint4*>(keys + i0);
    const uint32_t k4[4] = {kv.x, kv.y, kv.z, kv.w};
    const bool anyeq = (k4[0] == T) | (k4[1] == T) | (k4[2] == T) | (k4[3] == T);
    if (!__any_sync(kFull, anyeq && T != 0u)) {
      unsigned gm[4];
      int pre = 0, tot = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        gm[e] = __ballot_sync(kFull, k4[e] > T);
        pre += __popc(gm[e] & lt);
        tot += __popc(gm[e]);
      }
      int pos = gbase + pre + min(ebase, q);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (k4[e] > T) {
          orow[pos] = base + i0 + e;
          if (srow) srow[pos] = load_elem(a, row, base + i0 + e);
          if (sel_local) sel_local[pos - sel0] = base + i0 + e;
          ++pos;
        }
      }
      gbase += tot;
      continue;
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int i = r * 128 + x * 32 + lane;
      const uint32_t key = keys[i];
      const bool isgt = key > T, iseq = key != 0u && key == T;
      const unsigned gmx = __ballot_sync(kFull, isgt), em = __ballot_sync(kFull, iseq);
      const int gr = gbase + __popc(gmx & lt), er = ebase + __popc(em & lt);
      if (isgt || (iseq && er < q)) {
        const int p = gr + min(er, q);
        orow[p] = base + i;
        if (srow) srow[p] = load_elem(a, row, base + i);
        if (sel_local) sel_local[p - sel0] = base + i;
      }
      gbase += __popc(gmx);
      ebase += __popc(em);
    }
  }
  TK_TRACE(12);
  if (crank == 0) {
    for (int p = (int)k_out + tid; p < a.k; p += kTopkThreads) {
      orow[p] = -1;
      if (srow) srow[p] = -INFINITY;
    }
    if (tid == 0) a.cnt[row] = (int)k_out;
  }
  TK_TRACE(13);
  // keep shared memory alive until every CTA finished its remote reads (their
  // values are consumed): a relaxed arrive -- the default release arrive would
  // first drain this CTA's outstanding global idx stores (ncu: membar stalls)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

}  // namespace sk
