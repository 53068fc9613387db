// Alg. 3 l.244 TopK with forced sink / local window (l.686), and
// the exact resolve step of sequence sharding.
//
// One thread-block CLUSTER per selection row.  Each CTA owns a contiguous
// slice of the row and keeps it in shared memory as monotone u32 keys (larger
// score <=> larger key; invalid = 0; forced sink/window keys = 0xFFFFFFFF).
// Selection = keys > T plus the first `quota` keys == T in index order, which
// is exactly "score descending, ties to the smaller index" (reading R-15).
//
// Finding T (the k_eff-th largest key), no sort:
//   1. cluster-reduce (#valid, #forced, min and max regular key) through
//      distributed shared memory (DSMEM);
//   2. one 2048-bin histogram over the row's actual key range [min, max]
//      (bin = (key - min) >> shift, the smallest shift that fits: monotone,
//      exact integer arithmetic), summed across the cluster through DSMEM; the bin holding
//      the target rank is found by a suffix scan;
//   3. the keys of that bin (typically tens) are gathered from every CTA and
//      T is resolved exactly by a local radix select over them.
//   If the bin is too full to gather (massive exact ties, degenerate ranges),
//   a 4-pass MSB radix select over the whole cluster (8-bit digits) is used.
// A stable ballot compaction then writes the selected indices in ascending order.
#include <cooperative_groups.h>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace sk {

constexpr int kTopkThreads = 512;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kBins = 2048;
constexpr int kCandCap = 2048;

struct TopkArgs {
  // mode 0: scores [rows][N_max], n = seq_lens[b]
  // mode 1: resolve; candidates cand_scores [G][rows][k]; n = G*k
  int mode;
  const float* scores;
  const int32_t* seq_lens;
  const float* cand_scores;
  const int32_t* cand_idx;
  int rows, H_sel, N_max, k, sink, window, G, rank;
  int per;                 // slice length per CTA (multiple of 32)
  int32_t* idx;
  int32_t* cnt;
  float* sel_scores;
};

__device__ __forceinline__ float load_elem(const TopkArgs& a, int row, int e) {
  if (a.mode == 0) return a.scores[(size_t)row * a.N_max + e];
  const int s = e / a.k, i = e % a.k;
  return a.cand_scores[((size_t)s * a.rows + row) * a.k + i];
}

__device__ __forceinline__ uint32_t make_key(float s, int e, int n, int sink, int window, int mode) {
  if (s == -INFINITY) return 0u;
  if (mode == 0 && (e < sink || e >= n - window)) return 0xFFFFFFFFu;
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

struct TopkShared {
  uint32_t hist[kBins];          // local histogram (also radix fallback buffers)
  uint32_t ghist[kBins];         // cluster-summed histogram
  uint32_t cand[kCandCap];       // local candidates
  uint32_t gcand[kCandCap];      // gathered candidates
  uint32_t rhist[256];           // local radix histogram for candidate resolve
  int scan[kTopkWarps];
  int scan2[kTopkWarps];
  uint32_t stat[8];              // nvalid, nforced, kmin, kmax, ncand, gt, eq, emit
  uint32_t dec[4];
};

// Local exact select over a small candidate array: the `need`-th largest key
// (1-based) and how many candidates are strictly greater.
__device__ void local_select(const uint32_t* c, int C, uint32_t need, TopkShared& S, int tid,
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

__global__ void __launch_bounds__(kTopkThreads, 2) topk_cluster_kernel(TopkArgs a) {
  extern __shared__ __align__(16) uint32_t keys[];          // [per]
  __shared__ TopkShared S;

  asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: scores of the predecessor
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int csize = (int)cluster.num_blocks();
  const int row = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = row / a.H_sel;
  const int n = a.mode == 0 ? a.seq_lens[b] : a.G * a.k;
  const int base = crank * a.per;
  int len = n - base;
  len = len < 0 ? 0 : (len > a.per ? a.per : len);
  const int len32 = (len + 31) & ~31;

  // ---- 0. load slice as keys (4 elements per thread per step) ---------------
  uint32_t nvalid = 0, nforced = 0, kmin = 0xFFFFFFFFu, kmax = 0u;
  if (a.mode == 0) {
    const float* src = a.scores + (size_t)row * a.N_max + base;   // 128-B aligned
    constexpr int U = 4;                                          // float4 loads in flight
    for (int i0 = tid * 4; i0 < len32; i0 += kTopkThreads * 4 * U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i4 = i0 + u * kTopkThreads * 4;
        v[u] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        if (i4 + 3 < len) v[u] = *reinterpret_cast<const float4*>(src + i4);
        else if (i4 < len) {
          v[u].x = src[i4];
          if (i4 + 1 < len) v[u].y = src[i4 + 1];
          if (i4 + 2 < len) v[u].z = src[i4 + 2];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i4 = i0 + u * kTopkThreads * 4;
        if (i4 >= len32) break;
        const float vs[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
        uint4 kk;
        uint32_t* kp = &kk.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t key = make_key(vs[e], base + i4 + e, n, a.sink, a.window, 0);
          kp[e] = key;
          nvalid += key != 0u;
          nforced += key == 0xFFFFFFFFu;
          if (key != 0u && key != 0xFFFFFFFFu) { kmin = min(kmin, key); kmax = max(kmax, key); }
        }
        *reinterpret_cast<uint4*>(keys + i4) = kk;
      }
    }
  } else {
    for (int i = tid; i < len32; i += kTopkThreads) {
      uint32_t key = 0;
      if (i < len) key = make_key(load_elem(a, row, base + i), base + i, n, 0, 0, 1);
      keys[i] = key;
      nvalid += key != 0u;
      if (key != 0u) { kmin = min(kmin, key); kmax = max(kmax, key); }
    }
  }
  if (tid < 8) S.stat[tid] = (tid == 2) ? 0xFFFFFFFFu : 0u;   // kmin starts at +max
  for (int i = tid; i < kBins; i += kTopkThreads) S.hist[i] = 0;
  __syncthreads();
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    nvalid += __shfl_xor_sync(0xffffffffu, nvalid, o);
    nforced += __shfl_xor_sync(0xffffffffu, nforced, o);
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if (lane == 0) {
    atomicAdd(&S.stat[0], nvalid);
    atomicAdd(&S.stat[1], nforced);
    atomicMin(&S.stat[2], kmin);
    atomicMax(&S.stat[3], kmax);
  }
  cluster.sync();
  uint32_t tvalid = 0, tforced = 0, gmin = 0xFFFFFFFFu, gmax = 0;
  for (int c = 0; c < csize; ++c) {
    const uint32_t* rs = cluster.map_shared_rank(S.stat, c);
    tvalid += rs[0];
    tforced += rs[1];
    gmin = min(gmin, rs[2]);
    gmax = max(gmax, rs[3]);
  }
  const uint32_t k_eff = min((uint32_t)a.k, tvalid);

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
  bool fallback = false;
  if (!done) {
    // 2. adaptive histogram over [gmin, gmax]
    // bin = (key - gmin) >> sh with the smallest sh that maps [gmin, gmax] into
    // kBins bins: monotone and exact (no division)
    const uint32_t span = gmax - gmin;
    const int sh = span < (uint32_t)kBins ? 0 : (32 - __clz(span)) - 11;
    for (int i = tid; i < len32; i += kTopkThreads) {
      const uint32_t key = keys[i];
      if (key != 0u && key != 0xFFFFFFFFu) {
        atomicAdd(&S.hist[(key - gmin) >> sh], 1u);
      }
    }
    cluster.sync();
    for (int i = tid; i < kBins; i += kTopkThreads) {
      uint32_t s = 0;
      for (int c = 0; c < csize; ++c) s += *cluster.map_shared_rank(&S.hist[i], c);
      S.ghist[i] = s;
    }
    __syncthreads();
    // suffix scan over bins (descending): each warp owns 128 bins, lane 4 of them
    {
      const int b0 = kBins - 1 - (warp * 128 + lane * 4);
      uint32_t c4[4], tot = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) { c4[q] = S.ghist[b0 - q]; tot += c4[q]; }
      uint32_t inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) S.scan[warp] = (int)inc;
      __syncthreads();
      uint32_t wpre = 0;
      for (int w = 0; w < warp; ++w) wpre += (uint32_t)S.scan[w];
      const uint32_t excl = wpre + inc - tot;
      if (excl < need && excl + tot >= need) {
        uint32_t run = excl;
        for (int q = 0; q < 4; ++q) {
          if (run + c4[q] >= need) { S.dec[0] = (uint32_t)(b0 - q); S.dec[1] = need - run; S.dec[2] = c4[q]; break; }
          run += c4[q];
        }
      }
      __syncthreads();
    }
    const uint32_t bstar = S.dec[0], need2 = S.dec[1], C = S.dec[2];
    if (C <= (uint32_t)kCandCap) {
      // 3. gather the bin's keys from every CTA, resolve T exactly
      for (int i = tid; i < len32; i += kTopkThreads) {
        const uint32_t key = keys[i];
        if (key != 0u && key != 0xFFFFFFFFu && ((key - gmin) >> sh) == bstar) {
          const uint32_t pos = atomicAdd(&S.stat[4], 1u);
          S.cand[pos] = key;
        }
      }
      cluster.sync();
      uint32_t off = 0;
      for (int c = 0; c < csize; ++c) {
        const uint32_t nc = *cluster.map_shared_rank(&S.stat[4], c);
        const uint32_t* rc = cluster.map_shared_rank(S.cand, c);
        for (uint32_t i = tid; i < nc; i += kTopkThreads) S.gcand[off + i] = rc[i];
        off += nc;
      }
      __syncthreads();
      uint32_t above;
      local_select(S.gcand, (int)C, need2, S, tid, warp, lane, T, above);
      quota = need2 - above;
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
        const uint32_t peers = __match_any_sync(0xffffffffu, bin);
        if (m && lane == __ffs(peers) - 1) atomicAdd(&hb[bin], (uint32_t)__popc(peers));
      }
      cluster.sync();
      if (warp == 0) {
        uint32_t c8[8], tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int bin = 255 - (lane * 8 + q);
          uint32_t s = 0;
          for (int c = 0; c < csize; ++c) s += *cluster.map_shared_rank(&hb[bin], c);
          c8[q] = s;
          tot += s;
        }
        uint32_t inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        const uint32_t excl = inc - tot;
        const unsigned hbits = __ballot_sync(0xffffffffu, excl < k_rem && inc >= k_rem);
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
  // Output position of a selected key = gt_rank + min(eq_rank, quota), where
  // gt_rank / eq_rank count keys > T / == T at smaller indices (row-global).
  int em_all = 0;
  if (a.mode == 0) {
    // warp w owns a contiguous block of 4-key chunks; in each round the warp's
    // lanes read 32 consecutive chunks (conflict-free 16-byte loads), so index
    // order = (round, lane, element)
    const int nchunk = len32 >> 2;
    const int cpw = ((nchunk + kTopkWarps - 1) / kTopkWarps + 31) & ~31;   // chunks per warp
    const int c0 = warp * cpw, c1 = min(nchunk, c0 + cpw);
    int gt_w = 0, eq_w = 0;
    for (int cc = c0 + lane; cc - lane < c1; cc += 32) {
      uint4 kv = make_uint4(0, 0, 0, 0);
      if (cc < c1) kv = *reinterpret_cast<const uint4*>(keys + cc * 4);
      const uint32_t* kp = &kv.x;
      int g = 0, e = 0;
#pragma unroll
      for (int x = 0; x < 4; ++x) { g += kp[x] != 0u && kp[x] > T; e += kp[x] != 0u && kp[x] == T; }
      gt_w += g;
      eq_w += e;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      gt_w += __shfl_xor_sync(0xffffffffu, gt_w, o);
      eq_w += __shfl_xor_sync(0xffffffffu, eq_w, o);
    }
    __syncthreads();
    if (lane == 0) { S.scan[warp] = gt_w; S.scan2[warp] = eq_w; }
    __syncthreads();
    int gw = 0, ew = 0, gtot = 0, etot = 0;
#pragma unroll
    for (int w = 0; w < kTopkWarps; ++w) {
      const int xg = S.scan[w], xe = S.scan2[w];
      gw += w < warp ? xg : 0; ew += w < warp ? xe : 0;
      gtot += xg; etot += xe;
    }
    if (tid == 0) { S.stat[5] = (uint32_t)gtot; S.stat[6] = (uint32_t)etot; }
    cluster.sync();
    int gt_before = 0, eq_before = 0;
    for (int c = 0; c < crank; ++c) {
      const uint32_t* rs = cluster.map_shared_rank(S.stat, c);
      gt_before += (int)rs[5];
      eq_before += (int)rs[6];
    }
    em_all = (int)k_eff;
    int gbase = gt_before + gw, ebase = eq_before + ew;   // ranks at the start of the round
    int32_t* orow = a.idx + (size_t)row * a.k;
    float* srow = a.sel_scores ? a.sel_scores + (size_t)row * a.k : nullptr;
    for (int cc = c0 + lane; cc - lane < c1; cc += 32) {
      uint4 kv = make_uint4(0, 0, 0, 0);
      if (cc < c1) kv = *reinterpret_cast<const uint4*>(keys + cc * 4);
      const uint32_t* kp = &kv.x;
      int g = 0, e = 0;
#pragma unroll
      for (int x = 0; x < 4; ++x) { g += kp[x] != 0u && kp[x] > T; e += kp[x] != 0u && kp[x] == T; }
      int gi = g, ei = e;                          // inclusive scans over lanes
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int yg = __shfl_up_sync(0xffffffffu, gi, o), ye = __shfl_up_sync(0xffffffffu, ei, o);
        if (lane >= o) { gi += yg; ei += ye; }
      }
      int gr = gbase + gi - g, er = ebase + ei - e;   // exclusive ranks of this lane's first key
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const uint32_t key = kp[x];
        if (key == 0u) continue;
        const int j = base + cc * 4 + x;
        if (key > T) {
          const int pos = gr + min(er, (int)quota);
          orow[pos] = j;
          if (srow) srow[pos] = load_elem(a, row, j);
          ++gr;
        } else if (key == T) {
          if (er < (int)quota) {
            orow[gr + er] = j;
            if (srow) srow[gr + er] = load_elem(a, row, j);
          }
          ++er;
        }
      }
      gbase += __shfl_sync(0xffffffffu, gi, 31);
      ebase += __shfl_sync(0xffffffffu, ei, 31);
    }
  } else {
    const int groups = len32 >> 5;
    const int gpw = (groups + kTopkWarps - 1) / kTopkWarps;
    const int g0 = warp * gpw;
    const int g1 = min(groups, g0 + gpw);
    int eq_w = 0;
    for (int gi = g0; gi < g1; ++gi) {
      const uint32_t key = keys[gi * 32 + lane];
      eq_w += __popc(__ballot_sync(0xffffffffu, key != 0u && key == T));
    }
    int eq_tot;
    const int eq_pre = block_excl_scan_warps(eq_w, S.scan, warp, lane, eq_tot);
    if (tid == 0) S.stat[6] = (uint32_t)eq_tot;
    cluster.sync();
    int eq_before = 0;
    for (int c = 0; c < crank; ++c) eq_before += (int)*cluster.map_shared_rank(&S.stat[6], c);
    const int emit_lo = a.rank * a.k;
    const int emit_hi = (a.rank + 1) * a.k;
    int em_w = 0;
    {
      int eq_run = eq_before + eq_pre;
      for (int gi = g0; gi < g1; ++gi) {
        const int i = gi * 32 + lane;
        const uint32_t key = keys[i];
        const bool valid = key != 0u;
        const unsigned eb = __ballot_sync(0xffffffffu, valid && key == T);
        const int my_eq = eq_run + __popc(eb & ((1u << lane) - 1u));
        const int e = base + i;
        const bool sel = valid && (key > T || (key == T && (uint32_t)my_eq < quota)) &&
                         e >= emit_lo && e < emit_hi;
        em_w += __popc(__ballot_sync(0xffffffffu, sel));
        eq_run += __popc(eb);
      }
    }
    int em_tot;
    const int em_pre = block_excl_scan_warps(em_w, S.scan, warp, lane, em_tot);
    if (tid == 0) S.stat[7] = (uint32_t)em_tot;
    cluster.sync();
    int em_before = 0;
    for (int c = 0; c < csize; ++c) {
      const int x = (int)*cluster.map_shared_rank(&S.stat[7], c);
      em_all += x;
      em_before += c < crank ? x : 0;
    }
    int eq_run = eq_before + eq_pre;
    int pos = em_before + em_pre;
    int32_t* orow = a.idx + (size_t)row * a.k;
    for (int gi = g0; gi < g1; ++gi) {
      const int i = gi * 32 + lane;
      const uint32_t key = keys[i];
      const bool valid = key != 0u;
      const unsigned eb = __ballot_sync(0xffffffffu, valid && key == T);
      const int my_eq = eq_run + __popc(eb & ((1u << lane) - 1u));
      const int e = base + i;
      const bool sel = valid && (key > T || (key == T && (uint32_t)my_eq < quota)) &&
                       e >= emit_lo && e < emit_hi;
      const unsigned sb = __ballot_sync(0xffffffffu, sel);
      if (sel) orow[pos + __popc(sb & ((1u << lane) - 1u))] =
          a.cand_idx[((size_t)a.rank * a.rows + row) * a.k + (e - emit_lo)];
      pos += __popc(sb);
      eq_run += __popc(eb);
    }
  }
  if (crank == 0) {
    int32_t* orow = a.idx + (size_t)row * a.k;
    for (int p = em_all + tid; p < a.k; p += kTopkThreads) {
      orow[p] = -1;
      if (a.sel_scores) a.sel_scores[(size_t)row * a.k + p] = -INFINITY;
    }
    if (tid == 0) a.cnt[row] = em_all;
  }
  cluster.sync();   // keep shared memory alive until every CTA finished remote reads
}

static socket_status launch_topk_common(TopkArgs a, int n_max_row, cudaStream_t st, bool pdl = false) {
  // cluster size: enough CTAs to keep the machine busy, slices fit in smem
  const size_t kMaxSlice = 40 * 1024;   // keys per CTA (160 KB)
  int cs = 1;
  while (cs < 16 && ((size_t)(n_max_row + cs - 1) / cs > kMaxSlice || a.rows * cs < kNumSMs))
    cs *= 2;
  int per = (n_max_row + cs - 1) / cs;
  per = (per + 31) & ~31;
  if ((size_t)per > kMaxSlice) return fail(SOCKET_EUNSUPPORTED, "topk: row too long for one cluster");
  a.per = per;
  const size_t smem = (size_t)per * sizeof(uint32_t);
  auto kfn = topk_cluster_kernel;
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cs > 8) cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, a.rows, 1);
  cfg.blockDim = dim3(kTopkThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, a);
  if (e != cudaSuccess) return fail(SOCKET_ECUDA, std::string("topk launch: ") + cudaGetErrorString(e));
  return check_launch("topk_cluster_kernel");
}

socket_status launch_topk_pdl(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                              int k, int sink, int window, int32_t* idx, int32_t* cnt,
                              float* sel_scores, cudaStream_t st, bool pdl) {
  TopkArgs a = {};
  a.mode = 0;
  a.scores = scores;
  a.seq_lens = seq_lens;
  a.H_sel = num_sel_rows(c);
  a.rows = c.B * a.H_sel;
  a.N_max = c.N_max;
  a.k = k;
  a.sink = sink;
  a.window = window;
  a.idx = idx;
  a.cnt = cnt;
  a.sel_scores = sel_scores;
  if (a.rows == 0) return SOCKET_OK;
  return launch_topk_common(a, c.N_max, st, pdl);
}

socket_status launch_topk(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                          int k, int sink, int window, int32_t* idx, int32_t* cnt,
                          float* sel_scores, cudaStream_t st) {
  return launch_topk_pdl(c, scores, seq_lens, k, sink, window, idx, cnt, sel_scores, st, false);
}

socket_status launch_topk_resolve(const socket_cfg& c, const float* cand_scores,
                                  const int32_t* cand_idx, int G, int rank, int k, int32_t* idx,
                                  int32_t* cnt, cudaStream_t st) {
  TopkArgs a = {};
  a.mode = 1;
  a.cand_scores = cand_scores;
  a.cand_idx = cand_idx;
  a.H_sel = num_sel_rows(c);
  a.rows = c.B * a.H_sel;
  a.N_max = c.N_max;
  a.k = k;
  a.G = G;
  a.rank = rank;
  a.idx = idx;
  a.cnt = cnt;
  if (a.rows == 0) return SOCKET_OK;
  return launch_topk_common(a, G * k, st);
}

}  // namespace sk
