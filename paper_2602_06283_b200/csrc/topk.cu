// Alg. 3 l.244 TopK with forced sink / local window (l.686), and
// the per-shard passes of the exact sequence-shard top-k (DESIGN.md
// "Multi-GPU"; the resolve kernels are in shard_topk.cu).
//
// One thread-block CLUSTER per selection row.  Each CTA owns a contiguous
// slice of the row and keeps it as monotone u32 keys (larger score <=> larger
// key; invalid = 0; forced sink/window keys = 0xFFFFFFFF) in shared memory, or
// for rows longer than one cluster's shared memory (> 16 x 40960 keys) in a
// global-memory workspace.  Selection = keys > T plus the first `quota` keys
// == T in index order, which is exactly "score descending, ties to the smaller
// index" (reading R-15).
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
//
// The same kernel runs the shard passes (op 1-3): the digest (exact counts
// #keys >= edge at bin edges of the same histogram), the window message (keys
// or a histogram of a bracket), and the emit with a resolved threshold.
#include "topk_dev.cuh"

namespace sk {

// ---- op 1: digest -----------------------------------------------------------
// Pairs (edge, #keys >= edge) of this shard's row, all exact:
//   pair 0 = (1, #valid), pair 1 = (0xFFFFFFFF, #forced), pair 2 = (max + 1, #forced),
//   pairs 3.. = (lower edge of the bin holding local rank t, #keys >= that edge)
// for target ranks t spread over (0, 2 ceil(k / shards)] (where the global
// threshold is expected) and over the rest of (0, min(k, #valid)].  Unused
// pairs are (0, 0).
__device__ __forceinline__ void topk_digest(const TopkArgs& a, uint32_t* keys, TopkShared& S, int row, int len,
                                            uint32_t nvalid, uint32_t nforced, uint32_t kmin, uint32_t kmax,
                                            int shards) {
  constexpr unsigned kFull = 0xffffffffu;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int csize = (int)cluster.num_blocks();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int len128 = (len + 127) & ~127;
  if (tid < 8) S.stat[tid] = (tid == 2) ? 0xFFFFFFFFu : 0u;
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
  cluster.sync();
  if (warp == 0) {
    uint32_t v0 = 0, v1 = 0, v2 = 0xFFFFFFFFu, v3 = 0;
    if (lane < csize) {
      const uint4 rs = *reinterpret_cast<const uint4*>(cluster.map_shared_rank(S.stat, lane));
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
  const bool regular = tvalid > tforced;          // some key that is neither invalid nor forced
  const uint32_t span = gmax - gmin;
  const int sh = span < (uint32_t)kBins ? 0 : (32 - __clz(span)) - 11;
  if (regular) {
    for (int i = tid * 4; i < len128; i += kTopkThreads * 4) {
      const uint4 kv = *reinterpret_cast<const uint4*>(keys + i);
      const uint32_t k4[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (k4[e] != 0u && k4[e] != 0xFFFFFFFFu) atomicAdd(&S.hist[(k4[e] - gmin) >> sh], 1u);
    }
  }
  cluster.sync();
  if (crank == 0) {
    uint32_t* out = a.digest + (size_t)row * a.Q * 2;
    // cluster sum of bins 4 tid .. 4 tid + 3, then a suffix scan over the bins
    uint32_t h[4], tot = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t x = 0;
      for (int r = 0; r < csize; ++r) x += cluster.map_shared_rank(S.hist, r)[tid * 4 + e];
      h[e] = x;
      tot += x;
    }
    // suffix over threads: sum of tot of threads > tid
    uint32_t inc = tot;   // inclusive suffix within the warp (lanes >= lane)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_down_sync(kFull, inc, o);
      if (lane + o < 32) inc += y;
    }
    if (lane == 0) S.scan[warp] = (int)inc;
    __syncthreads();
    uint32_t after = 0;   // keys in warps above mine
    for (int w = warp + 1; w < kTopkWarps; ++w) after += (uint32_t)S.scan[w];
    uint32_t suff = after + inc - tot + tforced;   // keys >= bin 4 tid + 4 (regular) + forced
    for (int e = 3; e >= 0; --e) {
      suff += h[e];
      S.gcand[tid * 4 + e] = suff;                 // #keys >= lower edge of bin 4 tid + e
    }
    __syncthreads();
    const uint32_t k_loc = min((uint32_t)a.k, tvalid);
    const int nt = a.Q - 3;
    for (int qi = tid; qi < a.Q; qi += kTopkThreads) {
      uint32_t e = 0, c = 0;
      if (qi == 0) { e = 1u; c = tvalid; }
      else if (qi == 1) { e = 0xFFFFFFFFu; c = tforced; }
      else if (qi == 2) { if (regular) { e = gmax + 1u; c = tforced; } }
      else if (regular && k_loc > tforced) {
        // target rank t in (0, k_loc]: 3/4 of the points on (0, R1], the rest on (R1, k_loc]
        const int t_i = qi - 3;
        const int m1 = max(1, nt * 3 / 4), m2 = nt - m1;
        const uint32_t exp_share = (uint32_t)((a.k + shards - 1) / shards);
        const uint32_t R1 = min(k_loc, 2u * exp_share);
        uint32_t t;
        if (t_i < m1) t = (uint32_t)(((unsigned long long)(t_i + 1) * R1 + m1 - 1) / m1);
        else t = R1 + (uint32_t)(((unsigned long long)(t_i - m1 + 1) * (k_loc - R1) + m2 - 1) / max(m2, 1));
        t = max(t, 1u);
        if (t > tforced) {
          // largest bin b with suff[b] >= t (suff is non-increasing in b)
          int lo = 0, hi = kBins - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (S.gcand[mid] >= t) lo = mid; else hi = mid - 1;
          }
          e = gmin + ((uint32_t)lo << sh);
          c = S.gcand[lo];
        }
      }
      out[2 * qi] = e;
      out[2 * qi + 1] = c;
    }
  }
  cluster.sync();   // keep the histograms alive until CTA 0 is done
}

// ---- op 2: window message ----------------------------------------------------
// For the bracket [lo, hi) of the row's state (hi = 0: 2^32): above = #keys >=
// hi, wc = #keys in the bracket; the message carries the bracket's keys
// (wc <= kMsgCap, any order) or their histogram over kMsgCap bins
// (bin = (key - lo) >> sh, the smallest sh that fits).
__device__ __forceinline__ void topk_window(const TopkArgs& a, uint32_t* keys, TopkShared& S, int row, int len) {
  constexpr unsigned kFull = 0xffffffffu;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int csize = (int)cluster.num_blocks();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int len128 = (len + 127) & ~127;
  const uint32_t* st = a.state + (size_t)row * kStateWords;
  const uint32_t lo = st[0];
  const unsigned long long hi = st[1] == 0u ? (1ull << 32) : (unsigned long long)st[1];
  uint32_t* msg = a.msg + (size_t)row * kMsgWords;
  if (tid < 8) S.stat[tid] = 0u;
  __syncthreads();
  uint32_t above = 0, wc = 0;
  for (int i = tid; i < len128; i += kTopkThreads) {
    const uint32_t key = keys[i];
    above += (unsigned long long)key >= hi ? 1u : 0u;
    const bool in = key != 0u && key >= lo && (unsigned long long)key < hi;
    const unsigned bal = __ballot_sync(kFull, in);
    wc += in;
    if (bal) {
      uint32_t slot = 0;
      if (lane == __ffs(bal) - 1) slot = atomicAdd(&S.stat[4], (uint32_t)__popc(bal));
      slot = __shfl_sync(kFull, slot, __ffs(bal) - 1) + __popc(bal & ((1u << lane) - 1u));
      if (in && slot < (uint32_t)kCandCap) S.cand[slot] = key;
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    above += __shfl_xor_sync(kFull, above, o);
    wc += __shfl_xor_sync(kFull, wc, o);
  }
  if (lane == 0) { atomicAdd(&S.stat[5], above); atomicAdd(&S.stat[6], wc); }
  cluster.sync();
  if (warp == 0) {
    uint32_t ab = 0, w = 0;
    if (lane < csize) {
      const uint32_t* rs = cluster.map_shared_rank(S.stat, lane);
      ab = rs[5];
      w = rs[6];
    }
    uint32_t inc = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    const uint32_t off = __shfl_sync(kFull, inc - w, crank);
    uint32_t abt = ab, wt = w;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      abt += __shfl_xor_sync(kFull, abt, o);
      wt += __shfl_xor_sync(kFull, wt, o);
    }
    if (lane == 0) { S.dec[0] = abt; S.dec[1] = wt; S.dec[2] = off; }
  }
  __syncthreads();
  const uint32_t above_tot = S.dec[0], wc_tot = S.dec[1], off = S.dec[2];
  if (wc_tot <= (uint32_t)kMsgCap) {
    const uint32_t mine = S.stat[6];
    for (uint32_t i = tid; i < mine; i += kTopkThreads) msg[kMsgHdr + off + i] = S.cand[i];
    if (crank == 0 && tid == 0) {
      msg[0] = lo; msg[1] = st[1]; msg[2] = above_tot; msg[3] = wc_tot; msg[4] = 0u; msg[5] = 0u;
    }
  } else {
    const unsigned long long span = hi - lo;   // >= 2
    int sh = 0;
    while (((span - 1ull) >> sh) >= (unsigned long long)kMsgCap) ++sh;
    for (int i = tid; i < kBins; i += kTopkThreads) S.hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < len128; i += kTopkThreads) {
      const uint32_t key = keys[i];
      if (key != 0u && key >= lo && (unsigned long long)key < hi) atomicAdd(&S.hist[(key - lo) >> sh], 1u);
    }
    cluster.sync();
    if (crank == 0) {
      for (int bn = tid; bn < kMsgCap; bn += kTopkThreads) {
        uint32_t x = 0;
        for (int r = 0; r < csize; ++r) x += cluster.map_shared_rank(S.hist, r)[bn];
        msg[kMsgHdr + bn] = x;
      }
      if (tid == 0) {
        msg[0] = lo; msg[1] = st[1]; msg[2] = above_tot; msg[3] = wc_tot; msg[4] = 1u; msg[5] = (uint32_t)sh;
      }
    }
  }
  cluster.sync();   // remote reads of S.stat / S.hist are done
}

template <bool GK>
__global__ void __launch_bounds__(kTopkThreads, 2) topk_cluster_kernel(TopkArgs a, int shards) {
  extern __shared__ __align__(16) uint32_t skeys[];          // [per], per % 128 == 0
  __shared__ TopkShared S;
  TK_TRACE(0);
  // cluster barrier phase 1 of 2: every CTA must be running before topk_core
  // pushes into its shared memory (waited for after the slice load)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: scores of the predecessor
  TK_TRACE(1);
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int csize = (int)cluster.num_blocks();
  const int row = blockIdx.y;
  const int tid = threadIdx.x;
  const int b = row / a.H_sel;
  const int n_glob = a.seq_lens[b];
  const int n = local_len(n_glob, a.index_base, a.N_max);
  uint32_t* keys = GK ? a.gkeys + ((size_t)row * csize + crank) * a.per : skeys;
  if (a.op >= 2) {
    const uint32_t* st = a.state + (size_t)row * kStateWords;
    if (a.op == 2 && st[3] != 0u) {          // already resolved: empty message
      if (crank == 0 && tid < kMsgHdr) {
        uint32_t* msg = a.msg + (size_t)row * kMsgWords;
        msg[tid] = tid == 0 ? st[0] : (tid == 1 ? st[1] : 0u);
      }
      return;
    }
    if (a.op == 3 && st[3] == 0u) {          // unresolved threshold: report, select nothing
      if (crank == 0) {
        for (int p = tid; p < a.k; p += kTopkThreads) a.idx[(size_t)row * a.k + p] = -1;
        if (tid == 0) a.cnt[row] = -1;
      }
      return;
    }
  }
  const int base = crank * a.per;
  int len = n - base;
  len = len < 0 ? 0 : (len > a.per ? a.per : len);
  const int len128 = (len + 127) & ~127;

  // ---- 0. load slice as keys (4 elements per thread per step) ---------------
  uint32_t nvalid = 0, nforced = 0, kmin = 0xFFFFFFFFu, kmax = 0u;
  {
    const float* src = a.scores + (size_t)row * a.N_max + base;   // 128-B aligned
    const long long gb = a.index_base + base;                     // global position of key 0
    const bool forced_free = (a.sink <= 0 || gb >= a.sink) &&
                             (a.window <= 0 || gb + len <= (long long)n_glob - a.window);
    constexpr int U = 8;                                          // float4 loads in flight
    for (int i0 = tid * 4; i0 < len128; i0 += kTopkThreads * 4 * U) {
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
        if (i4 >= len128) break;
        const float vs[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
        uint4 kk;
        uint32_t* kp = &kk.x;
        if (forced_free) {           // no sink / window key in this slice: lean path
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t key = vs[e] == -INFINITY ? 0u : f2key(vs[e]);
            kp[e] = key;
            nvalid += key != 0u;
            kmin = min(kmin, key - 1u);      // invalid (0) wraps to the maximum
            kmax = max(kmax, key);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t key = make_key(vs[e], base + i4 + e, n_glob, a.index_base, a.sink, a.window);
            kp[e] = key;
            nvalid += key != 0u;
            nforced += key == 0xFFFFFFFFu;
            if (key != 0u && key != 0xFFFFFFFFu) { kmin = min(kmin, key - 1u); kmax = max(kmax, key); }
          }
        }
        *reinterpret_cast<uint4*>(keys + i4) = kk;
      }
    }
  }
  kmin += 1u;   // back from key - 1 (no regular key: 0xFFFFFFFF + 1 = 0, fixed below)
  if (kmin == 0u) kmin = 0xFFFFFFFFu;
  if (GK) __syncthreads();   // global slices: written and re-read by other threads
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");   // every CTA of the cluster runs
  switch (a.op) {
    case 0:
      topk_core(a, keys, S, row, n, base, len, nvalid, nforced, kmin, kmax, nullptr, nullptr, nullptr);
      break;
    case 1:
      topk_digest(a, keys, S, row, len, nvalid, nforced, kmin, kmax, shards);
      break;
    case 2:
      __syncthreads();
      topk_window(a, keys, S, row, len);
      break;
    default: {
      __syncthreads();
      const uint32_t* st = a.state + (size_t)row * kStateWords;
      topk_emit(a, keys, S, row, base, len, st[4], st[5], st[7] + st[5], false, nullptr, nullptr, nullptr);
    }
  }
  TK_TRACE(14);
}

#ifdef SK_TRACE
extern "C" int socket_debug_topk_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_topk_trace, (size_t)n * sizeof(unsigned long long));
}
#endif

// Cluster geometry of a row of n_max_row keys: enough CTAs to keep the machine
// busy, slices in shared memory when they fit (<= 40960 keys = 160 KB),
// otherwise 16 CTAs with slices in the global workspace.
constexpr size_t kMaxSlice = 40 * 1024;
static void topk_geometry(int rows, int n_max_row, int& cs, int& per, bool& gk) {
  cs = 1;
  // grow the cluster while a slice is too big for shared memory, or while the grid
  // is below one CTA per SM and the slices stay >= 4096 keys (smaller slices cost
  // more in cluster synchronization than they save; tools/tune_step.py, B = 1-16)
  constexpr int kMinSlice = 4096;
#ifdef SK_TOPK_MIN_CTAS   // experiments only (tools/variant_build.py); not a runtime knob
  const int min_ctas = SK_TOPK_MIN_CTAS;
#else
  const int min_ctas = num_sms();
#endif
  while (cs < 16 && ((size_t)(n_max_row + cs - 1) / cs > kMaxSlice ||
                     (rows * cs < min_ctas && (n_max_row + 2 * cs - 1) / (2 * cs) >= kMinSlice)))
    cs *= 2;
  per = (n_max_row + cs - 1) / cs;
  per = (per + 127) & ~127;
  gk = (size_t)per > kMaxSlice;
  if (per < 128) per = 128;
}

size_t topk_workspace_bytes(const socket_cfg& c) {
  int cs, per;
  bool gk;
  const int rows = c.B * num_sel_rows(c);
  topk_geometry(rows, c.N_max, cs, per, gk);
  return gk ? (size_t)rows * cs * per * sizeof(uint32_t) : 0;
}

static socket_status launch_topk_common(TopkArgs a, int shards, cudaStream_t st, bool pdl,
                                        void* ws, size_t ws_bytes) {
  int cs, per;
  bool gk;
  topk_geometry(a.rows, a.N_max, cs, per, gk);
  a.per = per;
  if (gk) {
    const size_t need = (size_t)a.rows * cs * per * sizeof(uint32_t);
    if (!ws || ws_bytes < need) return fail(SOCKET_EWORKSPACE, "topk: rows > 655360 keys need the workspace");
    a.gkeys = static_cast<uint32_t*>(ws);
  }
  const size_t smem = gk ? 0 : (size_t)per * sizeof(uint32_t);
  auto kfn = gk ? topk_cluster_kernel<true> : topk_cluster_kernel<false>;
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, a, shards);
  if (e != cudaSuccess) return fail(SOCKET_ECUDA, std::string("topk launch: ") + cudaGetErrorString(e));
  return check_launch("topk_cluster_kernel");
}

static TopkArgs topk_args(const socket_cfg& c, const float* scores, const int32_t* seq_lens, int k,
                          int sink, int window) {
  TopkArgs a = {};
  a.scores = scores;
  a.seq_lens = seq_lens;
  a.H_sel = num_sel_rows(c);
  a.rows = c.B * a.H_sel;
  a.N_max = c.N_max;
  a.k = k;
  a.sink = sink;
  a.window = window;
  a.index_base = c.index_base;
  return a;
}

socket_status launch_topk_pdl(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                              int k, int sink, int window, int32_t* idx, int32_t* cnt,
                              float* sel_scores, cudaStream_t st, bool pdl, void* ws, size_t ws_bytes) {
  TopkArgs a = topk_args(c, scores, seq_lens, k, sink, window);
  a.op = 0;
  a.idx = idx;
  a.cnt = cnt;
  a.sel_scores = sel_scores;
  if (a.rows == 0) return SOCKET_OK;
  return launch_topk_common(a, 1, st, pdl, ws, ws_bytes);
}

socket_status launch_topk(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                          int k, int sink, int window, int32_t* idx, int32_t* cnt,
                          float* sel_scores, void* ws, size_t ws_bytes, cudaStream_t st) {
  return launch_topk_pdl(c, scores, seq_lens, k, sink, window, idx, cnt, sel_scores, st, false, ws,
                         ws_bytes);
}

socket_status launch_topk_digest(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                                 int k, int sink, int window, int shards, int Q, uint32_t* digest,
                                 void* ws, size_t ws_bytes, cudaStream_t st) {
  TopkArgs a = topk_args(c, scores, seq_lens, k, sink, window);
  a.op = 1;
  a.Q = Q;
  a.digest = digest;
  if (a.rows == 0) return SOCKET_OK;
  return launch_topk_common(a, shards, st, false, ws, ws_bytes);
}

socket_status launch_topk_window(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                                 int sink, int window, const uint32_t* state, uint32_t* msg,
                                 void* ws, size_t ws_bytes, cudaStream_t st) {
  TopkArgs a = topk_args(c, scores, seq_lens, 1, sink, window);
  a.op = 2;
  a.state = state;
  a.msg = msg;
  if (a.rows == 0) return SOCKET_OK;
  return launch_topk_common(a, 1, st, false, ws, ws_bytes);
}

socket_status launch_topk_emit(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                               int k, int sink, int window, const uint32_t* state, int32_t* idx,
                               int32_t* cnt, float* sel_scores, void* ws, size_t ws_bytes,
                               cudaStream_t st) {
  TopkArgs a = topk_args(c, scores, seq_lens, k, sink, window);
  a.op = 3;
  a.state = state;
  a.idx = idx;
  a.cnt = cnt;
  a.sel_scores = sel_scores;
  if (a.rows == 0) return SOCKET_OK;
  return launch_topk_common(a, 1, st, false, ws, ws_bytes);
}

}  // namespace sk
