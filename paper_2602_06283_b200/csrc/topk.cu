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
#include "topk_dev.cuh"

namespace sk {

__global__ void __launch_bounds__(kTopkThreads, 2) topk_cluster_kernel(TopkArgs a) {
  extern __shared__ __align__(16) uint32_t keys[];          // [per], per % 128 == 0
  __shared__ TopkShared S;
  TK_TRACE(0);
  asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: scores of the predecessor
  TK_TRACE(1);
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int csize = (int)cluster.num_blocks();
  const int row = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int b = row / a.H_sel;
  const int n = a.mode == 0 ? a.seq_lens[b] : a.G * a.k;
  const int base = crank * a.per;
  int len = n - base;
  len = len < 0 ? 0 : (len > a.per ? a.per : len);
  const int len128 = (len + 127) & ~127;
  // warp w owns the rounds [r0, r1) of 128 keys; round r covers keys r*128 + x*32 + lane
  const int nr = len128 >> 7;
  const int rpw = max(1, (nr + kTopkWarps - 1) / kTopkWarps);
  const int r0 = warp * rpw, r1 = min(nr, r0 + rpw);

  // ---- 0. load slice as keys (4 elements per thread per step) ---------------
  uint32_t nvalid = 0, nforced = 0, kmin = 0xFFFFFFFFu, kmax = 0u;
  if (a.mode == 0) {
    const float* src = a.scores + (size_t)row * a.N_max + base;   // 128-B aligned
    const bool forced_free = (a.sink <= 0 || base >= a.sink) && (a.window <= 0 || base + len <= n - a.window);
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
            const uint32_t key = make_key(vs[e], base + i4 + e, n, a.sink, a.window, 0);
            kp[e] = key;
            nvalid += key != 0u;
            nforced += key == 0xFFFFFFFFu;
            if (key != 0u && key != 0xFFFFFFFFu) { kmin = min(kmin, key - 1u); kmax = max(kmax, key); }
          }
        }
        *reinterpret_cast<uint4*>(keys + i4) = kk;
      }
    }
  } else {
    for (int i = tid; i < len128; i += kTopkThreads) {
      uint32_t key = 0;
      if (i < len) key = make_key(load_elem(a, row, base + i), base + i, n, 0, 0, 1);
      keys[i] = key;
      nvalid += key != 0u;
      if (key != 0u) { kmin = min(kmin, key - 1u); kmax = max(kmax, key); }
    }
  }
  kmin += 1u;   // back from key - 1 (no regular key: 0xFFFFFFFF + 1 = 0, fixed below)
  if (kmin == 0u) kmin = 0xFFFFFFFFu;
  kmin += 0u;
  topk_core(a, keys, S, row, n, base, len, nvalid, nforced, kmin, kmax, nullptr, nullptr, nullptr);
  TK_TRACE(14);
}

#ifdef SK_TRACE
extern "C" int socket_debug_topk_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_topk_trace, (size_t)n * sizeof(unsigned long long));
}
#endif

static socket_status launch_topk_common(TopkArgs a, int n_max_row, cudaStream_t st, bool pdl = false) {
  // cluster size: enough CTAs to keep the machine busy, slices fit in smem
  const size_t kMaxSlice = 40 * 1024;   // keys per CTA (160 KB)
  int cs = 1;
  const char* tune = getenv("SOCKET_TOPK_MIN_CTAS");   // tuning experiments only
  const int min_ctas = tune ? atoi(tune) : kNumSMs;
  // grow the cluster while a slice is too big for shared memory, or while the grid
  // is below min_ctas and the slices stay >= 4096 keys (smaller slices cost more
  // in cluster synchronization than they save; tools/tune_step.py, B = 1-16)
  constexpr int kMinSlice = 4096;
  while (cs < 16 && ((size_t)(n_max_row + cs - 1) / cs > kMaxSlice ||
                     (a.rows * cs < min_ctas && (n_max_row + 2 * cs - 1) / (2 * cs) >= kMinSlice)))
    cs *= 2;
  int per = (n_max_row + cs - 1) / cs;
  per = (per + 127) & ~127;
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
