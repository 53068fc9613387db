// Alg. 3 l.244 TopK with forced sink / local window (l.686), and
// the exact resolve step of sequence sharding.
//
// One thread-block CLUSTER per selection row.  Each CTA of the cluster owns a
// contiguous slice of the row and keeps it in shared memory as monotone u32
// keys (larger score <=> larger key; invalid = 0; forced = 0xFFFFFFFF).  An
// MSB-first radix select with 8-bit digits finds the k_eff-th largest key T:
// every pass builds a local 256-bin histogram (match_any-aggregated shared
// atomics), the cluster sums the CTAs' histograms through distributed shared
// memory (DSMEM) and every CTA takes the same digit decision.  No sort.
// Selection = keys > T plus the first (quota) keys == T in index order, which
// is exactly "score descending, ties to the smaller index" (reading R-15).
// A stable ballot compaction writes the selected indices in ascending order.
#include <cooperative_groups.h>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace sk {

constexpr int kTopkThreads = 512;
constexpr int kTopkWarps = kTopkThreads / 32;

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

// exclusive scan over the 16 warps of one value per warp; returns prefix, total via ref
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

__global__ void __launch_bounds__(kTopkThreads, 1) topk_cluster_kernel(TopkArgs a) {
  extern __shared__ __align__(16) uint32_t keys[];          // [per]
  __shared__ uint32_t hist[2][256];
  __shared__ int sh_scan[kTopkWarps];
  __shared__ int sh_cnt[4];                                  // valid, gt, eq, emit
  __shared__ uint32_t sh_dec[2];                             // digit, k_rem

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

  // ---- load slice as keys -------------------------------------------------
  int nvalid = 0;
  for (int i = tid; i < len32; i += kTopkThreads) {
    uint32_t key = 0;
    if (i < len) {
      const int e = base + i;
      const float s = load_elem(a, row, e);
      if (s != -INFINITY) {
        key = f2key(s);
        if (a.mode == 0 && (e < a.sink || e >= n - a.window)) key = 0xFFFFFFFFu;
      }
    }
    keys[i] = key;
    nvalid += key != 0;
  }
  for (int i = tid; i < 512; i += kTopkThreads) (&hist[0][0])[i] = 0;
  if (tid < 4) sh_cnt[tid] = 0;
  __syncthreads();
  {
    int v = nvalid;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && v) atomicAdd(&sh_cnt[0], v);
  }
  cluster.sync();
  int total_valid = 0;
  for (int c = 0; c < csize; ++c) total_valid += *cluster.map_shared_rank(&sh_cnt[0], c);
  const int k_eff = a.k < total_valid ? a.k : total_valid;

  // ---- radix select --------------------------------------------------------
  uint32_t T = 0, quota = 0;       // select keys > T, plus `quota` keys == T
  if (k_eff < total_valid) {
    uint32_t prefix = 0, k_rem = (uint32_t)k_eff;
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      const int buf = pass & 1;
      const uint32_t hmask = pass == 0 ? 0u : (0xFFFFFFFFu << (shift + 8));
      for (int i = tid; i < len32; i += kTopkThreads) {
        const uint32_t key = keys[i];
        const bool m = (key & hmask) == (prefix & hmask) && i < len;
        const uint32_t bin = m ? ((key >> shift) & 255u) : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, bin);
        if (m && lane == __ffs(peers) - 1) atomicAdd(&hist[buf][bin], (uint32_t)__popc(peers));
      }
      cluster.sync();
      // warp 0: sum the cluster's histograms and pick the digit
      if (warp == 0) {
        uint32_t c8[8];
        uint32_t tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int bin = 255 - (lane * 8 + q);             // lane 0 holds the top bins
          uint32_t s = 0;
          for (int c = 0; c < csize; ++c) s += *cluster.map_shared_rank(&hist[buf][bin], c);
          c8[q] = s;
          tot += s;
        }
        // inclusive scan of lane totals (descending-bin order)
        uint32_t inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        const uint32_t excl = inc - tot;
        const bool hit = excl < k_rem && inc >= k_rem;
        const uint32_t hb = __ballot_sync(0xffffffffu, hit);
        const int src = __ffs(hb) - 1;
        if (lane == src) {
          uint32_t run = excl;
          for (int q = 0; q < 8; ++q) {
            if (run + c8[q] >= k_rem) {
              sh_dec[0] = (uint32_t)(255 - (lane * 8 + q));
              sh_dec[1] = k_rem - run;
              break;
            }
            run += c8[q];
          }
        }
      }
      // clear the other buffer (its last readers finished before this pass's sync)
      for (int i = tid; i < 256; i += kTopkThreads) hist[buf ^ 1][i] = 0;
      __syncthreads();
      prefix |= sh_dec[0] << shift;
      k_rem = sh_dec[1];
    }
    T = prefix;
    quota = k_rem;
  }
  // ---- stable compaction -----------------------------------------------------
  // warp w scans a contiguous block of the slice in 32-key groups
  const int groups = len32 >> 5;
  const int gpw = (groups + kTopkWarps - 1) / kTopkWarps;
  const int g0 = warp * gpw;
  const int g1 = min(groups, g0 + gpw);
  int gt_w = 0, eq_w = 0;
  for (int gi = g0; gi < g1; ++gi) {
    const int i = gi * 32 + lane;
    const uint32_t key = keys[i];
    const bool valid = i < len && key != 0;
    gt_w += __popc(__ballot_sync(0xffffffffu, valid && key > T));
    eq_w += __popc(__ballot_sync(0xffffffffu, valid && key == T));
  }
  int gt_tot, eq_tot;
  const int gt_pre = block_excl_scan_warps(gt_w, sh_scan, warp, lane, gt_tot);
  const int eq_pre = block_excl_scan_warps(eq_w, sh_scan, warp, lane, eq_tot);
  if (tid == 0) { sh_cnt[1] = gt_tot; sh_cnt[2] = eq_tot; }
  cluster.sync();
  int eq_before = 0, gt_before = 0;
  for (int c = 0; c < crank; ++c) {
    gt_before += *cluster.map_shared_rank(&sh_cnt[1], c);
    eq_before += *cluster.map_shared_rank(&sh_cnt[2], c);
  }
  // emission: mode 0 emits every selected key; mode 1 only keys of shard `rank`
  const int emit_lo = a.mode == 0 ? 0 : a.rank * a.k;
  const int emit_hi = a.mode == 0 ? n : (a.rank + 1) * a.k;
  auto take = [&](uint32_t key, int eq_rank_global) -> bool {
    return key > T || (key == T && (uint32_t)eq_rank_global < quota);
  };
  // pass 1: emitted count per warp
  int em_w = 0;
  {
    int eq_run = eq_before + eq_pre;
    for (int gi = g0; gi < g1; ++gi) {
      const int i = gi * 32 + lane;
      const uint32_t key = keys[i];
      const bool valid = i < len && key != 0;
      const bool isEq = valid && key == T;
      const unsigned eb = __ballot_sync(0xffffffffu, isEq);
      const int my_eq = eq_run + __popc(eb & ((1u << lane) - 1u));
      const int e = base + i;
      const bool sel = valid && take(key, my_eq) && e >= emit_lo && e < emit_hi;
      em_w += __popc(__ballot_sync(0xffffffffu, sel));
      eq_run += __popc(eb);
    }
  }
  int em_tot;
  const int em_pre = block_excl_scan_warps(em_w, sh_scan, warp, lane, em_tot);
  if (tid == 0) sh_cnt[3] = em_tot;
  cluster.sync();
  int em_before = 0, em_all = 0;
  for (int c = 0; c < csize; ++c) {
    const int x = *cluster.map_shared_rank(&sh_cnt[3], c);
    em_all += x;
    em_before += c < crank ? x : 0;
  }
  // pass 2: write
  {
    int eq_run = eq_before + eq_pre;
    int pos = em_before + em_pre;
    int32_t* orow = a.idx + (size_t)row * a.k;
    float* srow = a.sel_scores ? a.sel_scores + (size_t)row * a.k : nullptr;
    for (int gi = g0; gi < g1; ++gi) {
      const int i = gi * 32 + lane;
      const uint32_t key = keys[i];
      const bool valid = i < len && key != 0;
      const bool isEq = valid && key == T;
      const unsigned eb = __ballot_sync(0xffffffffu, isEq);
      const int my_eq = eq_run + __popc(eb & ((1u << lane) - 1u));
      const int e = base + i;
      const bool sel = valid && take(key, my_eq) && e >= emit_lo && e < emit_hi;
      const unsigned sb = __ballot_sync(0xffffffffu, sel);
      if (sel) {
        const int p = pos + __popc(sb & ((1u << lane) - 1u));
        if (a.mode == 0) {
          orow[p] = e;
          if (srow) srow[p] = load_elem(a, row, e);
        } else {
          orow[p] = a.cand_idx[((size_t)a.rank * a.rows + row) * a.k + (e - emit_lo)];
        }
      }
      pos += __popc(sb);
      eq_run += __popc(eb);
    }
  }
  // tail fill and count (CTA 0)
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

static socket_status launch_topk_common(TopkArgs a, int n_max_row, cudaStream_t st) {
  // cluster size: enough CTAs to keep the machine busy, slices fit in smem
  const size_t kMaxSlice = 48 * 1024;   // keys per CTA (192 KB)
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
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, a);
  if (e != cudaSuccess) return fail(SOCKET_ECUDA, std::string("topk launch: ") + cudaGetErrorString(e));
  return check_launch("topk_cluster_kernel");
}

socket_status launch_topk(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                          int k, int sink, int window, int32_t* idx, int32_t* cnt,
                          float* sel_scores, cudaStream_t st) {
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
  return launch_topk_common(a, c.N_max, st);
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
