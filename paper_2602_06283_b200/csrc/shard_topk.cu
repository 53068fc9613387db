// Exact global top-k over sequence shards (SURVEY
// 8(e) v2): the per-row bracket from the all-gathered digests, and the resolve
// of a bracket from the all-gathered window messages.  Both run identically on
// every rank (same inputs, deterministic), one CTA per selection row.
//
// Keys are the monotone u32 images of the scores (topk_dev.cuh: invalid 0,
// forced 0xFFFFFFFF).  T = the k_eff-th largest key over all shards; the
// selection is every key > T plus the first (k_eff - #keys > T) keys == T in
// global index order = shards in rank order, then local index (reading R-15;
// shard s owns global positions [s N_s, (s+1) N_s)).
//
// Bracket (from digests of exact pairs (e, c_s(e)), c_s(x) = #keys >= x in shard s):
//   lower_s(x) = max{c : (e, c) in D_s, e >= x}  <=  c_s(x)  <=  upper_s(x) = min{c : e <= x}
//   T_lo = max{x in E : sum_s lower_s(x) >= k_eff}   =>  T >= T_lo
//   T_hi = min{x in E : sum_s upper_s(x) <= k_eff - 1} =>  T <  T_hi  (none: 2^32)
// Resolve (from window messages of the bracket [lo, hi), above_s = c_s(hi)):
//   need = k_eff - sum_s above_s; T = the need-th largest bracket key.  If every
//   shard sent its bracket keys, T and the per-shard counts #> T, #== T are
//   exact.  Otherwise the summed histograms narrow the bracket to the bin of
//   rank `need` (exact if the bin is one key value wide, else one more round:
//   2048 bins take any 32-bit bracket to a single value in 3 rounds).
#include "topk_dev.cuh"

namespace sk {

constexpr int kShardThreads = 512;

__global__ void __launch_bounds__(kShardThreads) topk_bracket_kernel(const uint32_t* __restrict__ dig, int G,
                                                                     int rows, int Q, int k,
                                                                     uint32_t* __restrict__ state) {
  extern __shared__ uint32_t ec[];           // [G*Q] edges, then [G*Q] counts
  __shared__ unsigned long long s_lo, s_hi;
  __shared__ uint32_t s_valid;
  const int row = blockIdx.x, tid = threadIdx.x;
  const int n = G * Q;
  uint32_t* E = ec;
  uint32_t* C = ec + n;
  if (tid == 0) { s_lo = 0ull; s_hi = 1ull << 32; s_valid = 0u; }
  __syncthreads();
  for (int i = tid; i < n; i += kShardThreads) {
    const int s = i / Q, j = i % Q;
    const uint32_t* p = dig + (((size_t)s * rows + row) * Q + j) * 2;
    E[i] = p[0];
    C[i] = p[1];
    if (j == 0) atomicAdd(&s_valid, p[1]);   // pair 0 = (1, #valid)
  }
  __syncthreads();
  const uint32_t k_eff = min((uint32_t)k, s_valid);
  uint32_t* st = state + (size_t)row * kStateWords;
  if (k_eff == 0u) {
    if (tid < kStateWords) st[tid] = tid == 0 ? 1u : (tid == 3 ? 1u : (tid == 4 ? 0xFFFFFFFFu : 0u));
    return;
  }
  for (int i = tid; i < n; i += kShardThreads) {
    const uint32_t x = E[i];
    if (x == 0u) continue;                  // unused pair
    unsigned long long Ls = 0, Us = 0;
    for (int s = 0; s < G; ++s) {
      uint32_t lo_c = 0u, up_c = 0xFFFFFFFFu;
      for (int j = 0; j < Q; ++j) {
        const uint32_t e = E[s * Q + j], c = C[s * Q + j];
        if (e == 0u) continue;
        if (e >= x) lo_c = max(lo_c, c);
        if (e <= x) up_c = min(up_c, c);
      }
      Ls += lo_c;
      Us += up_c;                           // pair (1, #valid) bounds every x >= 1
    }
    if (Ls >= k_eff) atomicMax(&s_lo, (unsigned long long)x);
    if (Us + 1 <= k_eff) atomicMin(&s_hi, (unsigned long long)x);
  }
  __syncthreads();
  if (tid == 0) {
    st[0] = (uint32_t)s_lo;                 // >= 1: x = 1 has sum lower = #valid >= k_eff
    st[1] = s_hi == (1ull << 32) ? 0u : (uint32_t)s_hi;
    st[2] = k_eff;
    st[3] = 0u;
    st[4] = st[5] = st[6] = st[7] = 0u;
  }
}

__global__ void __launch_bounds__(kShardThreads) topk_resolve_kernel(const uint32_t* __restrict__ msgs, int G,
                                                                     int rows, int rank,
                                                                     uint32_t* __restrict__ state) {
  __shared__ uint32_t H[kMsgCap];            // combined histogram (histogram mode)
  __shared__ uint32_t rh[256];
  __shared__ uint32_t s_gt[64], s_eq[64];
  __shared__ uint32_t s_dec[4];
  __shared__ int s_any_hist;
  const int row = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t* st = state + (size_t)row * kStateWords;
  if (st[3] != 0u) return;                    // resolved in an earlier round
  const uint32_t lo = st[0];
  const unsigned long long hi = st[1] == 0u ? (1ull << 32) : (unsigned long long)st[1];
  const uint32_t k_eff = st[2];
  auto M = [&](int s) { return msgs + ((size_t)s * rows + row) * kMsgWords; };
  uint32_t above = 0;
  if (tid == 0) s_any_hist = 0;
  __syncthreads();
  for (int s = 0; s < G; ++s) {
    above += M(s)[2];
    if (tid == 0 && M(s)[4] != 0u) s_any_hist = 1;
  }
  if (tid < 64) { s_gt[tid] = 0; s_eq[tid] = 0; }
  __syncthreads();
  const uint32_t need = k_eff - above;       // 1 <= need <= sum wc (T in [lo, hi))
  int sh = 0;
  while (((hi - lo - 1ull) >> sh) >= (unsigned long long)kMsgCap) ++sh;
  uint32_t T = 0u;
  bool resolved = false;
  if (!s_any_hist) {
    // exact select over the union of the shards' bracket keys: 4 passes of 8 bits
    uint32_t prefix = 0u, k_rem = need;
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      const uint32_t hmask = pass == 0 ? 0u : (0xFFFFFFFFu << (shift + 8));
      for (int i = tid; i < 256; i += kShardThreads) rh[i] = 0u;
      __syncthreads();
      for (int s = 0; s < G; ++s) {
        const uint32_t* m = M(s);
        const int wc = (int)m[3];
        for (int i = tid; i < wc; i += kShardThreads) {
          const uint32_t key = m[kMsgHdr + i];
          if ((key & hmask) == (prefix & hmask)) atomicAdd(&rh[(key >> shift) & 255u], 1u);
        }
      }
      __syncthreads();
      if (warp == 0) {
        uint32_t c8[8], tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) { c8[q] = rh[255 - (lane * 8 + q)]; tot += c8[q]; }
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
    for (int s = 0; s < G; ++s) {
      const uint32_t* m = M(s);
      const int wc = (int)m[3];
      uint32_t g = 0, e = 0;
      for (int i = tid; i < wc; i += kShardThreads) {
        const uint32_t key = m[kMsgHdr + i];
        g += key > T;
        e += key == T;
      }
      if (g) atomicAdd(&s_gt[s], g);
      if (e) atomicAdd(&s_eq[s], e);
    }
    __syncthreads();
    resolved = true;
  } else {
    for (int i = tid; i < kMsgCap; i += kShardThreads) H[i] = 0u;
    __syncthreads();
    for (int s = 0; s < G; ++s) {
      const uint32_t* m = M(s);
      if (m[4] != 0u) {
        for (int i = tid; i < kMsgCap; i += kShardThreads) H[i] += m[kMsgHdr + i];
      } else {
        const int wc = (int)m[3];
        for (int i = tid; i < wc; i += kShardThreads) atomicAdd(&H[(m[kMsgHdr + i] - lo) >> sh], 1u);
      }
      __syncthreads();
    }
    // bin of rank `need` from the top: thread t holds bins 4t .. 4t+3 (kMsgCap = 4 * 512)
    uint32_t h4[4], tot = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) { h4[e] = H[tid * 4 + e]; tot += h4[e]; }
    uint32_t inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_down_sync(0xffffffffu, inc, o);
      if (lane + o < 32) inc += y;
    }
    __shared__ uint32_t wsum[kShardThreads / 32];
    if (lane == 0) wsum[warp] = inc;
    __syncthreads();
    uint32_t after = inc - tot;
    for (int w = warp + 1; w < kShardThreads / 32; ++w) after += wsum[w];
    uint32_t run = after;                      // keys in bins above 4 tid + 3
    for (int e = 3; e >= 0; --e) {
      if (run < need && run + h4[e] >= need) { s_dec[0] = (uint32_t)(tid * 4 + e); s_dec[1] = run; }
      run += h4[e];
    }
    __syncthreads();
    const uint32_t bstar = s_dec[0];
    if (sh == 0) {
      T = lo + bstar;
      // per shard: #> T and #== T from its histogram or its keys
      for (int s = 0; s < G; ++s) {
        const uint32_t* m = M(s);
        uint32_t g = 0, e = 0;
        if (m[4] != 0u) {
          for (int i = tid; i < kMsgCap; i += kShardThreads) {
            g += (uint32_t)i > bstar ? m[kMsgHdr + i] : 0u;
            e += (uint32_t)i == bstar ? m[kMsgHdr + i] : 0u;
          }
        } else {
          const int wc = (int)m[3];
          for (int i = tid; i < wc; i += kShardThreads) {
            g += m[kMsgHdr + i] > T;
            e += m[kMsgHdr + i] == T;
          }
        }
        if (g) atomicAdd(&s_gt[s], g);
        if (e) atomicAdd(&s_eq[s], e);
      }
      __syncthreads();
      resolved = true;
    } else if (tid == 0) {
      const unsigned long long nlo = (unsigned long long)lo + ((unsigned long long)bstar << sh);
      unsigned long long nhi = nlo + (1ull << sh);
      if (nhi > hi) nhi = hi;
      st[0] = (uint32_t)nlo;
      st[1] = nhi == (1ull << 32) ? 0u : (uint32_t)nhi;
    }
  }
  if (resolved && tid == 0) {
    uint32_t gt_tot = 0, eq_before = 0;
    for (int s = 0; s < G; ++s) {
      gt_tot += M(s)[2] + s_gt[s];
      if (s < rank) eq_before += s_eq[s];
    }
    const uint32_t ties = k_eff - gt_tot;      // keys == T to take, in global index order
    const uint32_t q = ties > eq_before ? min(ties - eq_before, s_eq[rank]) : 0u;
    st[3] = 1u;
    st[4] = T;
    st[5] = q;
    st[6] = need;
    st[7] = M(rank)[2] + s_gt[rank];
  }
}

socket_status launch_topk_bracket(const socket_cfg& c, const uint32_t* digests, int G, int Q, int k,
                                  uint32_t* state, cudaStream_t st) {
  const int rows = c.B * num_sel_rows(c);
  if (rows == 0) return SOCKET_OK;
  const size_t smem = (size_t)2 * G * Q * sizeof(uint32_t);
  cudaFuncSetAttribute(topk_bracket_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  topk_bracket_kernel<<<rows, kShardThreads, smem, st>>>(digests, G, rows, Q, k, state);
  return check_launch("topk_bracket_kernel");
}

socket_status launch_topk_resolve(const socket_cfg& c, const uint32_t* msgs, int G, int rank,
                                  uint32_t* state, cudaStream_t st) {
  const int rows = c.B * num_sel_rows(c);
  if (rows == 0) return SOCKET_OK;
  topk_resolve_kernel<<<rows, kShardThreads, 0, st>>>(msgs, G, rows, rank, state);
  return check_launch("topk_resolve_kernel");
}

}  // namespace sk
