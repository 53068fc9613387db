// Eq. 2 sparse attention over the selected rows with exact
// logits (l.271, l.309), as a split flash-decode with online softmax, and the
// log-sum-exp combine of partial states.  The dense variant (Eq. 1, every key
// j < seq_len) is the same kernel with an implicit contiguous index list.
//
// Work unit = (b, selection row, split).  A unit's NH query heads share the
// gathered K/V rows (NH = G in KV_SHARED and dense mode, 1 in PER_QHEAD mode).
// Within a CTA every half-warp (16 lanes, 8 d-elements per lane = one 128-bit
// load per 256-byte row) runs its own online softmax over blocks of 4 rows;
// the 8 half-warp states of a CTA are merged in shared memory into one
// partial (m, l, o) per (b, head, split), and a combine kernel merges splits.
#include "internal.cuh"

namespace sk {

constexpr int kDecWarps = 4;
constexpr int kDecThreads = kDecWarps * 32;
constexpr int kRowsPerIter = kDecWarps * 8;     // rows a CTA consumes per iteration
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct DecArgs {
  const uint16_t* q;
  const uint16_t* K;
  const uint16_t* V;
  const int32_t* idx;
  const int32_t* cnt;
  const int32_t* seq_lens;
  int k_stride;
  int H_q, H_kv, H_sel, N_max;
  int G;               // H_q / H_kv
  int per_qhead;       // selection per query head
  int n_splits, rows_per_split;
  float scale_log2;    // sm_scale * log2(e)
  float* part;         // [B][H_q][n_splits][d+2]
};

template <int NH, bool DENSE>
__global__ void __launch_bounds__(kDecThreads)
decode_split_kernel(DecArgs a) {
  constexpr int NV = 4 * NH;        // (row, head) scores per half-warp block
  const int unit = blockIdx.y;      // b * H_sel + r
  const int split = blockIdx.x;
  const int b = unit / a.H_sel, r = unit % a.H_sel;
  const int g = a.per_qhead ? r / a.G : r;
  const int h0 = a.per_qhead ? r : r * a.G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int half = lane >> 4, hl = lane & 15;

  const int n_rows = DENSE ? a.seq_lens[b] : a.cnt[unit];
  const int i_begin = split * a.rows_per_split;
  int i_end = i_begin + a.rows_per_split;
  if (i_end > n_rows) i_end = n_rows;

  // q fragment: 8 elements per lane, pre-scaled by sm_scale*log2(e)
  float qf[NH][8];
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const uint4 u = *reinterpret_cast<const uint4*>(a.q + ((size_t)b * a.H_q + h0 + h) * kD + hl * 8);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      qf[h][2 * e] = bf16lo(w[e]) * a.scale_log2;
      qf[h][2 * e + 1] = bf16hi(w[e]) * a.scale_log2;
    }
  }
  float o[NH][8];
  float m[NH], l[NH];
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    m[h] = -INFINITY;
    l[h] = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) o[h][e] = 0.f;
  }
  const uint16_t* Kbase = a.K + ((size_t)b * a.H_kv + g) * a.N_max * kD + hl * 8;
  const uint16_t* Vbase = a.V + ((size_t)b * a.H_kv + g) * a.N_max * kD + hl * 8;
  const int32_t* irow = DENSE ? nullptr : a.idx + (size_t)unit * a.k_stride;

  for (int it = i_begin; it < i_end; it += kRowsPerIter) {
    const int rb = it + warp * 8 + half * 4;     // first row of this half-warp's block
    int tok[4];
    bool ok[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = rb + q;
      ok[q] = i < i_end;
      tok[q] = ok[q] ? (DENSE ? i : irow[i]) : 0;
    }
    uint4 kv[4], vv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) kv[q] = ldg_nc_v4(Kbase + (size_t)tok[q] * kD);
#pragma unroll
    for (int q = 0; q < 4; ++q) vv[q] = ldg_nc_v4(Vbase + (size_t)tok[q] * kD);
    // partial dots: s[q*NH + h]
    float s[NV];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t w[4] = {kv[q].x, kv[q].y, kv[q].z, kv[q].w};
      float kf[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) { kf[2 * e] = bf16lo(w[e]); kf[2 * e + 1] = bf16hi(w[e]); }
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        float acc = qf[h][0] * kf[0];
#pragma unroll
        for (int e = 1; e < 8; ++e) acc = fmaf(qf[h][e], kf[e], acc);
        s[q * NH + h] = acc;
      }
    }
    // reduce-scatter over the 16 lanes of the half-warp
    int nv = NV;
    int own = 0;   // index of the value this lane owns after the reduction
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
      if (nv > 1) {
        const int hnv = nv >> 1;
        const bool up = (hl & off) != 0;
#pragma unroll
        for (int i = 0; i < NV / 2; ++i) {
          if (i < hnv) {
            const float send = up ? s[i] : s[i + hnv];
            const float keep = up ? s[i + hnv] : s[i];
            s[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
        if (up) own += hnv;
        nv = hnv;
      } else {
        s[0] += __shfl_xor_sync(0xffffffffu, s[0], off);
      }
    }
    // now lane owns nv (>=1) consecutive values starting at `own`: index q*NH + h
    // rows occupy lane bits 3 and 2 (off 8 and 4); mask invalid rows
    float sv[NV > 16 ? 2 : 1];
    const int nown = NV > 16 ? 2 : 1;
#pragma unroll
    for (int t = 0; t < nown; ++t) {
      const int vi = own + t;
      const int q = vi / NH;
      sv[t] = ok[q] ? s[t] : -INFINITY;
    }
    // block max over the 4 rows, per owned head
    float mb[2];
#pragma unroll
    for (int t = 0; t < nown; ++t) {
      float x = sv[t];
      x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 8));
      x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 4));
      mb[t] = x;
    }
    // broadcast block maxima and p values to every lane of the half-warp
    float mnew[NH], sc[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      // owner of (row 0, head h): value index h -> lane whose `own` covers h
      // lane bits: rows at bits 3..2, heads below; find lane id of value h
      int src, slot;
      if (NV <= 16) {
        src = h * (16 / NV);          // values map to lanes in order with 16/NV duplicates
        slot = 0;
      } else {
        src = h >> 1;
        slot = h & 1;
      }
      const float x = __shfl_sync(0xffffffffu, slot ? mb[1 % nown] : mb[0], (half << 4) | src);
      mnew[h] = fmaxf(m[h], x);
      sc[h] = (mnew[h] == -INFINITY) ? 1.f : exp2f(m[h] - mnew[h]);
    }
    // own p values
    float pv[2];
#pragma unroll
    for (int t = 0; t < nown; ++t) {
      const int vi = own + t;
      const int h = vi % NH;
      float mh = mnew[0];
#pragma unroll
      for (int hh = 1; hh < NH; ++hh) mh = (h == hh) ? mnew[hh] : mh;
      pv[t] = (mh == -INFINITY) ? 0.f : exp2f(sv[t] - mh);
    }
    float p[NV];
#pragma unroll
    for (int vi = 0; vi < NV; ++vi) {
      int src, slot;
      if (NV <= 16) {
        src = vi * (16 / NV);
        slot = 0;
      } else {
        src = vi >> 1;
        slot = vi & 1;
      }
      p[vi] = __shfl_sync(0xffffffffu, slot ? pv[1 % nown] : pv[0], (half << 4) | src);
    }
    // update l, o
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      float ps = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) ps += p[q * NH + h];
      l[h] = l[h] * sc[h] + ps;
      m[h] = mnew[h];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[h][e] *= sc[h];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t w[4] = {vv[q].x, vv[q].y, vv[q].z, vv[q].w};
      float vf[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) { vf[2 * e] = bf16lo(w[e]); vf[2 * e + 1] = bf16hi(w[e]); }
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const float pq = p[q * NH + h];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[h][e] = fmaf(pq, vf[e], o[h][e]);
      }
    }
  }

  // ---- merge the 8 half-warp states of the CTA ---------------------------
  __shared__ float sm_m[2 * kDecWarps][NH];
  __shared__ float sm_l[2 * kDecWarps][NH];
  __shared__ float sm_o[2 * kDecWarps][NH][kD];
  const int st = warp * 2 + half;
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    if (hl == 0) { sm_m[st][h] = m[h]; sm_l[st][h] = l[h]; }
#pragma unroll
    for (int e = 0; e < 8; ++e) sm_o[st][h][hl * 8 + e] = o[h][e];
  }
  __syncthreads();
  float* pbase = a.part + (((size_t)b * a.H_q + h0) * a.n_splits + split) * (kD + 2);
  for (int x = tid; x < NH * kD; x += kDecThreads) {
    const int h = x / kD, e = x % kD;
    float M = -INFINITY;
    for (int s2 = 0; s2 < 2 * kDecWarps; ++s2) M = fmaxf(M, sm_m[s2][h]);
    float Lsum = 0.f, O = 0.f;
    if (M != -INFINITY) {
      for (int s2 = 0; s2 < 2 * kDecWarps; ++s2) {
        const float w = exp2f(sm_m[s2][h] - M);
        Lsum = fmaf(w, sm_l[s2][h], Lsum);
        O = fmaf(w, sm_o[s2][h][e], O);
      }
    }
    float* pp = pbase + (size_t)h * a.n_splits * (kD + 2);
    pp[2 + e] = O;
    if (e == 0) { pp[0] = M; pp[1] = Lsum; }   // m in log2 units
  }
}

// Merge S partial states per (b, h).  part(bh, s) at base + s*s_stride + bh*bh_stride.
// m is in log2 units when log2_units != 0 (split partials of this library),
// natural units otherwise (socket_lse_combine input / partial output).
__global__ void combine_kernel(const float* __restrict__ part, int S, long long s_stride,
                               long long bh_stride, int log2_units, uint16_t* __restrict__ out,
                               float* __restrict__ lse, float* __restrict__ part_out) {
  const int bh = blockIdx.x;
  const int e = threadIdx.x;     // 128 threads
  const float* pb = part + (size_t)bh * bh_stride;
  const float cvt = log2_units ? 1.0f : kLog2e;    // to log2 units
  float M = -INFINITY;
  for (int s = 0; s < S; ++s) M = fmaxf(M, pb[(size_t)s * s_stride] * cvt);
  float Lsum = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int s = 0; s < S; ++s) {
      const float* p = pb + (size_t)s * s_stride;
      const float w = exp2f(p[0] * cvt - M);
      Lsum = fmaf(w, p[1], Lsum);
      O = fmaf(w, p[2 + e], O);
    }
  }
  if (out) {
    const float y = (Lsum > 0.f) ? O / Lsum : 0.f;
    out[(size_t)bh * kD + e] = (uint16_t)f2bf_bits(y);
  }
  if (e == 0 && lse) lse[bh] = (Lsum > 0.f) ? (M + log2f(Lsum)) * kLn2 : -INFINITY;
  if (part_out) {
    float* po = part_out + (size_t)bh * (kD + 2);
    po[2 + e] = O;
    if (e == 0) { po[0] = (M == -INFINITY) ? -INFINITY : M * kLn2; po[1] = Lsum; }
  }
}

static void pick_splits(int units, int max_rows, int& n_splits, int& rows_per_split) {
  const int target = 6 * kNumSMs;                  // CTAs in flight
  int ns = (target + units - 1) / units;
  const int max_ns = (max_rows + 2 * kRowsPerIter - 1) / (2 * kRowsPerIter);  // >= 2 iterations
  if (ns > max_ns) ns = max_ns;
  if (ns < 1) ns = 1;
  int rps = (max_rows + ns - 1) / ns;
  rps = (rps + kRowsPerIter - 1) / kRowsPerIter * kRowsPerIter;
  if (rps < kRowsPerIter) rps = kRowsPerIter;
  n_splits = (max_rows + rps - 1) / rps;
  if (n_splits < 1) n_splits = 1;
  rows_per_split = rps;
}

static void decode_geometry(const socket_cfg& c, int k, bool dense, int& units, int& NH,
                            int& n_splits, int& rps) {
  const bool per_q = !dense && c.group_mode == SOCKET_GROUP_PER_QHEAD;
  const int H_sel = per_q ? c.H_q : c.H_kv;
  units = c.B * H_sel;
  NH = per_q ? 1 : c.H_q / c.H_kv;
  pick_splits(units, dense ? c.N_max : k, n_splits, rps);
}

size_t decode_workspace_bytes(const socket_cfg& c, int k, bool dense) {
  int units, NH, ns, rps;
  decode_geometry(c, k, dense, units, NH, ns, rps);
  return (size_t)c.B * c.H_q * ns * (kD + 2) * sizeof(float);
}

socket_status launch_decode(const socket_cfg& c, const void* q, const void* K, const void* V,
                            const int32_t* idx, const int32_t* cnt, int k,
                            const int32_t* seq_lens, bool dense, void* out, float* lse,
                            float* partial, void* ws, size_t ws_bytes, cudaStream_t st) {
  int units, NH, ns, rps;
  decode_geometry(c, k, dense, units, NH, ns, rps);
  const size_t need = (size_t)c.B * c.H_q * ns * (kD + 2) * sizeof(float);
  if (ws_bytes < need) return fail(SOCKET_EWORKSPACE, "decode: workspace too small");
  if (units == 0) return SOCKET_OK;
  DecArgs a;
  a.q = (const uint16_t*)q;
  a.K = (const uint16_t*)K;
  a.V = (const uint16_t*)V;
  a.idx = idx;
  a.cnt = cnt;
  a.seq_lens = seq_lens;
  a.k_stride = k;
  a.H_q = c.H_q;
  a.H_kv = c.H_kv;
  a.H_sel = units / c.B;
  a.N_max = c.N_max;
  a.G = c.H_q / c.H_kv;
  a.per_qhead = (!dense && c.group_mode == SOCKET_GROUP_PER_QHEAD) ? 1 : 0;
  a.n_splits = ns;
  a.rows_per_split = rps;
  a.scale_log2 = c.sm_scale * kLog2e;
  a.part = (float*)ws;
  dim3 grid(ns, units);
#define SK_DEC(NHV, DN)                                                         \
  decode_split_kernel<NHV, DN><<<grid, kDecThreads, 0, st>>>(a);                \
  break;
  if (dense) {
    switch (NH) {
      case 1: SK_DEC(1, true)
      case 2: SK_DEC(2, true)
      case 4: SK_DEC(4, true)
      case 8: SK_DEC(8, true)
      default: return fail(SOCKET_EUNSUPPORTED, "decode: group size must be 1, 2, 4 or 8");
    }
  } else {
    switch (NH) {
      case 1: SK_DEC(1, false)
      case 2: SK_DEC(2, false)
      case 4: SK_DEC(4, false)
      case 8: SK_DEC(8, false)
      default: return fail(SOCKET_EUNSUPPORTED, "decode: group size must be 1, 2, 4 or 8");
    }
  }
#undef SK_DEC
  socket_status s = check_launch("decode_split_kernel");
  if (s != SOCKET_OK) return s;
  combine_kernel<<<c.B * c.H_q, kD, 0, st>>>((const float*)ws, ns, (kD + 2), (long long)ns * (kD + 2),
                                            1, (uint16_t*)out, lse, partial);
  return check_launch("combine_kernel");
}

socket_status launch_lse_combine(const socket_cfg& c, const float* partials, int G, void* out,
                                 float* lse, cudaStream_t st) {
  const int BH = c.B * c.H_q;
  if (BH == 0) return SOCKET_OK;
  combine_kernel<<<BH, kD, 0, st>>>(partials, G, (long long)BH * (kD + 2), (kD + 2), 0,
                                   (uint16_t*)out, lse, nullptr);
  return check_launch("combine_kernel");
}

}  // namespace sk
