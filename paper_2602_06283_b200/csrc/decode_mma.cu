// Tensor-core split flash-decode over gathered rows: Eq. 2 (PAPER.md l.169-174,
// exact logits per l.271 / l.309) and the dense Eq. 1 variant.
//
// Per warp and tile of 16 selected rows (all NH <= 8 query heads of the unit
// at once, heads padded to the MMA's N = 8):
//   S^T[16 rows x 8 heads]  = K_tile[16 x 128] . Q^T[128 x 8]      8 x mma.m16n8k16
//   online softmax on S^T (fp32, log2 domain)
//   O^T[128 x 8 heads]     += V_tile^T[128 x 16] . P[16 x 8]        8 x mma.m16n8k16
// K and V rows are gathered by cp.async into a per-warp 3-stage shared-memory
// ring, XOR-swizzled in 16-byte chunks so `ldmatrix` (A = K, A = V^T via .trans)
// is bank-conflict free.  P is rounded to bf16 (row sums use the same rounded
// values) and moved from the accumulator layout to the B-operand layout with
// `movmatrix.trans`.  The O^T accumulator layout gives every lane the same two
// heads it holds the softmax state of, so the rescale is lane-local.
#include "mma_dev.cuh"

namespace sk {

#ifndef SK_DECODE_WARPS
#define SK_DECODE_WARPS 4   // experiments only (tools/variant_build.py)
#endif
constexpr int kMmaWarps = SK_DECODE_WARPS;
constexpr int kMmaThreads = kMmaWarps * 32;
#ifndef SK_DECODE_STAGES
#define SK_DECODE_STAGES 3   // experiments only (tools/variant_build.py)
#endif
constexpr int kMmaStages = SK_DECODE_STAGES;   // cp.async ring depth (tiles per warp)
constexpr int kMmaRing = kMmaWarps * kMmaStages * kTileBytes;   // 96 KB
constexpr int kMmaMaxRows = 2048;                                // rows per split (idx staging)

struct MmaArgs {
  const uint16_t* q;
  const uint16_t* K;
  const uint16_t* V;
  const int32_t* idx;
  const int32_t* cnt;
  const int32_t* seq_lens;
  int k_stride;
  int H_q, H_kv, H_sel, N_max, G, NH;
  int per_qhead;
  int n_splits, rows_per_split;
  float scale_log2;
  float* part;   // [B][H_q][n_splits][d+2], m in log2 units
  int* tickets;  // [units], zero on entry; the last split of a unit merges
  uint16_t* out; // [B][H_q][d] bf16 (nullable)
  float* lse;    // [B][H_q] (nullable)
  float* part_out;  // [B][H_q][d+2] natural-log units (nullable)
};

template <bool DENSE>
__global__ void __launch_bounds__(kMmaThreads)
decode_mma_kernel(MmaArgs a) {
  __shared__ int s_idx[DENSE ? 1 : kMmaMaxRows];
  extern __shared__ __align__(1024) char ring[];
  const int unit = blockIdx.y, split = blockIdx.x;
  const int b = unit / a.H_sel, r = unit % a.H_sel;
  const int g = a.per_qhead ? r / a.G : r;
  const int h0 = a.per_qhead ? r : r * a.G;
  const int NH = a.NH;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;

  asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: idx / cnt of the predecessor
  const int n_rows = DENSE ? a.seq_lens[b] : a.cnt[unit];
  const int i_begin = split * a.rows_per_split;
  const int i_end = min(i_begin + a.rows_per_split, n_rows);
  if (!DENSE) {
    const int32_t* irow = a.idx + (size_t)unit * a.k_stride;
    for (int i = i_begin + tid; i < i_end; i += kMmaThreads) s_idx[i - i_begin] = irow[i];
    __syncthreads();
  }

  // Q^T as B fragments: b0 = Q[h = gid][ks*16 + 2 tig .. +1], b1 = ... + 8
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
  float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;   // heads 2 tig, 2 tig + 1

  const uint16_t* Kb = a.K + ((size_t)b * a.H_kv + g) * a.N_max * kD;
  const uint16_t* Vb = a.V + ((size_t)b * a.H_kv + g) * a.N_max * kD;
  const uint32_t ring0 = smem_u32(ring) + (uint32_t)warp * (kMmaStages * kTileBytes);

  const int ntiles = (i_end - i_begin + kTileRows - 1) / kTileRows;
  // warp w handles tiles w, w + 4, ...
  auto issue = [&](int t, int stage) {
    const int row0 = i_begin + t * kTileRows;
    const uint32_t kbuf = ring0 + stage * kTileBytes, vbuf = kbuf + kTileRows * 256;
#pragma unroll
    for (int it = 0; it < 8; ++it) {                // 16 rows x 16 chunks / 32 lanes
      const int c = (it * 32 + lane) & 15, rr = (it * 32 + lane) >> 4;
      const int i = row0 + rr;
      const bool v = i < i_end;
      const int tok = v ? (DENSE ? i : s_idx[i - i_begin]) : 0;
      cp16(kbuf + swz(rr, c), Kb + (size_t)tok * kD + c * 8, v);
      cp16(vbuf + swz(rr, c), Vb + (size_t)tok * kD + c * 8, v);
    }
  };
  int my = 0;   // number of tiles this warp owns
  for (int t = warp; t < ntiles; t += kMmaWarps) ++my;
#pragma unroll
  for (int s = 0; s < kMmaStages - 1; ++s) {
    if (s < my) issue(warp + s * kMmaWarps, s);
    cp_commit();
  }
  for (int j = 0; j < my; ++j) {
    const int t = warp + j * kMmaWarps;
    const int jn = j + kMmaStages - 1;
    if (jn < my) issue(warp + jn * kMmaWarps, jn % kMmaStages);
    cp_commit();
    cp_wait<kMmaStages - 1>();
    __syncwarp();
    const uint32_t kbuf = ring0 + (j % kMmaStages) * kTileBytes, vbuf = kbuf + kTileRows * 256;
    // ---- S^T = K . Q^T ---------------------------------------------------------
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
    // ---- online softmax (rows gid, gid + 8; heads 2 tig, 2 tig + 1) -------------
    const int row0 = i_begin + t * kTileRows;
    const bool v0 = row0 + gid < i_end, v1 = row0 + gid + 8 < i_end;
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
    // row sums of the bf16-rounded weights (numerator and denominator agree)
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
    const uint32_t pb0 = movm_t(P01), pb1 = movm_t(P23);   // B fragments: P[k rows][n heads]
    // ---- O^T += V^T . P ---------------------------------------------------------
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
    __syncwarp();   // all lanes done reading this stage before it is refilled
  }
  cp_wait<0>();

  // ---- merge the warps' states (reuse the ring) ----------------------------------
  __syncthreads();
  float* sm_o = reinterpret_cast<float*>(ring);                   // [warps][8 heads][128]
  float* sm_m = sm_o + kMmaWarps * 8 * kD;                          // [warps][8]
  float* sm_l = sm_m + kMmaWarps * 8;
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
  __syncthreads();
  float* pbase = a.part + (((size_t)b * a.H_q + h0) * a.n_splits + split) * (kD + 2);
  for (int x = tid; x < NH * kD; x += kMmaThreads) {
    const int h = x / kD, e = x % kD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kMmaWarps; ++w) M = fmaxf(M, sm_m[w * 8 + h]);
    float Ls = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kMmaWarps; ++w) {
        const float wt = exp2f(sm_m[w * 8 + h] - M);
        Ls = fmaf(wt, sm_l[w * 8 + h], Ls);
        O = fmaf(wt, sm_o[(w * 8 + h) * kD + e], O);
      }
    }
    float* pp = pbase + (size_t)h * a.n_splits * (kD + 2);
    pp[2 + e] = O;
    if (e == 0) { pp[0] = M; pp[1] = Ls; }
  }

  // ---- the last split CTA of this unit merges all splits (LSE combine) --------
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&a.tickets[unit], 1) == a.n_splits - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  constexpr float kLn2M = 0.6931471805599453f;
  // (a) per head: M = max_s m_s, split weights w_s = 2^(m_s - M) into smem (the
  //     ring is free now), L = sum_s w_s l_s.  One warp per head, lanes over splits.
  const int ns = a.n_splits;
  float* sw = reinterpret_cast<float*>(ring);                 // [NH][ns] weights
  float* sML = sw + NH * ns;                                  // [NH][2]  M, L
  const size_t pstride = (size_t)ns * (kD + 2);
  for (int h = warp; h < NH; h += kMmaWarps) {
    const float* pb = a.part + ((size_t)b * a.H_q + h0 + h) * pstride;
    float M = -INFINITY;
    for (int s2 = lane; s2 < ns; s2 += 32) M = fmaxf(M, __ldcg(pb + (size_t)s2 * (kD + 2)));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float Ls = 0.f;
    for (int s2 = lane; s2 < ns; s2 += 32) {
      const float* p2 = pb + (size_t)s2 * (kD + 2);
      const float wt = (M == -INFINITY) ? 0.f : exp2f(__ldcg(p2) - M);
      sw[h * ns + s2] = wt;
      Ls = fmaf(wt, __ldcg(p2 + 1), Ls);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) Ls += __shfl_xor_sync(0xffffffffu, Ls, o);
    if (lane == 0) { sML[2 * h] = M; sML[2 * h + 1] = Ls; }
  }
  __syncthreads();
  // (b) each thread owns 4 consecutive dims of one head and streams the split
  //     partials with independent float2 loads (the row pitch d + 2 keeps 8-byte
  //     alignment), 8 splits in flight
  for (int x = tid; x < NH * (kD / 4); x += kMmaThreads) {
    const int h = x / (kD / 4), e = (x % (kD / 4)) * 4;
    const float* pb = a.part + ((size_t)b * a.H_q + h0 + h) * pstride + 2 + e;
    const float* wh = sw + h * ns;
    float O0 = 0.f, O1 = 0.f, O2 = 0.f, O3 = 0.f;
    int s2 = 0;
    for (; s2 + 8 <= ns; s2 += 8) {
      float2 u[8], v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        u[j] = __ldcg(reinterpret_cast<const float2*>(pb + (size_t)(s2 + j) * (kD + 2)));
        v[j] = __ldcg(reinterpret_cast<const float2*>(pb + (size_t)(s2 + j) * (kD + 2) + 2));
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float wt = wh[s2 + j];
        O0 = fmaf(wt, u[j].x, O0); O1 = fmaf(wt, u[j].y, O1);
        O2 = fmaf(wt, v[j].x, O2); O3 = fmaf(wt, v[j].y, O3);
      }
    }
    for (; s2 < ns; ++s2) {
      const float2 u = __ldcg(reinterpret_cast<const float2*>(pb + (size_t)s2 * (kD + 2)));
      const float2 v = __ldcg(reinterpret_cast<const float2*>(pb + (size_t)s2 * (kD + 2) + 2));
      const float wt = wh[s2];
      O0 = fmaf(wt, u.x, O0); O1 = fmaf(wt, u.y, O1);
      O2 = fmaf(wt, v.x, O2); O3 = fmaf(wt, v.y, O3);
    }
    const float M = sML[2 * h], Ls = sML[2 * h + 1];
    const size_t bh = (size_t)b * a.H_q + h0 + h;
    if (a.out) {
      uint2 pk;
      pk.x = pack_bf16(Ls > 0.f ? O0 / Ls : 0.f, Ls > 0.f ? O1 / Ls : 0.f);
      pk.y = pack_bf16(Ls > 0.f ? O2 / Ls : 0.f, Ls > 0.f ? O3 / Ls : 0.f);
      *reinterpret_cast<uint2*>(a.out + bh * kD + e) = pk;
    }
    if (e == 0 && a.lse) a.lse[bh] = (Ls > 0.f) ? (M + log2f(Ls)) * kLn2M : -INFINITY;
    if (a.part_out) {
      float* po = a.part_out + bh * (kD + 2);
      po[2 + e] = O0; po[3 + e] = O1; po[4 + e] = O2; po[5 + e] = O3;
      if (e == 0) { po[0] = (M == -INFINITY) ? -INFINITY : M * kLn2M; po[1] = Ls; }
    }
  }
  if (tid == 0) a.tickets[unit] = 0;   // ready for the next launch / graph replay
}

socket_status launch_decode_mma(const socket_cfg& c, const void* q, const void* K, const void* V,
                                const int32_t* idx, const int32_t* cnt, int k,
                                const int32_t* seq_lens, bool dense, int units, int NH,
                                int n_splits, int rps, float* part, int* tickets, void* out,
                                float* lse, float* part_out, cudaStream_t st, bool pdl) {
  MmaArgs a;
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
  a.NH = NH;
  a.per_qhead = (!dense && c.group_mode == SOCKET_GROUP_PER_QHEAD) ? 1 : 0;
  a.n_splits = n_splits;
  a.rows_per_split = rps;
  a.scale_log2 = c.sm_scale * kLog2eM;
  a.part = part;
  a.tickets = tickets;
  a.out = (uint16_t*)out;
  a.lse = lse;
  a.part_out = part_out;
  if ((size_t)NH * n_splits * sizeof(float) + 64 > (size_t)kMmaRing)
    return fail(SOCKET_EUNSUPPORTED, "decode: too many splits for the in-kernel LSE merge");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_splits, units);
  cfg.blockDim = dim3(kMmaThreads);
  cfg.dynamicSmemBytes = kMmaRing;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e;
  if (dense) {
    cudaFuncSetAttribute(decode_mma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMmaRing);
    e = cudaLaunchKernelEx(&cfg, decode_mma_kernel<true>, a);
  } else {
    cudaFuncSetAttribute(decode_mma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMmaRing);
    e = cudaLaunchKernelEx(&cfg, decode_mma_kernel<false>, a);
  }
  if (e != cudaSuccess) return fail(SOCKET_ECUDA, std::string("decode launch: ") + cudaGetErrorString(e));
  return check_launch("decode_mma_kernel");
}

}  // namespace sk
