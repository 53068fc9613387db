// Device routines shared by several kernels of libsocket_b200 (not part of the ABI).
#pragma once
#include "internal.cuh"

namespace sk {

#ifdef SK_TRACE
// per-CTA phase stamps of the tables / append CTAs (tools/trace_prologue.py):
// [cta][0] = globaltimer at entry, [cta][1..7] = clock64 at phase ends, [cta][8] = smid
static __device__ unsigned long long g_pro_trace[8192 * 12];   // per translation unit
#define PRO_STAMP(i)                                                                        \
  do {                                                                                      \
    if (threadIdx.x == 0 && blockIdx.x < 8192) {                                            \
      unsigned long long v;                                                                 \
      if ((i) == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));                   \
      else v = clock64();                                                                   \
      g_pro_trace[blockIdx.x * 12 + (i)] = v;                                               \
      if ((i) == 1) { unsigned sm; asm("mov.u32 %0, %%smid;" : "=r"(sm)); g_pro_trace[blockIdx.x * 12 + 11] = sm; } \
    }                                                                                       \
  } while (0)
#else
#define PRO_STAMP(i) \
  do {               \
  } while (0)
#endif

constexpr int kTabThreads = 256;  // one thread per (table, hyperplane row) of a 32-table chunk
constexpr int kTabPerCta = 32;    // tables per CTA
constexpr int kMaxHeads = 8;      // heads per selection row

// Byte offset of (row-local key j, slot s) inside one (b, kv-head) code region.
__device__ __forceinline__ size_t code_off(int j, int s, int Lp) {
  const int CB = Lp < 16 ? Lp : 16;
  return ((size_t)(j >> 5) * (Lp / CB) + s / CB) * (32 * CB) + (j & 31) * CB + (s % CB);
}
// table held by slot s of key j
__device__ __forceinline__ int slot_table(int s, int j, int Lp) {
  const int M = (Lp < 32 ? Lp : 32) - 1;
  return (s & ~M) | ((s + j) & M);
}

// bf16 bits -> fp64, exactly (bf16 -> fp32 is a shift; fp32 -> fp64 is exact)
__device__ __forceinline__ double bf16_to_f64(uint32_t h) {
  return (double)__uint_as_float(h << 16);
}

// Shared memory of one tables CTA (dynamic; tables_smem_bytes(NH) bytes):
//   qd   [kD][NH]  fp64 query heads (phase 1)      } union
//   half [NH][2][16][kTabPerCta] fp32 (phase 3-4)  }
//   fx   [NH][8][2][kTabPerCta]  fp64 sigma factors (table fastest: conflict-free reads)
__host__ __device__ constexpr size_t tables_smem_bytes(int NH) {
  return (size_t)NH * kTabPerCta * 16 * 8 +
         ((size_t)NH * kD * 8 > (size_t)NH * 2 * 16 * kTabPerCta * 4
              ? (size_t)NH * kD * 8
              : (size_t)NH * 2 * 16 * kTabPerCta * 4);
}

// One CTA = (b, selection row) x kTabPerCta tables [l0, l0 + 32), NH query heads.
//  1. thread (tl, i) = (tid >> 3, tid & 7) owns W row (l0 + tl, i) and computes
//     x_h = sum_t W[t] q_h[t] for every head h in fp64 (bf16 x bf16 products
//     are exact in fp64; CH interleaved partial sums hide the DFMA latency, so
//     x is the double dot product up to a few fp64 roundings);
//  2. u = tanh(x)/sqrt(d) (Alg. 2 l.217) and the two sigma factors
//     sigma(+-2u/tau) with the accurate fp32 functions (<= 2 ulp each);
//  3. half tables lo(r & 15) = prod_{i<4} f_i, hi(r >> 4) = prod_{i>=4} f_i in
//     fp64, rounded once to fp32;
//  4. T(r) = sum_h lo_h * hi_h (fp32 fma, h ascending); consecutive threads
//     write consecutive table columns of one LUT row (and/or the plain tables).
template <int NH>
__device__ __forceinline__ void tables_cta(const uint16_t* __restrict__ q,
                                           const uint16_t* __restrict__ W, float* __restrict__ plain,
                                           float* __restrict__ lut, int H_q, int H_sel, int L, int P,
                                           int Lp, float tau, int row, int l0, char* smem) {
  double* fx = reinterpret_cast<double*>(smem);                                   // [NH][8][2][32]
  double* qd = reinterpret_cast<double*>(smem + (size_t)NH * kTabPerCta * 16 * 8);  // [kD][NH]
  float* half = reinterpret_cast<float*>(qd);                                     // [NH][2][16][32]
  const int b = row / H_sel, r = row % H_sel;
  const int h0 = (NH == 1) ? r : r * NH;     // first query head of the row
  const int R = 1 << P;
  const int tid = threadIdx.x;
  PRO_STAMP(0);
  PRO_STAMP(1);
  for (int e = tid; e < NH * kD; e += kTabThreads) {
    const int h = e / kD, t = e % kD;
    qd[t * NH + h] = bf16_to_f64(q[((size_t)b * H_q + h0 + h) * kD + t]);
  }
  __syncthreads();
  PRO_STAMP(2);
  // 1. projections
  const int tl = tid >> 3, i = tid & 7;
  const int l = l0 + tl;
  const bool active = l < L && i < P;
  // CH independent partial sums per head (t = CH m + c goes to chain c), so
  // the fp64 FMA latency is hidden; the chains are added pairwise at the end
  constexpr int CH = NH >= 8 ? 2 : (NH >= 4 ? 4 : 8);
  double acc[NH];
  {
    double part[NH][CH];
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
      for (int c = 0; c < CH; ++c) part[h][c] = 0.0;
    if (active) {
      const uint4* wrow = reinterpret_cast<const uint4*>(W + ((size_t)l * P + i) * kD);
#pragma unroll 1
      for (int c = 0; c < kD / 32; ++c) {          // 4 batches of 32 elements
        uint4 wv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) wv[u] = __ldg(wrow + c * 4 + u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t wd[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int t = c * 32 + u * 8 + e;
            const double w = bf16_to_f64((e & 1) ? (wd[e >> 1] >> 16) : (wd[e >> 1] & 0xFFFFu));
            const double* qt = qd + t * NH;
#pragma unroll
            for (int h = 0; h < NH; ++h) part[h][e % CH] = fma(w, qt[h], part[h][e % CH]);
          }
        }
      }
    }
#pragma unroll
    for (int h = 0; h < NH; ++h) {
#pragma unroll
      for (int w = CH / 2; w >= 1; w >>= 1)
#pragma unroll
        for (int c = 0; c < w; ++c) part[h][c] += part[h][c + w];
      acc[h] = part[h][0];
    }
  }
  PRO_STAMP(3);
  // 2. sigma factors (c_{r,i} = +1 iff bit i of r is set, reading R-5)
  if (active) {
    const float inv_sqrt_d = 0.08838834764831845f;   // 1/sqrt(128), correctly rounded
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const float uu = tanhf((float)acc[h]) * inv_sqrt_d;   // Alg. 2 l.217
      const float a = 2.0f * uu / tau;                       // logit gap of bit i
      const float fp = 1.0f / (1.0f + expf(-a));             // c_{r,i} = +1 (bit set)
      const float fm = 1.0f / (1.0f + expf(a));              // c_{r,i} = -1
      fx[((h * 8 + i) * 2 + 1) * kTabPerCta + tl] = (double)fp;
      fx[((h * 8 + i) * 2 + 0) * kTabPerCta + tl] = (double)fm;
    }
  }
  __syncthreads();   // qd dead from here: `half` reuses it
  PRO_STAMP(4);
  // 3. half tables (bits 0..3 and 4..P-1; a missing bit contributes 1): one
  //    thread per (head, table, half) builds its 16 entries as the product
  //    ((f0 f1) f2) f3 by doubling (4 + 8 + 16 fp64 multiplies).
  for (int task = tid; task < NH * 2 * kTabPerCta; task += kTabThreads) {
    const int t2 = task % kTabPerCta, hi = (task / kTabPerCta) & 1, h = task / (2 * kTabPerCta);
    double f[4][2];
#pragma unroll
    for (int bit = 0; bit < 4; ++bit) {
      const int ib = hi * 4 + bit;
      f[bit][0] = ib < P ? fx[((h * 8 + ib) * 2 + 0) * kTabPerCta + t2] : 1.0;
      f[bit][1] = ib < P ? fx[((h * 8 + ib) * 2 + 1) * kTabPerCta + t2] : 1.0;
    }
    double p01[4], p012[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) p01[e] = f[0][e & 1] * f[1][e >> 1];
#pragma unroll
    for (int e = 0; e < 8; ++e) p012[e] = p01[e & 3] * f[2][e >> 2];
    float* hrow = half + (size_t)((h * 2 + hi) * 16) * kTabPerCta + t2;
#pragma unroll
    for (int e = 0; e < 16; ++e) hrow[e * kTabPerCta] = (float)(p012[e & 7] * f[3][e >> 3]);
  }
  __syncthreads();
  PRO_STAMP(5);
  // 4. entries T(rr) = sum_h lo_h(rr & 15) hi_h(rr >> 4) (fp32 fma, h ascending):
  //    thread (t2 = tid & 31, g = tid >> 5) writes rows rr = 16 rh + rl for
  //    rh in {g, g + 8}; a warp stores 32 consecutive LUT columns per row.
  const int panels = Lp <= 64 ? 1 : (Lp + 63) / 64;
  float* lrow = lut ? lut + (size_t)row * panels * (256 * 64) : nullptr;
  {
    const int t2 = tid & 31, g = tid >> 5;
    const int ll = l0 + t2;
    if (ll < Lp) {
      const bool lvalid = ll < L;
      float hv[2][NH];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int h = 0; h < NH; ++h) hv[m][h] = half[((h * 2 + 1) * 16 + g + 8 * m) * kTabPerCta + t2];
#pragma unroll 4
      for (int rl = 0; rl < 16; ++rl) {
        float lo[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) lo[h] = half[((h * 2 + 0) * 16 + rl) * kTabPerCta + t2];
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int rr = (g + 8 * m) * 16 + rl;
          float T = 0.f;
          if (lvalid && rr < R) {
#pragma unroll
            for (int h = 0; h < NH; ++h) T = fmaf(lo[h], hv[m][h], T);
            if (plain) plain[((size_t)row * L + ll) * R + rr] = T;
          }
          if (lrow) {
            if (Lp >= 32) {
              lrow[(size_t)(ll >> 6) * (256 * 64) + rr * 64 + (ll & 63)] = T;
            } else {
              for (int cc = ll; cc < 32; cc += Lp) lrow[rr * 64 + cc] = T;
            }
          }
        }
      }
    }
  }
  PRO_STAMP(6);
}

// Append path (Alg. 1 on a few new keys; the decode step's per-step hash).
// One CTA = (key, 32-table chunk); thread (tl, i) = (tid >> 3, tid & 7) owns
// W row (l0 + tl, i): x = sum_t W[t] k[t] in fp32 with fmaf, t ascending --
// the same arithmetic as the SIMT prefill kernel, so both give identical
// codes.  The 8 rows of a table sit in 8 consecutive lanes, so one ballot
// yields 4 code bytes per warp; slot s = (l & ~M) | ((l - j) & M) of key j
// (inverse of slot_table).  Warp 0 of chunk 0 also writes ||v_j|| with
// exactly vnorm_kernel's summation order.  With append_last, key j is
// seq_lens[b] - 1 of each (b, kv head) (skipped for empty sequences).
// `ks` is 128 floats of shared memory.
__device__ __forceinline__ void append_cta(
    const uint16_t* __restrict__ K, const uint16_t* __restrict__ W, uint8_t* __restrict__ codes,
    const uint16_t* __restrict__ V, float* __restrict__ vnorm, int N_max, int L, int P, int Lp,
    int n_begin, int n_count, int append_last, const int32_t* __restrict__ seq_lens, int H_kv,
    int key, int l0, float* ks) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int bh = key / n_count;
  int j = n_begin + key % n_count;
  if (append_last) {                      // decode step: the newest key j = seq_lens[b] - 1
    const int n = seq_lens[bh / H_kv];
    if (n <= 0) return;                   // uniform over the CTA
    j = n - 1;
  }
  PRO_STAMP(0);
  PRO_STAMP(1);
  const uint16_t* krow = K + ((size_t)bh * N_max + j) * kD;
  if (tid < kD / 2) {
    const uint32_t u = reinterpret_cast<const uint32_t*>(krow)[tid];
    ks[2 * tid] = bf16lo(u);
    ks[2 * tid + 1] = bf16hi(u);
  }
  __syncthreads();
  PRO_STAMP(2);
  const int tl = tid >> 3, i = tid & 7;
  const int l = l0 + tl;
  bool bit = false;
  if (l < L && i < P) {
    const uint4* wrow = reinterpret_cast<const uint4*>(W + ((size_t)l * P + i) * kD);
    float x = 0.f;
#pragma unroll 1
    for (int c = 0; c < kD / 32; ++c) {
      uint4 wv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) wv[u] = __ldg(wrow + c * 4 + u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t wd[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float w = (e & 1) ? bf16hi(wd[e >> 1]) : bf16lo(wd[e >> 1]);
          x = fmaf(w, ks[c * 32 + u * 8 + e], x);
        }
      }
    }
    bit = x >= 0.f;                        // sign(0) = +1 (R-3)
  }
  PRO_STAMP(3);
  const unsigned bal = __ballot_sync(0xffffffffu, bit);
  if (i == 0 && l < Lp) {
    const uint32_t code = (bal >> (lane & 24)) & 0xFFu;   // row i -> bit i (R-4)
    const int M = (Lp < 32 ? Lp : 32) - 1;
    const int s = (l & ~M) | ((l - j) & M);
    codes[(size_t)bh * N_max * Lp + code_off(j, s, Lp)] = (uint8_t)code;
  }
  if (V && l0 == 0 && tid < 32) {
    const uint2 u = *reinterpret_cast<const uint2*>(V + ((size_t)bh * N_max + j) * kD + lane * 4);
    float a = bf16lo(u.x), b = bf16hi(u.x), c = bf16lo(u.y), e = bf16hi(u.y);
    float sq = fmaf(a, a, fmaf(b, b, fmaf(c, c, e * e)));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) vnorm[(size_t)bh * N_max + j] = sqrtf(sq);
  }
  PRO_STAMP(6);
}

}  // namespace sk
