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

// bf16 bits -> fp64 / fp32, exactly
__device__ __forceinline__ double bf16_to_f64(uint32_t h) {
  return (double)__uint_as_float(h << 16);
}

// ============================================================================
// Projection prologue of a decode step: Alg. 2 tables and Alg. 1 on the new
// keys, both as small tiled GEMMs (one 256-thread CTA per tile):
//
//   tables tile  = 16 query vectors x 8 tables (8P W rows), fp64:
//     x[m][w] = sum_t q_m[t] W_w[t], t ascending (bf16 x bf16 products are
//     exact in fp64, so this is the double dot product); staged in shared
//     memory as fp64 (each element converted once per tile), 2 x 2 register
//     micro-tile per thread.  Epilogue: u = tanh(x)/sqrt(d) (Alg. 2 l.217),
//     the sigma factors sigma(+-2u/tau) in accurate fp32, half tables
//     lo(r & 15) = prod_{i<4} f_i, hi(r >> 4) = prod_{i>=4} f_i in fp64
//     (rounded once), T(r) = sum_h lo_h hi_h in fp32 (h ascending), written as
//     the score kernel's LUT image and/or the plain [L][R] tables.
//   append tile  = 32 keys x 8 tables, fp32: x = sum_t W[t] k[t] with fmaf,
//     t ascending (the SIMT prefill's arithmetic, so both give identical
//     codes); bit = x >= 0 (R-3), row i -> bit i (R-4), written to slot
//     s = (l & ~M) | ((l - j) & M) of key j; the first table tile also writes
//     ||v_j|| (vnorm_kernel's summation order).
// ============================================================================
constexpr int kPT = 512;   // threads per tile CTA (16 warps)
constexpr int kTQ = 16;    // query vectors per tables tile
constexpr int kTT = 8;     // tables per tile
constexpr int kAK = 32;    // keys per append tile
constexpr int kQS = 24;    // row stride (doubles) of the staged q tile [t][m]  (= 16 words mod 32:
constexpr int kWS = 72;    // row stride (doubles) of the staged W tile [t][w]   conflict-free MMA fragments)
constexpr int kKS = 36;    // row stride (floats) of the staged key tile   [t][m]
constexpr int kAWS = 68;   // row stride (floats) of the staged W tile     [t][w]
constexpr int kFXS = 9;    // padded table stride of the factor array

__host__ __device__ constexpr size_t prologue_smem_bytes() {
  return (size_t)kD * (kQS + kWS) * 8;    // >= append staging and the epilogue arrays
}

struct ProArgs {
  const uint16_t* q;
  const uint16_t* W;
  float* plain;           // [B][H_sel][L][R] or null
  float* lut;             // LUT images [B*H_sel][panels][256][64] or null
  const uint16_t* K;
  const uint16_t* V;      // null: no norms
  const uint16_t* k_new;  // decode step: the new rows [B*H_kv][d] (append_last), or null --
  const uint16_t* v_new;  //   then the tiles read them here and store them into K_w / V_w
  uint16_t* K_w;
  uint16_t* V_w;
  uint8_t* codes;
  float* vnorm;
  const int32_t* seq_lens;
  int* tickets;           // zeroed by block 0 (decode tickets), or null
  int n_tickets;
  int B, H_q, H_sel, H_kv, N_max, L, P, Lp;
  float tau;
  int hard;               // SOCKET_SCORING_HARD: indicator factors [bit == (x >= 0)]
  int tpt;                // tables per tile: 8 for P <= 8, 64 / P for wide codes
  int n_wtiles;           // ceil(Lp / tpt)
  int n_tab_ctas;         // ceil(B*H_q / kTQ) * n_wtiles (0: no tables)
  int n_keys, n_begin, n_count, append_last;   // append: key kk -> (bh, j)
  int pdl;                // launched as a PDL dependent (griddepcontrol.wait first)
};

// 8 bf16 (one uint4) -> 8 fp64 with integer ops (exact for zero and normal
// numbers: sign | (exponent + 896) << 52 | mantissa << 45); any subnormal / inf /
// nan in the group goes through the exact fp32 path instead.
__device__ __forceinline__ void bf16x8_to_f64(const uint4 v, double* out, int stride) {
  const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
  bool special = false;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t mag = ((e & 1) ? (w4[e >> 1] >> 16) : w4[e >> 1]) & 0x7FFFu;
    special |= mag != 0u && (mag < 0x80u || mag >= 0x7F80u);
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t h = ((e & 1) ? (w4[e >> 1] >> 16) : w4[e >> 1]) & 0xFFFFu;
    const uint32_t mag = h & 0x7FFFu;
    double d;
    if (special) {
      d = (double)__uint_as_float(h << 16);
    } else {
      const uint32_t hi = ((h & 0x8000u) << 16) | (mag ? (mag << 13) + 0x38000000u : 0u);
      d = __hiloint2double((int)hi, 0);
    }
    out[e * stride] = d;
  }
}

// D(8x8) += A(8x4, row) B(4x8, col) in fp64 on the tensor cores (DMMA).
// Fragments: a = A[lane >> 2][lane & 3], b = B[lane & 3][lane >> 2],
// d{0,1} = D[lane >> 2][2 (lane & 3) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Wide codes (P > 8): the tables are not materialized (2^P entries per table);
// the score kernel's LUT image holds, per query head h and table l, the two
// factor half-tables of the exact product form (factorization):
//   A_h(e) = prod_{i < Pl} f_i(bit i of e),   B_h(e) = prod_{Pl <= i < P} f_i(bit i - Pl of e)
// (fp64 products in bit order, rounded once), so p_h(r) = A_h(r mod 2^Pl) B_h(r >> Pl)
// and T(r) = sum_h A_h B_h.  Image of a selection row: [h][half][E = 2^(P-Pl)][64 cols].
// The plain tables (socket_query_tables) are expanded from the same halves.
template <int NH>
__device__ __forceinline__ void wide_tables_epilogue(const ProArgs& a, const double* fx, int qv0,
                                                     int l0, int nqv) {
  const int P = a.P, L = a.L, Pl = P / 2, E = 1 << (P - Pl), R = 1 << P;
  const int tid = threadIdx.x;
  const size_t row_floats = (size_t)NH * 2 * E * 64;
  auto half_entry = [&](int m, int tl, int hi, int e) -> float {
    const int b0 = hi ? Pl : 0, nb = hi ? P - Pl : Pl;
    double p = 1.0;
    for (int i = 0; i < nb; ++i) p *= fx[((m * 16 + b0 + i) * 2 + ((e >> i) & 1)) * kFXS + tl];
    return (float)p;
  };
  if (a.lut) {   // one (vector, table, half) per task
    for (int task = tid; task < kTQ * a.tpt * 2; task += kPT) {
      const int hi = task & 1, tl = (task >> 1) % a.tpt, m = (task >> 1) / a.tpt;
      const int l = l0 + tl;
      if (qv0 + m >= nqv || l >= a.Lp) continue;
      const int nent = 1 << (hi ? P - Pl : Pl);
      float* img = a.lut + (size_t)((qv0 + m) / NH) * row_floats + (size_t)(((m % NH) * 2 + hi) * E) * 64;
      for (int e = 0; e < nent; ++e) {
        const float v = l < L ? half_entry(m, tl, hi, e) : 0.f;
        if (a.Lp >= 32) img[e * 64 + l] = v;
        else for (int cc = l; cc < 32; cc += a.Lp) img[e * 64 + cc] = v;
      }
    }
  }
  if (a.plain) {   // T(r) = sum_h A_h(r mod 2^Pl) B_h(r >> Pl), fp32 fma, h ascending
    constexpr int kRows = kTQ / NH;
    const long long n_ent = (long long)kRows * a.tpt * R;
    for (long long e = tid; e < n_ent; e += kPT) {
      const int r = (int)(e % R), tl = (int)((e / R) % a.tpt), srow = (int)(e / R / a.tpt);
      const int l = l0 + tl;
      if (qv0 + srow * NH >= nqv || l >= L) continue;
      float T = 0.f;
      for (int h = 0; h < NH; ++h) {
        const int m = srow * NH + h;
        T = fmaf(half_entry(m, tl, 0, r & ((1 << Pl) - 1)), half_entry(m, tl, 1, r >> Pl), T);
      }
      a.plain[((size_t)(qv0 / NH + srow) * L + l) * R + r] = T;
    }
  }
}

template <int NH>
__device__ __forceinline__ void tables_tile(const ProArgs& a, int qt, int wt, char* smem) {
  double* qs = reinterpret_cast<double*>(smem);    // [kD][kQS]
  double* ws = qs + kD * kQS;                      // [kD][kWS]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P = a.P, L = a.L, R = 1 << P;
  const int nqv = a.B * a.H_q;
  const int qv0 = qt * kTQ;
  const int l0 = wt * a.tpt;
  const int nw = (L - l0 < a.tpt ? L - l0 : a.tpt) * P;   // valid W rows of the tile (<= 0: padding)
  PRO_STAMP(0);
  PRO_STAMP(1);
  {   // stage q (16 vectors) and W (64 rows): all loads first, then convert
    constexpr int KW = 64 * 16 / kPT;          // W uint4 per thread
    uint4 vq, vw[KW];
    const int m = tid & 15, cq = (tid >> 4) & 15;
    vq = make_uint4(0, 0, 0, 0);
    if (tid < 256 && qv0 + m < nqv) vq = __ldg(reinterpret_cast<const uint4*>(a.q + (size_t)(qv0 + m) * kD) + cq);
#pragma unroll
    for (int k = 0; k < KW; ++k) {
      const int e = tid + k * kPT, w = e & 63, c = e >> 6;
      vw[k] = make_uint4(0, 0, 0, 0);
      if (w < nw) vw[k] = __ldg(reinterpret_cast<const uint4*>(a.W + (size_t)(l0 * P + w) * kD) + c);
    }
    if (tid < 256) bf16x8_to_f64(vq, qs + (cq * 8) * kQS + m, kQS);
#pragma unroll
    for (int k = 0; k < KW; ++k) {
      const int e = tid + k * kPT, w = e & 63, c = e >> 6;
      bf16x8_to_f64(vw[k], ws + (c * 8) * kWS + w, kWS);
    }
  }
  __syncthreads();
  PRO_STAMP(2);
  // X[m][w] = sum_t q_m[t] W_w[t]: warp w owns W rows 8 (w & 7) .. + 7 for both
  // 8-vector halves of the tile (two 8x8 fp64 accumulators) over the K half
  // w >> 3 (16 k-steps of 4); x = (K half 0) + (K half 1)
  double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
  const int nt8 = warp & 7, kh = warp >> 3;
  {
    const int kr = lane & 3, col = lane >> 2;
#pragma unroll 8
    for (int k0 = kh * (kD / 2); k0 < (kh + 1) * (kD / 2); k0 += 4) {
      const double* qrow = qs + (k0 + kr) * kQS;
      const double b = ws[(k0 + kr) * kWS + nt8 * 8 + col];
      dmma_8x8x4(c00, c01, qrow[col], b);
      dmma_8x8x4(c10, c11, qrow[8 + col], b);
    }
  }
  PRO_STAMP(3);
  __syncthreads();   // staging dead: the epilogue arrays reuse it
  double* fx = reinterpret_cast<double*>(smem);                         // [m][bit < 16][s][kFXS]
  float* half = reinterpret_cast<float*>(fx + kTQ * 16 * 2 * kFXS);    // [m][hi][ent][kTT]
  double* xs = reinterpret_cast<double*>(smem + 64 * 1024);             // [kh][m 16][w 64]
  {
    const int col = lane >> 2, q2 = 2 * (lane & 3);
    xs[(kh * 16 + col) * 64 + nt8 * 8 + q2] = c00;
    xs[(kh * 16 + col) * 64 + nt8 * 8 + q2 + 1] = c01;
    xs[(kh * 16 + 8 + col) * 64 + nt8 * 8 + q2] = c10;
    xs[(kh * 16 + 8 + col) * 64 + nt8 * 8 + q2 + 1] = c11;
  }
  __syncthreads();
  {   // sigma factors: 1024 projections over the 512 threads
    const float inv_sqrt_d = 0.08838834764831845f;   // 1/sqrt(128), correctly rounded
#pragma unroll
    for (int u = 0; u < kTQ * 64 / kPT; ++u) {
      const int e = tid + u * kPT, m = e >> 6, w = e & 63;
      const double xval = xs[m * 64 + w] + xs[(16 + m) * 64 + w];
      {
        if (w < nw) {
          const int tl = w / P, bit = w - tl * P;
          double fp, fm;
          if (a.hard) {            // Eq. 3: the product over bits is the indicator of b_q
            fp = xval >= 0.0 ? 1.0 : 0.0;                           // sign(0) = +1 (R-3)
            fm = 1.0 - fp;
          } else {
            const float uu = tanhf((float)xval) * inv_sqrt_d;       // Alg. 2 l.217
            const float av = 2.0f * uu / a.tau;                      // logit gap of bit i
            fp = (double)(1.0f / (1.0f + expf(-av)));                // c_{r,i} = +1 (bit set, R-5)
            fm = (double)(1.0f / (1.0f + expf(av)));                 // c_{r,i} = -1
          }
          fx[((m * 16 + bit) * 2 + 1) * kFXS + tl] = fp;
          fx[((m * 16 + bit) * 2 + 0) * kFXS + tl] = fm;
        }
      }
    }
  }
  __syncthreads();
  if (P > 8) {   // wide codes (NEXT-2): per-head factor half-tables, no group sum
    wide_tables_epilogue<NH>(a, fx, qv0, l0, nqv);
    PRO_STAMP(6);
    return;
  }
  PRO_STAMP(4);
  if (tid < kTQ * kTT * 2) {   // half tables: one (vector, table, half) per thread, ((f0 f1) f2) f3
    const int tl = tid & 7, hi = (tid >> 3) & 1, m = tid >> 4;
    double f[4][2];
#pragma unroll
    for (int bit = 0; bit < 4; ++bit) {
      const int ib = hi * 4 + bit;
      f[bit][0] = ib < P ? fx[((m * 16 + ib) * 2 + 0) * kFXS + tl] : 1.0;
      f[bit][1] = ib < P ? fx[((m * 16 + ib) * 2 + 1) * kFXS + tl] : 1.0;
    }
    double p01[4], p012[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) p01[e] = f[0][e & 1] * f[1][e >> 1];
#pragma unroll
    for (int e = 0; e < 8; ++e) p012[e] = p01[e & 3] * f[2][e >> 2];
    float* hrow = half + ((m * 2 + hi) * 16) * kTT + tl;
#pragma unroll
    for (int e = 0; e < 16; ++e) hrow[e * kTT] = (float)(p012[e & 7] * f[3][e >> 3]);
  }
  __syncthreads();
  PRO_STAMP(5);
  // LUT entries T(rr) = sum_h lo_h(rr & 15) hi_h(rr >> 4): task = (selection row,
  // LUT row rr, 4-table group), one float4 store of 4 consecutive columns
  constexpr int kRows = kTQ / NH;
  const int panels = a.Lp <= 64 ? 1 : (a.Lp + 63) / 64;
  // task = (selection row, 4-row quarter lq of the 16 low-half entries, high-half
  // entry hi, table group g4): its 4 LUT rows rr = 16 hi + 4 lq + u share the hi
  // factors (one 16-B load per head) and a warp's lo loads are broadcasts
  for (int task = tid; task < kRows * 4 * 16 * 2; task += kPT) {
    const int g4 = task & 1, hi = (task >> 1) & 15, lq = (task >> 5) & 3, srow = task >> 7;
    const int row = qv0 / NH + srow;
    const int lb = l0 + 4 * g4;
    if (qv0 + srow * NH >= nqv || lb >= a.Lp) continue;
    float4 hv[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h)
      hv[h] = *reinterpret_cast<const float4*>(half + (((srow * NH + h) * 2 + 1) * 16 + hi) * kTT + 4 * g4);
    float* lrow = a.lut ? a.lut + (size_t)row * panels * (256 * 64) : nullptr;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int rr = hi * 16 + lq * 4 + u;
      float4 T = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rr < R) {
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const float4 lo = *reinterpret_cast<const float4*>(half + (((srow * NH + h) * 2 + 0) * 16 + (rr & 15)) * kTT + 4 * g4);
          T.x = fmaf(lo.x, hv[h].x, T.x);
          T.y = fmaf(lo.y, hv[h].y, T.y);
          T.z = fmaf(lo.z, hv[h].z, T.z);
          T.w = fmaf(lo.w, hv[h].w, T.w);
        }
        // tables >= L are padding: 0
        if (lb + 0 >= L) T.x = 0.f;
        if (lb + 1 >= L) T.y = 0.f;
        if (lb + 2 >= L) T.z = 0.f;
        if (lb + 3 >= L) T.w = 0.f;
        if (a.plain) {
          const float tv[4] = {T.x, T.y, T.z, T.w};
#pragma unroll
          for (int v = 0; v < 4; ++v)
            if (lb + v < L) a.plain[((size_t)row * L + lb + v) * R + rr] = tv[v];
        }
      }
      if (lrow) {
        if (a.Lp >= 32) {
          *reinterpret_cast<float4*>(lrow + (size_t)(lb >> 6) * (256 * 64) + rr * 64 + (lb & 63)) = T;
        } else {
          const float tv[4] = {T.x, T.y, T.z, T.w};
#pragma unroll
          for (int v = 0; v < 4; ++v)
            if (lb + v < a.Lp)
              for (int cc = lb + v; cc < 32; cc += a.Lp) lrow[rr * 64 + cc] = tv[v];
        }
      }
    }
  }
  PRO_STAMP(6);
}

__device__ __forceinline__ void append_tile(const ProArgs& a, int at, int wt, char* smem) {
  float* ks = reinterpret_cast<float*>(smem);      // [kD][kKS]
  float* ws = ks + kD * kKS;                       // [kD][kAWS]
  uint8_t* bits = reinterpret_cast<uint8_t*>(ws + kD * kAWS);   // [kAK][64]
  int* kj = reinterpret_cast<int*>(bits + kAK * 64);            // [kAK] j (-1: no key)
  int* kbh = kj + kAK;                                           // [kAK] bh
  const int tid = threadIdx.x;
  const int P = a.P, L = a.L;
  const int l0 = wt * a.tpt;
  const int nw = (L - l0 < a.tpt ? L - l0 : a.tpt) * P;
  PRO_STAMP(0);
  PRO_STAMP(1);
  {   // stage W first (independent of the keys): 64 rows x 16 uint4
    constexpr int KW = 64 * 16 / kPT;
    uint4 vw[KW];
#pragma unroll
    for (int k = 0; k < KW; ++k) {
      const int e = tid + k * kPT, w = e & 63, c = e >> 6;
      vw[k] = make_uint4(0, 0, 0, 0);
      if (w < nw) vw[k] = __ldg(reinterpret_cast<const uint4*>(a.W + (size_t)(l0 * P + w) * kD) + c);
    }
#pragma unroll
    for (int k = 0; k < KW; ++k) {
      const int e = tid + k * kPT, w = e & 63, c = e >> 6;
      const uint32_t w4[4] = {vw[k].x, vw[k].y, vw[k].z, vw[k].w};
#pragma unroll
      for (int e2 = 0; e2 < 8; ++e2)
        ws[(c * 8 + e2) * kAWS + w] = (e2 & 1) ? bf16hi(w4[e2 >> 1]) : bf16lo(w4[e2 >> 1]);
    }
  }
  if (tid < kAK) {
    const int kk = at * kAK + tid;
    int j = -1, bh = 0;
    if (kk < a.n_keys) {
      bh = kk / a.n_count;
      j = a.n_begin + kk % a.n_count;
      if (a.append_last) {               // decode step: the newest key j = seq_lens[b] - 1
        const int n = a.seq_lens[bh / a.H_kv];
        j = (n > 0 && n <= a.N_max) ? n - 1 : -1;   // a cache that outgrew N_max: no write
      }
    }
    kj[tid] = j;
    kbh[tid] = bh;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32 * 16 / kPT; ++k) {   // stage keys: 32 rows x 16 uint4
    const int e = tid + k * kPT, m = e & 31, c = e >> 5;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (kj[m] >= 0) {
      if (a.k_new) {   // the new row comes from k_new; the first table tile also fills the cache
        v = __ldg(reinterpret_cast<const uint4*>(a.k_new + (size_t)kbh[m] * kD) + c);
        if (wt == 0) {
          reinterpret_cast<uint4*>(a.K_w + ((size_t)kbh[m] * a.N_max + kj[m]) * kD)[c] = v;
          reinterpret_cast<uint4*>(a.V_w + ((size_t)kbh[m] * a.N_max + kj[m]) * kD)[c] =
              __ldg(reinterpret_cast<const uint4*>(a.v_new + (size_t)kbh[m] * kD) + c);
        }
      } else {
        v = __ldg(reinterpret_cast<const uint4*>(a.K + ((size_t)kbh[m] * a.N_max + kj[m]) * kD) + c);
      }
    }
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e2 = 0; e2 < 8; ++e2)
      ks[(c * 8 + e2) * kKS + m] = (e2 & 1) ? bf16hi(w4[e2 >> 1]) : bf16lo(w4[e2 >> 1]);
  }

  __syncthreads();
  PRO_STAMP(2);
  // keys 2kp, 2kp+1 x W rows 4wq .. 4wq+3 (threads >= 256 idle here), t ascending
  const int kp = tid & 15, wq = (tid >> 4) & 15;
  float x[2][4] = {};
#pragma unroll 8
  for (int t = 0; t < (tid < 256 ? kD : 0); ++t) {
    const float2 kv = *reinterpret_cast<const float2*>(ks + t * kKS + 2 * kp);
    const float4 wv = *reinterpret_cast<const float4*>(ws + t * kAWS + 4 * wq);
    x[0][0] = fmaf(wv.x, kv.x, x[0][0]); x[0][1] = fmaf(wv.y, kv.x, x[0][1]);
    x[0][2] = fmaf(wv.z, kv.x, x[0][2]); x[0][3] = fmaf(wv.w, kv.x, x[0][3]);
    x[1][0] = fmaf(wv.x, kv.y, x[1][0]); x[1][1] = fmaf(wv.y, kv.y, x[1][1]);
    x[1][2] = fmaf(wv.z, kv.y, x[1][2]); x[1][3] = fmaf(wv.w, kv.y, x[1][3]);
  }
  PRO_STAMP(3);
  if (tid < 256) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int w = 4 * wq + j;
        bits[(2 * kp + i) * 64 + w] = (w < nw && x[i][j] >= 0.f) ? 1 : 0;   // sign(0) = +1 (R-3)
      }
  }
  __syncthreads();
  {   // code byte of (key m, table tl): row i -> bit i (R-4)
    const int m = (tid >> 3) & 31, tl = tid & 7;
    const int l = l0 + tl, j = kj[m];
    if (tid < 256 && j >= 0 && tl < a.tpt && l < a.Lp) {
      uint32_t code = 0;
      for (int i = 0; i < P; ++i) code |= (uint32_t)bits[m * 64 + tl * P + i] << i;
      const int Lp = a.Lp;
      const int M = (Lp < 32 ? Lp : 32) - 1;
      const int s = (l & ~M) | ((l - j) & M);
      if (P > 8) {
        // packed wide codes: the slot's P bits in one or two words; other tiles'
        // CTAs write other slots of the same words, so clear and set only mine
        // with atomics (disjoint bit sets: the order does not matter)
        const int G = Lp >> 5, g = s >> 5, bp = (s & 31) * P, w = bp >> 5, sh = bp & 31;
        uint32_t* cw = reinterpret_cast<uint32_t*>(a.codes) + (size_t)kbh[m] * a.N_max * Lp * P / 32;
        const uint32_t fm = (1u << P) - 1u;
        uint32_t* w0 = cw + packed_word(j, g, w, G, P);
        atomicAnd(w0, ~(fm << sh));
        atomicOr(w0, code << sh);
        if (sh + P > 32) {
          uint32_t* w1 = cw + packed_word(j, g, w + 1, G, P);
          atomicAnd(w1, ~(fm >> (32 - sh)));
          atomicOr(w1, code >> (32 - sh));
        }
      } else {
        a.codes[(size_t)kbh[m] * a.N_max * Lp + code_off(j, s, Lp)] = (uint8_t)code;
      }
    }
  }
  if (a.V && wt == 0 && tid < 256) {   // ||v_j||: warp w handles keys 4w .. 4w+3
    const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int m = warp * 4 + r, j = kj[m];
      if (j < 0) continue;
      const uint2 u = a.v_new ? *reinterpret_cast<const uint2*>(a.v_new + (size_t)kbh[m] * kD + lane * 4)
                              : *reinterpret_cast<const uint2*>(a.V + ((size_t)kbh[m] * a.N_max + j) * kD + lane * 4);
      float va = bf16lo(u.x), vb = bf16hi(u.x), vc = bf16lo(u.y), vd = bf16hi(u.y);
      float sq = fmaf(va, va, fmaf(vb, vb, fmaf(vc, vc, vd * vd)));
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
      if (lane == 0) a.vnorm[(size_t)kbh[m] * a.N_max + j] = sqrtf(sq);
    }
  }
  PRO_STAMP(6);
}

// Host: fill the shape fields of a ProArgs from cfg (tables: B*H_q query
// vectors when lut/plain set; append: n_keys keys) and launch prologue_kernel
// (defined in step.cu).
socket_status launch_prologue(const socket_cfg& c, ProArgs a, bool tables, cudaStream_t st);

template <int NH>
__global__ void __launch_bounds__(kPT, 2) prologue_kernel(ProArgs a) {
  extern __shared__ __align__(16) char psm[];
  if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: staged inputs
  if (blockIdx.x == 0 && a.tickets)
    for (int i = threadIdx.x; i < a.n_tickets; i += blockDim.x) a.tickets[i] = 0;
  if ((int)blockIdx.x < a.n_tab_ctas) {
    tables_tile<NH>(a, blockIdx.x / a.n_wtiles, blockIdx.x % a.n_wtiles, psm);
  } else {
    const int t = (int)blockIdx.x - a.n_tab_ctas;
    append_tile(a, t / a.n_wtiles, t % a.n_wtiles, psm);
  }
}

}  // namespace sk
