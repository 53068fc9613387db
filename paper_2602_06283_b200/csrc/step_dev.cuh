// Device routines shared by several kernels of libsocket_b200 (not part of the ABI).
#pragma once
#include "internal.cuh"

namespace sk {

constexpr int kTabThreads = 512;
constexpr int kTabPerCta = 16;    // tables per CTA
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

// One CTA = (b, selection row) x kTabPerCta tables.  Steps:
//  1+2. in round i, warp w owns the 4 W rows 4 (16 i + w) .. + 3.
//       A lane holds 4 elements (t = 4 lane .. 4 lane + 3) of every head's q and
//       of the W rows as fp64, so each of the 4*NH projections x = W_i . q_h is
//       4 fp64 FMAs per lane; a reduce-scatter over the warp leaves every lane
//       with one complete x.  bf16 x bf16 products and their partial sums are
//       exact in fp64, so x is exact.  Each lane then evaluates its
//       u = tanh(x)/sqrt(d) and sigma(+-2u/tau) with the accurate fp32
//       functions (<= 2 ulp each).
//  3.   half tables lo(r & 15) = prod_{i<4} f_i, hi(r >> 4) = prod_{i>=4} f_i
//       in fp64, rounded once to fp32;
//  4.   T(r) = sum_h lo_h * hi_h; consecutive threads write consecutive table
//       columns of one LUT row.
template <int NH>
struct TablesSmem {
  double fx[NH][kTabPerCta][8][2];                // sigma factors
  float half_lo[NH][16][kTabPerCta];
  float half_hi[NH][16][kTabPerCta];
};

template <int NH>
__device__ __forceinline__ void tables_cta(const uint16_t* __restrict__ q,
                                           const uint16_t* __restrict__ W, float* __restrict__ plain,
                                           float* __restrict__ lut, int H_q, int H_sel, int L, int P,
                                           int Lp, float tau, int row, int l0, TablesSmem<NH>& S) {
  constexpr int kWarps = kTabThreads / 32;
  constexpr int kRounds = (kTabPerCta * 8) / (4 * kWarps);   // 4 W rows per warp per round
  static_assert(kRounds * 4 * kWarps == kTabPerCta * 8, "W rows must tile the warps");
  constexpr int NV = 4 * NH;                                 // values per warp and round
  auto& fx = S.fx;
  auto& half_lo = S.half_lo;
  auto& half_hi = S.half_hi;
  const int b = row / H_sel, r = row % H_sel;
  const int h0 = (NH == 1) ? r : r * NH;     // first query head of the row
  const int R = 1 << P;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // W rows are enumerated as wr = 8 * tl + i (bit i < 8, rows with i >= P skipped)
  double qd[NH][4];
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const uint2 u = *reinterpret_cast<const uint2*>(q + ((size_t)b * H_q + h0 + h) * kD + lane * 4);
    qd[h][0] = bf16lo(u.x); qd[h][1] = bf16hi(u.x); qd[h][2] = bf16lo(u.y); qd[h][3] = bf16hi(u.y);
  }
  uint2 wu[kRounds][4];
#pragma unroll
  for (int round = 0; round < kRounds; ++round)
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int wr = (round * kWarps + warp) * 4 + rr;
      const int l = l0 + (wr >> 3), i = wr & 7;
      wu[round][rr] = make_uint2(0, 0);
      if (i < P && l < L) wu[round][rr] = *reinterpret_cast<const uint2*>(W + ((size_t)l * P + i) * kD + lane * 4);
    }
#pragma unroll
  for (int round = 0; round < kRounds; ++round) {
    double v[NV];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const double w0 = bf16lo(wu[round][rr].x), w1 = bf16hi(wu[round][rr].x);
      const double w2 = bf16lo(wu[round][rr].y), w3 = bf16hi(wu[round][rr].y);
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        double x = w0 * qd[h][0];
        x = fma(w1, qd[h][1], x);
        x = fma(w2, qd[h][2], x);
        v[rr * NH + h] = fma(w3, qd[h][3], x);
      }
    }
    // reduce-scatter over the 32 lanes: afterwards v[0] holds the full sum of
    // value `own` (lanes with equal `own` hold equal sums)
    int own = 0, nv = NV;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      if (nv > 1) {
        const int hnv = nv >> 1;
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < NV / 2; ++i) {
          if (i < hnv) {
            const double send = up ? v[i] : v[i + hnv];
            const double keep = up ? v[i + hnv] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
        if (up) own += hnv;
        nv = hnv;
      } else {
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
      }
    }
    const int rr = own / NH, h = own % NH;          // NH is a power of two
    const int wr = (round * kWarps + warp) * 4 + rr;
    const int tl = wr >> 3, i = wr & 7;
    const float inv_sqrt_d = 0.08838834764831845f;   // 1/sqrt(128), correctly rounded
    const float uu = tanhf((float)v[0]) * inv_sqrt_d;  // Alg. 2 l.217
    const float a = 2.0f * uu / tau;                   // logit gap of bit i
    const float fp = 1.0f / (1.0f + expf(-a));         // c_{r,i} = +1 (bit set)
    const float fm = 1.0f / (1.0f + expf(a));          // c_{r,i} = -1
    if ((lane & (32 / NV - 1)) == 0 && i < P) {
      fx[h][tl][i][1] = (double)fp;
      fx[h][tl][i][0] = (double)fm;
    }
  }
  __syncthreads();
  // 3. half tables (bits 0..3 and 4..P-1; an empty product is 1)
  for (int i = tid; i < NH * kTabPerCta * 32; i += kTabThreads) {  // NH is a template constant
    const int e = i & 15, hi = (i >> 4) & 1, tl = (i >> 5) % kTabPerCta, h = i / (32 * kTabPerCta);
    double p = 1.0;
#pragma unroll
    for (int bit = 0; bit < 4; ++bit) {
      const int ib = hi * 4 + bit;
      if (ib < P) p *= fx[h][tl][ib][(e >> bit) & 1];
    }
    if (hi) half_hi[h][e][tl] = (float)p; else half_lo[h][e][tl] = (float)p;
  }
  __syncthreads();
  // 4. entries: thread -> (row rr, table tl) with tl fastest
  const int panels = Lp <= 64 ? 1 : (Lp + 63) / 64;
  float* lrow = lut ? lut + (size_t)row * panels * (256 * 64) : nullptr;
  for (int e = tid; e < 256 * kTabPerCta; e += kTabThreads) {
    const int tl = e % kTabPerCta, rr = e / kTabPerCta;
    const int l = l0 + tl;
    if (l >= Lp) continue;
    float T = 0.f;
    if (l < L && rr < R) {
      for (int h = 0; h < NH; ++h) T = fmaf(half_lo[h][rr & 15][tl], half_hi[h][rr >> 4][tl], T);
      if (plain) plain[((size_t)row * L + l) * R + rr] = T;
    }
    if (lrow) {
      if (Lp >= 32) {
        lrow[(size_t)(l >> 6) * (256 * 64) + rr * 64 + (l & 63)] = T;
      } else {
        for (int cc = l; cc < 32; cc += Lp) lrow[rr * 64 + cc] = T;
      }
    }
  }
}

// Append path (decode step: n_count new keys per (b, kv-head), typically 1).
// One warp per (key, table): lane t holds elements 4t .. 4t+3 of the key, the
// P projections are 4 FMAs per lane each (t ascending within the lane) and a
// butterfly sum; lane 0 writes the code byte to slot s = (l & ~M) | ((l - j) & M)
// of key j (inverse of slot_table).  Warps with table 0 also write ||v_j||
// with exactly vnorm_kernel's summation order.  With append_last, key j is
// seq_lens[b] - 1 of each (b, kv head) (skipped for empty sequences).
// Note: the projection's summation order differs from the prefill kernels, so
// a bit whose projection is within fp32 rounding of 0 may differ between the
// paths; all are checked against the fp64 oracle with the same margin rule.
__device__ __forceinline__ void append_warp_job(
    const uint16_t* __restrict__ K, const uint16_t* __restrict__ W, uint8_t* __restrict__ codes,
    const uint16_t* __restrict__ V, float* __restrict__ vnorm, int N_max, int L, int P, int Lp,
    int n_begin, int n_count, int total_keys, int append_last, const int32_t* __restrict__ seq_lens,
    int H_kv, int job, int lane) {
  if (job >= total_keys * Lp) return;
  const int key = job / Lp, l = job % Lp;
  const int bh = key / n_count;
  int j = n_begin + key % n_count;
  if (append_last) {                      // decode step: the newest key j = seq_lens[b] - 1
    const int n = seq_lens[bh / H_kv];
    if (n <= 0) return;
    j = n - 1;
  }
  uint32_t code = 0;
  if (l < L) {
    const uint2 ku = *reinterpret_cast<const uint2*>(K + ((size_t)bh * N_max + j) * kD + lane * 4);
    const float k0 = bf16lo(ku.x), k1 = bf16hi(ku.x), k2 = bf16lo(ku.y), k3 = bf16hi(ku.y);
    uint2 wall[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)    // all W rows of the table in flight at once
      wall[i] = i < P ? *reinterpret_cast<const uint2*>(W + ((size_t)l * P + i) * kD + lane * 4)
                      : make_uint2(0, 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i >= P) break;
      const uint2 wu = wall[i];
      float x = bf16lo(wu.x) * k0;
      x = fmaf(bf16hi(wu.x), k1, x);
      x = fmaf(bf16lo(wu.y), k2, x);
      x = fmaf(bf16hi(wu.y), k3, x);
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      code |= (x >= 0.f ? 1u : 0u) << i;     // sign(0) = +1 (R-3), LSB = row 0 (R-4)
    }
  }
  if (lane == 0) {
    const int M = (Lp < 32 ? Lp : 32) - 1;
    const int s = (l & ~M) | ((l - j) & M);
    codes[(size_t)bh * N_max * Lp + code_off(j, s, Lp)] = (uint8_t)code;
  }
  if (V && l == 0) {
    const uint2 u = *reinterpret_cast<const uint2*>(V + ((size_t)bh * N_max + j) * kD + lane * 4);
    float a = bf16lo(u.x), b = bf16hi(u.x), c = bf16lo(u.y), e = bf16hi(u.y);
    float sq = fmaf(a, a, fmaf(b, b, fmaf(c, c, e * e)));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) vnorm[(size_t)bh * N_max + j] = sqrtf(sq);
  }
}

}  // namespace sk
