// Alg. 2 SoftBucketProbs and Eq. 4 / Alg. 4 soft
// collision scoring (l.183-188, l.1485-1506).
//
// query_tables_kernel: per (b, selection row) builds T^(l)(r) for all tables:
//   u_{l,i} = tanh(W^(l)_i . q) / sqrt(d),  p(r) = prod_i sigma(2 u_i c_{r,i} / tau)
//   (exact product form of the corner softmax), summed over the group's query
//   heads in KV_SHARED mode.  It writes the plain [L][R] tables and/or the
//   score kernel's shared-memory image ("LUT"): panels of [256 rows][64 cols]
//   fp32 where column c holds table c (Lp >= 32) or table c mod Lp (Lp < 32).
//
// score_reg_kernel: streams the tiled codes with 128-bit loads, lane = key j mod
// 32.  At slot step s lane l reads LUT column (s & 32) | ((s + l) & 31), so the
// 32 lanes hit 32 distinct banks (conflict-free).
#include "step_dev.cuh"
#include "score_dev.cuh"

namespace sk {


socket_status launch_query_tables(const socket_cfg& c, const void* q, const void* W,
                                  float* plain, float* lut, cudaStream_t st) {
  ProArgs a = {};
  a.q = (const uint16_t*)q;
  a.W = (const uint16_t*)W;
  a.plain = plain;
  a.lut = lut;
  return launch_prologue(c, a, true, st);
}

// ----------------------------------------------------------------------------
// score kernel
// ----------------------------------------------------------------------------
constexpr int kScoreThreads = 512;            // 16 warps, one CTA per SM (persistent)
constexpr int kScoreWarps = kScoreThreads / 32;

// ----------------------------------------------------------------------------
// wide-code score kernels (P > 8, NEXT-2).  Codes are tightly packed: per key
// and 32-slot group, one 32P-bit string (P u32 words, word-interleaved across
// the tile's keys; internal.cuh packed_word) -- 600 useful of 640 stored bits
// per key at the RULER setting L = 60, P = 10.  The LUT image holds per head
// the factor half-tables A_h (low Pl bits) and B_h (high P - Pl bits) of the
// exact product form p_h(r) = A_h(r mod 2^Pl) B_h(r >> Pl).
// ----------------------------------------------------------------------------
constexpr int kWideThreads = 512;
constexpr int kWideTilesPerCta = 256;

// the P-bit code of slot sl of a group string w[0..P), placed at bit `dst`
// (sl, P, dst compile-time after unrolling: one funnel shift, or a shift)
template <int P>
__device__ __forceinline__ uint32_t slot_bits(const uint32_t (&w)[P], int sl, int dst) {
  const int r = sl * P - dst;
  if (r < 0) return w[0] << (-r);
  const int i = r >> 5, sh = r & 31;
  const uint32_t hi = (i + 1 < P) ? w[i + 1 < P ? i + 1 : P - 1] : 0u;
  return sh == 0 ? w[i] : __funnelshift_r(w[i], hi, sh);
}

// P = 11..16 (and any group size): every slot and head adds A_h[lo] * B_h[hi]
//   w_hat(j) = sum_s sum_h A_h[l(s)](lo) * B_h[l(s)](hi)   (fp32 fma, s then h ascending)
// One CTA = (selection row, 256-tile chunk); lane = key, bank-rotated column
// c(s, lane) = (s & 32) | ((s + lane) & 31) as the byte-code kernel.
template <int NH, int P>
__global__ void __launch_bounds__(kWideThreads, 1)
score_wide_kernel(const float* __restrict__ lut_g, const uint32_t* __restrict__ codes,
                  const float* __restrict__ vnorm, const int32_t* __restrict__ seq_lens,
                  const uint8_t* __restrict__ mask, float* __restrict__ scores, int H_sel, int H_kv,
                  int G_sel, int N_max, int Lp, int E, int row_floats, long long index_base) {
  extern __shared__ __align__(16) float wlut[];
  constexpr int Pl = P / 2;
  constexpr uint32_t lomask = (1u << Pl) - 1u, fmask = (1u << P) - 1u;
  const int row = blockIdx.y;
  const int b = row / H_sel, r = row % H_sel, g = r / G_sel;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t pol_code = l2_policy_evict_first();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const float4* src = reinterpret_cast<const float4*>(lut_g + (size_t)row * row_floats);
  for (int i = threadIdx.x; i < row_floats / 4; i += kWideThreads)
    reinterpret_cast<float4*>(wlut)[i] = src[i];
  __syncthreads();
  const int n = local_len(seq_lens[b], index_base, N_max);
  const int G = Lp >> 5;
  const int tiles = N_max >> 5;
  const int t0 = blockIdx.x * kWideTilesPerCta;
  const int t1 = min(t0 + kWideTilesPerCta, tiles);
  const uint32_t* crow = codes + ((size_t)b * H_kv + g) * (size_t)N_max * Lp * P / 32;
  const float* vrow = vnorm + ((size_t)b * H_kv + g) * N_max;
  const uint8_t* mrow = mask ? mask + (size_t)b * N_max : nullptr;
  float* srow = scores + (size_t)row * N_max;
  for (int ti = t0 + warp; ti < t1; ti += kWideThreads / 32) {
    const int j = ti * 32 + lane;
    if (ti * 32 >= n) {                       // whole tile past seq_len
      srow[j] = -INFINITY;
      continue;
    }
    float acc = 0.f;
    for (int gi = 0; gi < G; ++gi) {
      uint32_t w[P];
#pragma unroll
      for (int wd = 0; wd < P; ++wd) w[wd] = ldg_nc_u32_hint(crow + packed_word(j, gi, wd, G, P), pol_code);
#pragma unroll
      for (int sl = 0; sl < 32; ++sl) {
        const uint32_t code = slot_bits<P>(w, sl, 0) & fmask;
        const int col = gi * 32 + ((sl + lane) & 31);
        const int lo = (int)(code & lomask), hi = (int)(code >> Pl);
#pragma unroll
        for (int h = 0; h < NH; ++h)
          acc = fmaf(wlut[((h * 2) * E + lo) * 64 + col], wlut[((h * 2 + 1) * E + hi) * 64 + col], acc);
      }
    }
    const bool ok = j < n && (!mrow || mrow[j]);
    srow[j] = ok ? vrow[j] * acc : -INFINITY;
  }
}

// Large half-table images (KV_SHARED at P >= 13: the row's image [NH][2][E][64]
// exceeds shared memory): the same arithmetic tiled over (32-slot group g, head
// chunk of NHC heads), i.e. sub-images [NHC][2][E][32] of <= 128 KB, one pass
// over the CTA's keys per tile; a key's partial sum is parked in `scores`
// between passes (the same thread owns the key in every pass) and the last
// pass multiplies by ||v_j|| and applies the mask.
template <int NHC, int P>
__global__ void __launch_bounds__(kWideThreads, 1)
score_wide_tiled_kernel(const float* __restrict__ lut_g, const uint32_t* __restrict__ codes,
                        const float* __restrict__ vnorm, const int32_t* __restrict__ seq_lens,
                        const uint8_t* __restrict__ mask, float* __restrict__ scores, int H_sel, int H_kv,
                        int G_sel, int N_max, int Lp, int NH, int E, int row_floats, long long index_base) {
  extern __shared__ __align__(16) float wsub[];   // [NHC][2][E][32]
  constexpr int Pl = P / 2;
  constexpr uint32_t lomask = (1u << Pl) - 1u, fmask = (1u << P) - 1u;
  const int row = blockIdx.y;
  const int b = row / H_sel, r = row % H_sel, g = r / G_sel;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t pol_code = l2_policy_evict_first();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n = local_len(seq_lens[b], index_base, N_max);
  const int G = Lp >> 5;
  const int tiles = N_max >> 5;
  const int t0 = blockIdx.x * kWideTilesPerCta;
  const int t1 = min(t0 + kWideTilesPerCta, tiles);
  const uint32_t* crow = codes + ((size_t)b * H_kv + g) * (size_t)N_max * Lp * P / 32;
  const float* vrow = vnorm + ((size_t)b * H_kv + g) * N_max;
  const uint8_t* mrow = mask ? mask + (size_t)b * N_max : nullptr;
  float* srow = scores + (size_t)row * N_max;
  const float* img = lut_g + (size_t)row * row_floats;
  const int nchunks = NH / NHC;
  const int npass = G * nchunks;
  for (int pass = 0; pass < npass; ++pass) {
    const int gi = pass / nchunks, hc = pass % nchunks;
    __syncthreads();                                    // previous pass done with wsub
    for (int e = threadIdx.x; e < NHC * 2 * E * 32; e += kWideThreads) {
      const int col = e & 31, ent = (e >> 5) % E, half = (e / (32 * E)) & 1, h = e / (64 * E);
      wsub[e] = img[(((hc * NHC + h) * 2 + half) * E + ent) * 64 + gi * 32 + col];
    }
    __syncthreads();
    const bool first = pass == 0, last = pass + 1 == npass;
    for (int ti = t0 + warp; ti < t1; ti += kWideThreads / 32) {
      const int j = ti * 32 + lane;
      if (ti * 32 >= n) {                               // whole tile past seq_len
        if (last) srow[j] = -INFINITY;
        continue;
      }
      uint32_t w[P];
#pragma unroll
      for (int wd = 0; wd < P; ++wd) w[wd] = ldg_nc_u32_hint(crow + packed_word(j, gi, wd, G, P), pol_code);
      float acc = first ? 0.f : srow[j];
#pragma unroll
      for (int sl = 0; sl < 32; ++sl) {
        const uint32_t code = slot_bits<P>(w, sl, 0) & fmask;
        const int col = (sl + lane) & 31;
        const int lo = (int)(code & lomask), hi = (int)(code >> Pl);
#pragma unroll
        for (int h = 0; h < NHC; ++h)
          acc = fmaf(wsub[((h * 2) * E + lo) * 32 + col], wsub[((h * 2 + 1) * E + hi) * 32 + col], acc);
      }
      if (!last) {
        srow[j] = acc;
      } else {
        const bool ok = j < n && (!mrow || mrow[j]);
        srow[j] = ok ? vrow[j] * acc : -INFINITY;
      }
    }
  }
}

// Wide codes with P <= 10: per 32-slot group (= 32 tables, the rotation
// group), the group-summed tables T_l(r) = sum_h A_h,l(r mod 2^Pl)
// B_h,l(r >> Pl) are materialized in shared memory ([2^P][32] fp32, <= 128 KB)
// from the half-table image, so a lookup is one conflict-free LDS as in the
// byte-code kernel; the CTA sweeps its keys once per group, keeping the first
// group's partial sums in `scores` (read back by the same thread).  A lookup's
// byte offset is a funnel shift of the packed words that lands the code at
// bit 7 (row stride 128 B) and one LOP3 with the lane's column offset.
template <int NH, int P>
__global__ void __launch_bounds__(kWideThreads, 1)
score_wide2_kernel(const float* __restrict__ lut_g, const uint32_t* __restrict__ codes,
                   const float* __restrict__ vnorm, const int32_t* __restrict__ seq_lens,
                   const uint8_t* __restrict__ mask, float* __restrict__ scores, int H_sel, int H_kv,
                   int G_sel, int N_max, int Lp, int E, int row_floats, long long total_tiles,
                   long long index_base) {
  extern __shared__ __align__(16) float w2[];
  constexpr int R = 1 << P, Pl = P / 2, RL = 1 << Pl;
  constexpr uint32_t amask = (uint32_t)(R - 1) << 7;
  float* tab = w2;                          // [R][32]
  const char* tabc = reinterpret_cast<const char*>(w2);
  float* ast = tab + R * 32;                // [NH][RL][32] staged A half-tables of the group
  float* bst = ast + NH * RL * 32;          // [NH][EH][32] staged B half-tables of the group
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t lane4 = 4u * lane;
  const uint64_t pol_code = l2_policy_evict_first(), pol_score = l2_policy_evict_last();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int tiles_per_row = N_max >> 5;
  const long long tb = total_tiles * blockIdx.x / gridDim.x;
  const long long te = total_tiles * (blockIdx.x + 1) / gridDim.x;
  const int groups = Lp / 32;
  const int EH = R / RL;                    // entries of the high half
  for (long long t = tb; t < te;) {         // persistent: one row segment at a time
    const int row = (int)(t / tiles_per_row);
    const long long seg_end = min(te, (long long)(row + 1) * tiles_per_row);
    const int t0 = (int)(t - (long long)row * tiles_per_row);
    const int t1 = (int)(seg_end - (long long)row * tiles_per_row);
    t = seg_end;
    const int b = row / H_sel, r = row % H_sel, g = r / G_sel;
    const int n = local_len(seq_lens[b], index_base, N_max);
    const uint32_t* crow = codes + ((size_t)b * H_kv + g) * (size_t)N_max * Lp * P / 32;
    const float* vrow = vnorm + ((size_t)b * H_kv + g) * N_max;
    const uint8_t* mrow = mask ? mask + (size_t)b * N_max : nullptr;
    float* srow = scores + (size_t)row * N_max;
    const float* img = lut_g + (size_t)row * row_floats;
    const int vt1 = min(t1, (n + 31) >> 5);   // tiles with valid keys
    for (int gi = 0; gi < groups; ++gi) {
      if (t0 >= vt1) break;
      __syncthreads();                        // previous sweep done with tab / ast / bst
      // stage the group's A and B half-tables (float4 loads, all in flight)
      for (int e4 = tid; e4 < NH * (RL + EH) * 8; e4 += kWideThreads) {
        const int c4 = e4 & 7, ent = (e4 >> 3) % (RL + EH), h = e4 / (8 * (RL + EH));
        const bool hiv = ent >= RL;
        const float4 v = __ldg(reinterpret_cast<const float4*>(
            img + ((h * 2 + (hiv ? 1 : 0)) * E + (hiv ? ent - RL : ent)) * 64 + gi * 32) + c4);
        float* dst = hiv ? bst + (h * EH + ent - RL) * 32 : ast + (h * RL + ent) * 32;
        reinterpret_cast<float4*>(dst)[c4] = v;
      }
      __syncthreads();
      // T_l(hi, lo) = sum_h A_h(lo) B_h(hi) (fp32 fma, h ascending): thread = (column,
      // 8-row block of lo, block of hi), its A / B values in registers
      {
        constexpr int BL = RL >= 8 ? 8 : RL;              // lo rows per thread
        constexpr int NBL = RL / BL;                      // lo blocks
        constexpr int NBH = kWideThreads / 32 / NBL;      // hi blocks over the 16 warps
        const int col = tid & 31, blo = (tid >> 5) % NBL, bhb = (tid >> 5) / NBL;
        const int hb1 = min(EH, (bhb + 1) * ((EH + NBH - 1) / NBH));
        for (int hb = bhb * ((EH + NBH - 1) / NBH); hb < hb1; hb += 8) {
          const int nh8 = min(8, hb1 - hb);
          float av[NH][BL];
#pragma unroll
          for (int h = 0; h < NH; ++h)
#pragma unroll
            for (int u = 0; u < BL; ++u) av[h][u] = ast[(h * RL + blo * BL + u) * 32 + col];
          for (int v8 = 0; v8 < nh8; ++v8) {
            const int hi = hb + v8;
            float bv[NH];
#pragma unroll
            for (int h = 0; h < NH; ++h) bv[h] = bst[(h * EH + hi) * 32 + col];
#pragma unroll
            for (int u = 0; u < BL; ++u) {
              float T = 0.f;
#pragma unroll
              for (int h = 0; h < NH; ++h) T = fmaf(av[h][u], bv[h], T);
              tab[(hi * RL + blo * BL + u) * 32 + col] = T;
            }
          }
        }
      }
      __syncthreads();
      // sweep: lane = key, slots gi*32 .. gi*32 + 31
      constexpr int kU = 2;                   // tiles per batch per warp
      constexpr int kStep = kU * (kWideThreads / 32);
      const bool last = gi + 1 == groups;
      struct Batch {
        uint32_t w[kU][P];
        float prev[kU], vn[kU];               // parked partial, ||v_j|| (loaded with the codes)
      };
      auto load = [&](Batch& B, int ti0) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int ti = ti0 + u * (kWideThreads / 32);
          const int j = ti * 32 + lane;
          B.prev[u] = 0.f;
          B.vn[u] = 0.f;
          if (ti < vt1) {
#pragma unroll
            for (int wd = 0; wd < P; ++wd) B.w[u][wd] = ldg_nc_u32_hint(crow + packed_word(j, gi, wd, groups, P), pol_code);
            if (gi > 0) B.prev[u] = srow[j];
            if (last) B.vn[u] = __ldg(vrow + j);
          }
        }
      };
      auto compute = [&](const Batch& B, int ti0) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int ti = ti0 + u * (kWideThreads / 32);
          if (ti >= vt1) break;
          const int j = ti * 32 + lane;
          uint64_t acc = 0ull;
#pragma unroll
          for (int sl = 0; sl < 32; sl += 2) {
            const uint32_t a0 = (slot_bits<P>(B.w[u], sl, 7) & amask) | ((lane4 + 4u * sl) & 124u);
            const uint32_t a1 = (slot_bits<P>(B.w[u], sl + 1, 7) & amask) | ((lane4 + 4u * sl + 4u) & 124u);
            const float v0 = *reinterpret_cast<const float*>(tabc + a0);
            const float v1 = *reinterpret_cast<const float*>(tabc + a1);
            const uint64_t pv = (uint64_t)__float_as_uint(v0) | ((uint64_t)__float_as_uint(v1) << 32);
            asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(pv));
          }
          const float accg = __uint_as_float((uint32_t)acc) + __uint_as_float((uint32_t)(acc >> 32));
          if (!last) {
            srow[j] = gi == 0 ? accg : B.prev[u] + accg;
          } else {
            const float tot = (gi > 0 ? B.prev[u] : 0.f) + accg;
            const bool ok = j < n && (!mrow || mrow[j]);
            st_f32_hint(srow + j, ok ? B.vn[u] * tot : -INFINITY, pol_score);   // top-k reads it next
          }
        }
      };
      // two batches per warp: the next batch's loads are in flight while the
      // current one is looked up
      Batch A, Bn;
      int ti0 = t0 + warp;
      if (ti0 < vt1) load(A, ti0);
      for (; ti0 < vt1; ti0 += 2 * kStep) {
        if (ti0 + kStep < vt1) load(Bn, ti0 + kStep);
        compute(A, ti0);
        if (ti0 + kStep >= vt1) break;
        if (ti0 + 2 * kStep < vt1) load(A, ti0 + 2 * kStep);
        compute(Bn, ti0 + kStep);
      }
    }
    for (int ti = max(t0, vt1) + warp; ti < t1; ti += kWideThreads / 32) srow[ti * 32 + lane] = -INFINITY;
  }
}

static socket_status launch_score_wide(const socket_cfg& c, const float* lut, const uint8_t* codes,
                                       const float* vnorm, const int32_t* seq_lens,
                                       const uint8_t* mask, float* scores, cudaStream_t st) {
  const int Lp = code_slots_p(c.L, c.P);
  if (Lp > 64) return fail(SOCKET_EUNSUPPORTED, "score: P > 8 with more than 64 tables");
  const size_t bytes = lut_row_bytes(c);
  const int NH = heads_per_row(c);
  const int H_sel = num_sel_rows(c);
  const int G_sel = c.group_mode == SOCKET_GROUP_PER_QHEAD ? c.H_q / c.H_kv : 1;
  const dim3 grid((c.N_max / 32 + kWideTilesPerCta - 1) / kWideTilesPerCta, c.B * H_sel);
  if (grid.x == 0 || grid.y == 0) return SOCKET_OK;
  const int E = wide_entries(c.P);
  const int row_floats = (int)(bytes / sizeof(float));
  const uint32_t* cw = reinterpret_cast<const uint32_t*>(codes);
  if (c.P <= 10) {
    // group-summed tables per 32-slot group (one LDS per lookup)
    const int R = 1 << c.P, RL = 1 << (c.P / 2);
    const size_t sm2 = ((size_t)R * 32 + (size_t)NH * (RL + R / RL) * 32) * sizeof(float);   // tab + A + B
    const long long total_tiles = (long long)c.B * H_sel * (c.N_max / 32);
    const unsigned pgrid = (unsigned)(total_tiles < num_sms() ? total_tiles : num_sms());
#define SK_WIDE2(N, PV)                                                                        \
  if (NH == N && c.P == PV) {                                                                  \
    cudaFuncSetAttribute(score_wide2_kernel<N, PV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2); \
    score_wide2_kernel<N, PV><<<pgrid, kWideThreads, sm2, st>>>(                               \
        lut, cw, vnorm, seq_lens, mask, scores, H_sel, c.H_kv, G_sel, c.N_max, Lp, E, row_floats, \
        total_tiles, c.index_base);                                                            \
    return check_launch("score_wide2_kernel");                                                 \
  }
    SK_WIDE2(1, 9) SK_WIDE2(2, 9) SK_WIDE2(4, 9) SK_WIDE2(8, 9)
    SK_WIDE2(1, 10) SK_WIDE2(2, 10) SK_WIDE2(4, 10) SK_WIDE2(8, 10)
#undef SK_WIDE2
    return fail(SOCKET_EUNSUPPORTED, "score: heads per selection row must be 1, 2, 4 or 8");
  }
  if (bytes > kWideLutMax) {
    // tiled over (32-slot group, head chunk): the largest chunk whose sub-image fits
    int nhc = NH > 4 ? 4 : NH;
    while (nhc > 1 && (size_t)nhc * 2 * E * 32 * sizeof(float) > kWideLutMax) nhc >>= 1;
    const size_t sub = (size_t)nhc * 2 * E * 32 * sizeof(float);
    if (sub > kWideLutMax) return fail(SOCKET_EUNSUPPORTED, "score: P > 8 half-table tile exceeds shared memory");
#define SK_WIDET(N, PV)                                                                        \
  if (nhc == N && c.P == PV) {                                                                 \
    cudaFuncSetAttribute(score_wide_tiled_kernel<N, PV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sub); \
    score_wide_tiled_kernel<N, PV><<<grid, kWideThreads, sub, st>>>(                           \
        lut, cw, vnorm, seq_lens, mask, scores, H_sel, c.H_kv, G_sel, c.N_max, Lp, NH, E, row_floats, \
        c.index_base);                                                                         \
    return check_launch("score_wide_tiled_kernel");                                            \
  }
    SK_WIDET(1, 13) SK_WIDET(2, 13) SK_WIDET(4, 13)
    SK_WIDET(1, 14) SK_WIDET(2, 14) SK_WIDET(4, 14)
    SK_WIDET(1, 15) SK_WIDET(2, 15) SK_WIDET(4, 15)
    SK_WIDET(1, 16) SK_WIDET(2, 16) SK_WIDET(4, 16)
    SK_WIDET(1, 11) SK_WIDET(2, 11) SK_WIDET(4, 11)
    SK_WIDET(1, 12) SK_WIDET(2, 12) SK_WIDET(4, 12)
#undef SK_WIDET
    return fail(SOCKET_EUNSUPPORTED, "score: wide-code tile shape not instantiated");
  }
#define SK_WIDE(N, PV)                                                                         \
  if (NH == N && c.P == PV) {                                                                  \
    cudaFuncSetAttribute(score_wide_kernel<N, PV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes); \
    score_wide_kernel<N, PV><<<grid, kWideThreads, bytes, st>>>(                               \
        lut, cw, vnorm, seq_lens, mask, scores, H_sel, c.H_kv, G_sel, c.N_max, Lp, E, row_floats, \
        c.index_base);                                                                         \
    return check_launch("score_wide_kernel");                                                  \
  }
  SK_WIDE(1, 11) SK_WIDE(2, 11) SK_WIDE(4, 11) SK_WIDE(8, 11)
  SK_WIDE(1, 12) SK_WIDE(2, 12) SK_WIDE(4, 12) SK_WIDE(8, 12)
  SK_WIDE(1, 13) SK_WIDE(2, 13) SK_WIDE(4, 13) SK_WIDE(8, 13)
  SK_WIDE(1, 14) SK_WIDE(2, 14) SK_WIDE(4, 14) SK_WIDE(8, 14)
  SK_WIDE(1, 15) SK_WIDE(2, 15) SK_WIDE(4, 15) SK_WIDE(8, 15)
  SK_WIDE(1, 16) SK_WIDE(2, 16) SK_WIDE(4, 16) SK_WIDE(8, 16)
#undef SK_WIDE
  return fail(SOCKET_EUNSUPPORTED, "score: heads per selection row must be 1, 2, 4 or 8");
}

// ----------------------------------------------------------------------------
// score kernel, register-fed (default): lane = key, the 64 code bytes and the
// norm of a lane's key come straight from global memory into registers with
// 16-byte non-allocating loads, double-buffered (tile i+1 is in flight while
// tile i is looked up).  Staging the codes through shared memory (cp.async or
// TMA rings) costs 32 extra shared-memory wavefronts per tile on top of the 64
// LUT lookups, and shared-memory bandwidth, not HBM, was the limit
// (ncu / tools/micro/stream_bw.cu: LDG.128 streams reach 6.6 TB/s).
// ----------------------------------------------------------------------------
template <int LP>
struct RegTile {
  uint32_t w[LP / 4];
  float vn;
};

template <int LP>
__device__ __forceinline__ void load_reg_tile(RegTile<LP>& t, const uint8_t* tile_codes,
                                              const float* tile_vn, int lane, uint64_t pol) {
  constexpr int CB = LP < 16 ? LP : 16;
#pragma unroll
  for (int ch = 0; ch < LP / CB; ++ch) {
    if constexpr (CB == 16) {
      const uint4 v = ldg_nc_v4_hint(tile_codes + ch * 512 + lane * 16, pol);
      t.w[ch * 4 + 0] = v.x; t.w[ch * 4 + 1] = v.y; t.w[ch * 4 + 2] = v.z; t.w[ch * 4 + 3] = v.w;
    } else {
      const uint2 v = ldg_nc_v2_hint(tile_codes + ch * 256 + lane * 8, pol);
      t.w[ch * 2 + 0] = v.x; t.w[ch * 2 + 1] = v.y;
    }
  }
  t.vn = __ldg(tile_vn + lane);
}

template <int LP>
__global__ void __launch_bounds__(kScoreThreads, 1)
score_reg_kernel(const float* __restrict__ lut_g, const uint8_t* __restrict__ codes,
                 const float* __restrict__ vnorm, const int32_t* __restrict__ seq_lens,
                 const uint8_t* __restrict__ mask, float* __restrict__ scores, int H_sel, int H_kv,
                 int G_sel, int N_max, long long total_tiles, long long index_base) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar;
  constexpr uint32_t LUT_BYTES = 256 * 64 * 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t pk[16];
#pragma unroll
  for (int m = 0; m < 16; ++m)
    pk[m] = (uint32_t)(((2 * m + lane) & 31) << 2) | ((uint32_t)(((2 * m + 1 + lane) & 31) << 2) << 8);
  const uint64_t pol_code = l2_policy_evict_first(), pol_score = l2_policy_evict_last();
  const int tiles_per_row = N_max >> 5;
  const long long t_begin = total_tiles * blockIdx.x / gridDim.x;
  const long long t_end = total_tiles * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: LUT / codes of the predecessor
  uint32_t phase = 0;
  for (long long t = t_begin; t < t_end;) {
    const int row = (int)(t / tiles_per_row);
    const long long seg_end = min(t_end, (long long)(row + 1) * tiles_per_row);
    const int tile0 = (int)(t - (long long)row * tiles_per_row);
    const int tile1 = (int)(seg_end - (long long)row * tiles_per_row);
    t = seg_end;
    const int b = row / H_sel, r = row % H_sel, g = r / G_sel;
    const int n = local_len(seq_lens[b], index_base, N_max);
    const int vt1 = min(tile1, (n + 31) >> 5);
    const bool need_lut = tile0 < vt1;
    if (need_lut && threadIdx.x == 0) {
      mbar_expect_tx(&bar, LUT_BYTES);
      const char* src = reinterpret_cast<const char*>(lut_g) + (size_t)row * LUT_BYTES;
#pragma unroll
      for (uint32_t off = 0; off < LUT_BYTES; off += 32768) bulk_g2s(smem + off, src + off, 32768, &bar);
    }
    const uint8_t* crow = codes + ((size_t)b * H_kv + g) * N_max * LP;
    const float* vrow = vnorm + ((size_t)b * H_kv + g) * N_max;
    const uint8_t* mrow = mask ? mask + (size_t)b * N_max : nullptr;
    float* srow = scores + (size_t)row * N_max;
    // my tiles: tile0 + warp + 16 i < vt1, two per iteration with the next two in
    // flight (4 tiles = 256 B per lane outstanding); the first two load while the
    // LUT arrives
    auto score_tile = [&](const RegTile<LP>& tt, int tix) {
      uint64_t acc = 0ull;
#pragma unroll
      for (int s2 = 0; s2 < LP; s2 += 2) {
        float v[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int ss = s2 + u, sl = ss & 31;
          const uint32_t sel = (uint32_t)(4 + (sl & 1)) | ((uint32_t)(ss & 3) << 4) | 0x7600u;
          const uint32_t addr = __byte_perm(tt.w[ss >> 2], pk[sl >> 1], sel);   // code*256 + 4 c
          v[u] = *reinterpret_cast<const float*>(smem + ((ss & 32) ? 128 : 0) + addr);
        }
        const uint64_t pv = (uint64_t)__float_as_uint(v[0]) | ((uint64_t)__float_as_uint(v[1]) << 32);
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(pv));
      }
      const float acc0 = __uint_as_float((uint32_t)acc), acc1 = __uint_as_float((uint32_t)(acc >> 32));
      const int j = tix * 32 + lane;
      const bool ok = j < n && (!mrow || mrow[j]);
      st_f32_hint(srow + j, ok ? tt.vn * (acc0 + acc1) : -INFINITY, pol_score);   // top-k reads it next
    };
    constexpr int W = kScoreWarps;
    int ti = tile0 + warp;
    RegTile<LP> a0, a1, b0, b1;
    if (ti < vt1) load_reg_tile<LP>(a0, crow + (size_t)ti * 32 * LP, vrow + ti * 32, lane, pol_code);
    if (ti + W < vt1) load_reg_tile<LP>(a1, crow + (size_t)(ti + W) * 32 * LP, vrow + (ti + W) * 32, lane, pol_code);
    if (need_lut) mbar_wait(&bar, phase);
    for (; ti < vt1; ti += 2 * W) {
      if (ti + 2 * W < vt1) load_reg_tile<LP>(b0, crow + (size_t)(ti + 2 * W) * 32 * LP, vrow + (ti + 2 * W) * 32, lane, pol_code);
      if (ti + 3 * W < vt1) load_reg_tile<LP>(b1, crow + (size_t)(ti + 3 * W) * 32 * LP, vrow + (ti + 3 * W) * 32, lane, pol_code);
      score_tile(a0, ti);
      if (ti + W < vt1) score_tile(a1, ti + W);
      a0 = b0;
      a1 = b1;
    }
    for (int tz = max(tile0, vt1) + warp; tz < tile1; tz += kScoreWarps) srow[tz * 32 + lane] = -INFINITY;
    if (need_lut) phase ^= 1;
    __syncthreads();   // everyone done with this LUT before it is overwritten
  }
}

socket_status launch_score_pdl(const socket_cfg& c, const float* lut, const uint8_t* codes,
                               const float* vnorm, const int32_t* seq_lens, const uint8_t* mask,
                               float* scores, cudaStream_t st, bool pdl) {
  if (c.P > 8) return launch_score_wide(c, lut, codes, vnorm, seq_lens, mask, scores, st);
  const int Lp = code_slots_p(c.L, c.P);
  const int H_sel = num_sel_rows(c);
  const int G_sel = c.group_mode == SOCKET_GROUP_PER_QHEAD ? c.H_q / c.H_kv : 1;
  const long long total_tiles = (long long)c.B * H_sel * (c.N_max / 32);
  long long grid = num_sms();
  if (grid > total_tiles) grid = total_tiles;
  if (grid < 1) return SOCKET_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kScoreThreads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
#define SK_SCORE_CASE(LPV)                                                                     \
  case LPV: {                                                                                  \
    const size_t smem3 = 256 * 64 * 4;                                                         \
    auto kfn3 = score_reg_kernel<LPV>;                                                         \
    cudaFuncSetAttribute(kfn3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);       \
    cfg.dynamicSmemBytes = smem3;                                                              \
    cudaError_t e3 = cudaLaunchKernelEx(&cfg, kfn3, lut, codes, vnorm, seq_lens, mask, scores, H_sel, \
                                        c.H_kv, G_sel, c.N_max, total_tiles, c.index_base);    \
    if (e3 != cudaSuccess) return fail(SOCKET_ECUDA, std::string("score launch: ") + cudaGetErrorString(e3)); \
    return check_launch("score_reg_kernel");                                                   \
  }
  switch (Lp) {
    SK_SCORE_CASE(8)
    SK_SCORE_CASE(16)
    SK_SCORE_CASE(32)
    SK_SCORE_CASE(64)
    default:
      return fail(SOCKET_EUNSUPPORTED, "score: L > 64 not supported by this kernel");
  }
#undef SK_SCORE_CASE
}

socket_status launch_score(const socket_cfg& c, const float* lut, const uint8_t* codes,
                           const float* vnorm, const int32_t* seq_lens, const uint8_t* mask,
                           float* scores, cudaStream_t st) {
  return launch_score_pdl(c, lut, codes, vnorm, seq_lens, mask, scores, st, false);
}

}  // namespace sk
