// Value-aware sampling decode: the estimator T(q) of Eq. 6 (PAPER.md l.338-346,
// "Sampling-based Estimator"), on the GPU.
//
// Per query row (b, h) (PER_QHEAD: the paper's single-query setting) with the
// masked value scores s_j = ||v_j|| w_hat_j of Alg. 4 (-inf = invalid):
//   a~_j = w_hat_j / sum_i w_hat_i,   p_j = a~_j ||v_j|| / sum_i a~_i ||v_i|| = s_j / sum_i s_i
//   J_m = min{ j : C_j > u_m C_n },   C_j = sum_{i <= j} s_i   (inverse CDF of p)
//   T   = (1/M) sum_m (a~_J / p_J) v_J = (sum s / sum w_hat) / M * sum_m v_J / ||v_J||
// with the M uniforms u_m in [0, 1) supplied by the caller (the random numbers
// the method draws are inputs, so the CPU oracle can replay them).
//
// One 256-thread CTA per row, 4 CTAs per SM (the whole batch is one wave):
//   1. the row's keys split into kSub = 4096 sub-blocks of S keys (S = 8 at 32K);
//      lane pairs sum s and w_hat = s / ||v|| per sub-block with float4 loads; a
//      block scan turns the sums into sub-block offsets off_t and the totals
//      C = C_n, Z = sum w_hat;
//   2. every draw (3 per thread in flight): binary search for the sub-block with
//      the largest off_t <= x_m = u_m C, then walk its S keys, J_m = first j with
//      off_t + prefix > x_m -- no sort of the uniforms, every draw costs one
//      short walk however the mass is spread; J into shared memory;
//   3. each warp gathers v_J / ||v_J|| for a contiguous run of draws (half-warp
//      per row, 16-B loads, 16 rows in flight), the CTA reduces across warps in
//      warp order and writes T = (C / Z) / M * sum, rounded to bf16.
// fp32 throughout; offsets and the walk are deterministic (no atomics on sums).
#include "internal.cuh"

namespace sk {

#ifdef SK_TRACE
static __device__ unsigned long long g_smp_trace[1024 * 8];
#define SM_STAMP(i)                                                                        \
  do {                                                                                     \
    if (threadIdx.x == 0 && blockIdx.x < 1024) g_smp_trace[blockIdx.x * 8 + (i)] = clock64(); \
  } while (0)
extern "C" int socket_debug_sample_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_smp_trace, (size_t)n * sizeof(unsigned long long));
}
#else
#define SM_STAMP(i) \
  do {              \
  } while (0)
#endif

constexpr int kSmpThreads = 256;
constexpr int kSmpWarps = kSmpThreads / 32;
constexpr int kSmpMaxM = 8192;
constexpr int kSub = 4096;          // CDF sub-blocks per row (the binary-search grid)
#ifndef SK_SMP_U
#define SK_SMP_U 16
#endif
constexpr int kSmpU = SK_SMP_U;     // V rows in flight per warp in the gather

struct SampleArgs {
  const float* scores;    // [B][H_q][N_max]
  const float* vnorm;     // [B][H_kv][N_max]
  const uint16_t* V;      // [B][H_kv][N_max][128] bf16
  const int32_t* seq_lens;
  const float* uniforms;  // [B][H_q][M]
  int32_t* samples;       // [B][H_q][M] or null
  uint16_t* out;          // [B][H_q][128] bf16
  int H_q, H_kv, N_max, M;
};

// 4 consecutive floats at p[j..j+3] (j % 4 == 0, 16-B aligned); lanes >= j1 read as 0
__device__ __forceinline__ float4 ld4_masked(const float* p, int j, int j1) {
  if (j + 4 <= j1) return __ldg(reinterpret_cast<const float4*>(p + j));
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j < j1) v.x = p[j];
  if (j + 1 < j1) v.y = p[j + 1];
  if (j + 2 < j1) v.z = p[j + 2];
  return v;
}
__device__ __forceinline__ float pick8(const float4& a, const float4& b, int i) {
  const float4 v = i < 4 ? a : b;
  const int k = i & 3;
  return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}

__global__ void __launch_bounds__(kSmpThreads, 4) sample_decode_kernel(SampleArgs a) {
  __shared__ float s_off[kSub + 1];              // sub-block sums, then their exclusive offsets
  __shared__ __align__(16) float red[kSmpWarps][kD];
  __shared__ float s_wtot[kSmpWarps], s_stot[kSmpWarps];
  __shared__ int s_jlast;
  extern __shared__ int sj[];                    // [M] J of each draw

  const int row = blockIdx.x;
  const int b = row / a.H_q, h = row % a.H_q;
  const int g = h / (a.H_q / a.H_kv);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = a.M;
  const int n = min(max(a.seq_lens[b], 0), a.N_max);
  const float* srow = a.scores + (size_t)row * a.N_max;
  const float* vrow = a.vnorm + ((size_t)b * a.H_kv + g) * a.N_max;

  if (tid == 0) s_jlast = -1;
  SM_STAMP(0);
  // ---- 1. sub-block sums -----------------------------------------------------------
  // kSub sub-blocks of S keys (S a multiple of 8); a lane pair sums one sub-block
  // with float4 loads (lane sl covers keys i + 4 sl .. + 3 of every 8), four
  // sub-blocks per pair in flight.
  const int S = max(8, ((n + kSub - 1) / kSub + 7) & ~7);
  constexpr int kGroups = kSmpThreads / 2;
  const int sl = lane & 1, grp = tid >> 1;
  float pw = 0.f;                                          // this lane's sum of w_hat
  int jpos = -1;
  for (int kb = 0; kb < kSub / kGroups; kb += 4) {
    float ps[4] = {0.f, 0.f, 0.f, 0.f};
    for (int i = 0; i < S; i += 8) {
      float4 sv[4], vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = (grp + (kb + u) * kGroups) * S + i + sl * 4;
        sv[u] = ld4_masked(srow, j, n);
        vv[u] = ld4_masked(vrow, j, n);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = (grp + (kb + u) * kGroups) * S + i + sl * 4;
        const float ss[4] = {sv[u].x, sv[u].y, sv[u].z, sv[u].w};
        const float vs[4] = {vv[u].x, vv[u].y, vv[u].z, vv[u].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (ss[e] > 0.f) {                 // -inf (invalid), 0 and padding carry no mass
            ps[u] += ss[e];
            pw += vs[e] > 0.f ? __fdividef(ss[e], vs[e]) : 0.f;   // w_hat_j = s_j / ||v_j||  (R-24)
            jpos = max(jpos, j + e);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float t = ps[u] + __shfl_xor_sync(0xffffffffu, ps[u], 1);
      if (sl == 0) s_off[grp + (kb + u) * kGroups] = t;
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    pw += __shfl_xor_sync(0xffffffffu, pw, o);
    jpos = max(jpos, __shfl_xor_sync(0xffffffffu, jpos, o));
  }
  __syncthreads();                           // s_jlast init and the sums are visible
  if (lane == 0) {
    s_wtot[warp] = pw;
    if (jpos >= 0) atomicMax(&s_jlast, jpos);
  }
  SM_STAMP(1);
  // ---- 2. exclusive scan of the kSub sums (kPer per thread, then warps) ------------
  constexpr int kPer = kSub / kSmpThreads;
  float tsum = 0.f;
#pragma unroll
  for (int e = 0; e < kPer; ++e) tsum += s_off[tid * kPer + e];
  float inc = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_stot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    float ti = lane < kSmpWarps ? s_stot[lane] : 0.f;
#pragma unroll
    for (int o = 1; o < kSmpWarps; o <<= 1) {
      const float y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    float tex = __shfl_up_sync(0xffffffffu, ti, 1);
    if (lane == 0) tex = 0.f;
    float w = lane < kSmpWarps ? s_wtot[lane] : 0.f;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    __syncwarp();
    if (lane < kSmpWarps) s_stot[lane] = tex;   // exclusive warp offsets
    if (lane == 0) s_wtot[0] = w;
  }
  __syncthreads();
  {
    float ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = 0.f;
    float c = s_stot[warp] + ex;             // exclusive offset of my kPer sub-blocks
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const float v = s_off[tid * kPer + e];
      s_off[tid * kPer + e] = c;
      c += v;
    }
    if (tid == kSmpThreads - 1) s_off[kSub] = c;
  }
  __syncthreads();
  const float C = s_off[kSub];
  const float Z = s_wtot[0];

  SM_STAMP(2);
  // ---- 3. the draws: J_m by thread, into shared memory ----------------------------
  // Draw m's target x = u_m C lies in the sub-block of the largest t with
  // off_t <= x (binary search over s_off); the thread walks that sub-block's keys
  // in order, c = off_t + s_j0 + ..., J = first j with c + s_j > x. A target past
  // the sub-block's last positive key (fp32 rounding of the offsets) takes that
  // key; one in a sub-block without mass takes the next key with mass.
  if (C > 0.f) {
    constexpr int kB = 3;                    // draws per thread in flight
    for (int m0 = tid; m0 < M; m0 += kB * kSmpThreads) {
      float x[kB];
      int t[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int m = m0 + u * kSmpThreads;
        x[u] = m < M ? a.uniforms[(size_t)row * M + m] * C : 0.f;
        t[u] = 0;
      }
#pragma unroll
      for (int w = kSub / 2; w >= 1; w >>= 1) {   // largest t with off_t <= x (off_0 = 0)
#pragma unroll
        for (int u = 0; u < kB; ++u)
          if (s_off[t[u] + w] <= x[u]) t[u] += w;
      }
      float4 p0[kB], p1[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int k0 = min(t[u] * S, n), k1 = min(k0 + S, n);
        p0[u] = ld4_masked(srow, k0, k1);
        p1[u] = ld4_masked(srow, k0 + 4, k1);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int m = m0 + u * kSmpThreads;
        if (m >= M) break;
        const int k0 = min(t[u] * S, n), k1 = min(k0 + S, n);
        float c = s_off[t[u]];
        int jl = -1, J = -2;
        float4 q0 = p0[u], q1 = p1[u];
        for (int j = k0; j < k1; j += 8) {
          if (j > k0) {
            q0 = ld4_masked(srow, j, k1);
            q1 = ld4_masked(srow, j + 4, k1);
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float sv = pick8(q0, q1, e);
            if (J == -2 && sv > 0.f) {
              jl = j + e;
              if (c + sv > x[u]) J = j + e;
              else c += sv;
            }
          }
          if (J != -2) break;
        }
        if (J == -2 && jl >= 0) J = jl;
        for (int j = k1; J == -2 && j < n; ++j)   // empty sub-block: the next key with mass
          if (srow[j] > 0.f) J = j;
        if (J == -2) J = s_jlast;
        sj[m] = J;
        if (a.samples) a.samples[(size_t)row * M + m] = J;
      }
    }
  } else if (a.samples) {
    for (int m = tid; m < M; m += kSmpThreads) a.samples[(size_t)row * M + m] = -1;
  }
  __syncthreads();
  SM_STAMP(3);
  // ---- 4. gather v_J / ||v_J||: a contiguous run of draws per warp ----------------
  // half-warp per row: lane l reads dims 8 (l & 15) .. + 7 of row (l >> 4) of each
  // pair, kSmpU rows in flight per warp; 1 / ||v_J|| by rcp.approx (1 ulp).
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (C > 0.f) {
    const int hl = lane >> 4;
    const uint16_t* vbase = a.V + ((size_t)b * a.H_kv + g) * a.N_max * kD + (lane & 15) * 8;
    const int per = (M + kSmpWarps - 1) / kSmpWarps;
    const int mb = min(warp * per, M), me = min(mb + per, M);
    for (int m0 = mb; m0 < me; m0 += kSmpU) {
      uint4 u[kSmpU / 2];
      float vn[kSmpU / 2];
#pragma unroll
      for (int x = 0; x < kSmpU / 2; ++x) {
        const int J = sj[min(m0 + 2 * x + hl, me - 1)];
        u[x] = ldg_nc_v4(vbase + (size_t)J * kD);
        vn[x] = __ldg(vrow + J);
      }
#pragma unroll
      for (int x = 0; x < kSmpU / 2; ++x) {  // accumulate in draw order (per half)
        if (m0 + 2 * x + hl < me) {
          float f;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"(vn[x]));
          const uint32_t w[4] = {u[x].x, u[x].y, u[x].z, u[x].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[2 * e] = fmaf(bf16lo(w[e]), f, acc[2 * e]);
            acc[2 * e + 1] = fmaf(bf16hi(w[e]), f, acc[2 * e + 1]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 16);
  if (lane < 16) {
    *reinterpret_cast<float4*>(&red[warp][lane * 8]) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    *reinterpret_cast<float4*>(&red[warp][lane * 8 + 4]) = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
  __syncthreads();
  if (tid < kD) {
    float t = 0.f;
    for (int w = 0; w < kSmpWarps; ++w) t += red[w][tid];
    const float scale = (C > 0.f && Z > 0.f && M > 0) ? (C / Z) / (float)M : 0.f;
    a.out[(size_t)row * kD + tid] = (uint16_t)f2bf_bits(t * scale);
  }
  SM_STAMP(4);
}

socket_status launch_sample_decode(const socket_cfg& c, const float* scores, const float* vnorm,
                                   const void* V, const int32_t* seq_lens, const float* uniforms,
                                   int M, int32_t* samples, void* out, cudaStream_t st) {
  if (c.group_mode != SOCKET_GROUP_PER_QHEAD)
    return fail(SOCKET_EUNSUPPORTED, "sample decode: PER_QHEAD selection rows only");
  if (M < 1 || M > kSmpMaxM) return fail(SOCKET_EINVAL, "sample decode: M must be in [1, 8192]");
  const int rows = c.B * c.H_q;
  if (rows == 0) return SOCKET_OK;
  SampleArgs a;
  a.scores = scores;
  a.vnorm = vnorm;
  a.V = (const uint16_t*)V;
  a.seq_lens = seq_lens;
  a.uniforms = uniforms;
  a.samples = samples;
  a.out = (uint16_t*)out;
  a.H_q = c.H_q;
  a.H_kv = c.H_kv;
  a.N_max = c.N_max;
  a.M = M;
  const int sm = M * (int)sizeof(int32_t);
  cudaFuncSetAttribute(sample_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  sample_decode_kernel<<<rows, kSmpThreads, sm, st>>>(a);
  return check_launch("sample_decode_kernel");
}

}  // namespace sk
