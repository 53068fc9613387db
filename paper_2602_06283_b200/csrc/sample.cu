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
// One 1024-thread CTA per row:
//   1. sort (u_m, m) ascending in shared memory (bitonic);
//   2. thread t owns the contiguous key segment [t S, (t+1) S): segment sums of
//      s and of w_hat = s / ||v|| (fp32, j ascending), a deterministic block
//      scan gives the segment offsets off_t and the totals C = C_n, Z = sum w_hat;
//   3. thread t takes the sorted targets x_m = u_m C in [off_t, off_{t+1}) and
//      walks its segment once (two pointers): J_m = first j with off_t + prefix > x_m;
//   4. the CTA gathers v_J / ||v_J|| (warps over contiguous sorted samples,
//      lanes over 4 dims), reduces across warps in warp order and writes
//      T = (C / Z) / M * sum, rounded to bf16.
#include "internal.cuh"

namespace sk {

constexpr int kSmpThreads = 1024;
constexpr int kSmpWarps = kSmpThreads / 32;
constexpr int kSmpMaxM = 8192;

struct SampleArgs {
  const float* scores;    // [B][H_q][N_max]
  const float* vnorm;     // [B][H_kv][N_max]
  const uint16_t* V;      // [B][H_kv][N_max][128] bf16
  const int32_t* seq_lens;
  const float* uniforms;  // [B][H_q][M]
  int32_t* samples;       // [B][H_q][M] or null
  uint16_t* out;          // [B][H_q][128] bf16
  int H_q, H_kv, N_max, M, Mp2;
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

__device__ __forceinline__ bool pair_less(float a, int ia, float b, int ib) {
  return a < b || (a == b && ia < ib);
}

__global__ void __launch_bounds__(kSmpThreads, 1) sample_decode_kernel(SampleArgs a) {
  extern __shared__ __align__(16) char smem[];
  float* su = reinterpret_cast<float*>(smem);            // [Mp2] sorted uniforms
  int* si = reinterpret_cast<int*>(su + a.Mp2);           // [Mp2] their original positions
  int* sj = si + a.Mp2;                                   // [M] J of the sorted samples
  float* red = reinterpret_cast<float*>(sj + a.M);        // [kSmpWarps][128]
  __shared__ float s_off[kSmpThreads + 1];
  __shared__ float s_wtot[kSmpWarps], s_stot[kSmpWarps];
  __shared__ int s_lo[kSmpThreads + 1];
  __shared__ int s_jlast;

  const int row = blockIdx.x;
  const int b = row / a.H_q, h = row % a.H_q;
  const int g = h / (a.H_q / a.H_kv);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = a.M;
  const int n = min(max(a.seq_lens[b], 0), a.N_max);
  const float* srow = a.scores + (size_t)row * a.N_max;
  const float* vrow = a.vnorm + ((size_t)b * a.H_kv + g) * a.N_max;

  // ---- 1. sort (u, m) ascending ------------------------------------------------
  for (int i = tid; i < a.Mp2; i += kSmpThreads) {
    su[i] = i < M ? a.uniforms[(size_t)row * M + i] : INFINITY;
    si[i] = i;
  }
  if (tid == 0) s_jlast = -1;
  __syncthreads();
  for (int size = 2; size <= a.Mp2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < a.Mp2; i += kSmpThreads) {
        const int p = i ^ stride;
        if (p > i) {
          const bool up = (i & size) == 0;
          const float x = su[i], y = su[p];
          const int ix = si[i], iy = si[p];
          if (pair_less(y, iy, x, ix) == up) { su[i] = y; su[p] = x; si[i] = iy; si[p] = ix; }
        }
      }
      __syncthreads();
    }
  }

  // ---- 2. segment sums and the block scan ----------------------------------------
  // segments are multiples of 4 keys so they can be read as float4 (j0 16-B aligned)
  const int S = (((n + kSmpThreads - 1) / kSmpThreads) + 3) & ~3;
  const int j0 = min(tid * S, n), j1 = min(j0 + S, n);
  float seg_s = 0.f, seg_w = 0.f;
  int jpos = -1;
#pragma unroll 4
  for (int j = j0; j < j1; j += 4) {
    const float4 sv = ld4_masked(srow, j, j1);
    const float4 vv = ld4_masked(vrow, j, j1);
    const float ss[4] = {sv.x, sv.y, sv.z, sv.w}, vs[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (ss[e] > 0.f) {                     // -inf (invalid), 0 and padding carry no mass
        seg_s += ss[e];
        seg_w += vs[e] > 0.f ? ss[e] / vs[e] : 0.f;   // w_hat_j = s_j / ||v_j||  (R-24)
        jpos = j + e;
      }
    }
  }
  if (jpos >= 0) atomicMax(&s_jlast, jpos);
  float inc = seg_s, wsum = seg_w;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  if (lane == 31) s_stot[warp] = inc;
  if (lane == 0) s_wtot[warp] = wsum;
  __syncthreads();
  if (warp == 0) {
    float ti = s_stot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    float tex = __shfl_up_sync(0xffffffffu, ti, 1);
    if (lane == 0) tex = 0.f;
    s_stot[lane] = tex;                      // exclusive warp offsets
    float w = s_wtot[lane];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (lane == 0) s_wtot[0] = w;
  }
  __syncthreads();
  float ex = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) ex = 0.f;
  const float off = s_stot[warp] + ex;                     // exclusive offset of my segment
  s_off[tid] = off;
  if (tid == kSmpThreads - 1) s_off[kSmpThreads] = s_stot[warp] + inc;
  __syncthreads();
  const float C = s_off[kSmpThreads];
  const float Z = s_wtot[0];

  // ---- 3. my targets: sorted x = u C in [off_t, off_{t+1}) ---------------------
  {   // lo_t = first sorted sample with u C >= off_t (binary search)
    int lo = 0, hi = M;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (su[mid] * C < off) lo = mid + 1; else hi = mid;
    }
    s_lo[tid] = tid == 0 ? 0 : lo;
    if (tid == 0) s_lo[kSmpThreads] = M;
  }
  __syncthreads();
  if (C > 0.f) {
    const int m0 = s_lo[tid], m1 = s_lo[tid + 1];
    float c = off;            // cumulative mass of the segment's keys before j
    int j = j0, jl = -1;
    // the segment is read 8 keys at a time (two float4), the next 8 prefetched
    int cj = j0;
    float4 a0 = ld4_masked(srow, cj, j1), a1 = ld4_masked(srow, cj + 4, j1);
    float4 b0 = ld4_masked(srow, cj + 8, j1), b1 = ld4_masked(srow, cj + 12, j1);
    for (int m = m0; m < m1; ++m) {
      const float x = su[m] * C;
      while (j < j1) {
        if (j >= cj + 8) {
          cj += 8;
          a0 = b0;
          a1 = b1;
          b0 = ld4_masked(srow, cj + 8, j1);
          b1 = ld4_masked(srow, cj + 12, j1);
        }
        const float s = pick8(a0, a1, j - cj);
        if (s > 0.f) {
          jl = j;
          if (c + s > x) break;  // J = j; key j stays unconsumed for the next target
          c += s;
        }
        ++j;
      }
      int J;
      if (j < j1) J = j;                     // first j with C_j > x
      else J = jl >= 0 ? jl : s_jlast;       // rounding at the segment end
      sj[m] = J;
      if (a.samples) a.samples[(size_t)row * M + si[m]] = J;
    }
  } else if (a.samples) {
    for (int m = tid; m < M; m += kSmpThreads) a.samples[(size_t)row * M + m] = -1;
  }
  __syncthreads();

  // ---- 4. gather v_J / ||v_J|| and reduce ----------------------------------------
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if (C > 0.f) {
    const int per = (M + kSmpWarps - 1) / kSmpWarps;
    const int mb = min(warp * per, M), me = min(mb + per, M);
    const uint16_t* vbase = a.V + ((size_t)b * a.H_kv + g) * a.N_max * kD + lane * 4;
    constexpr int U = 8;                     // rows in flight per warp
    for (int m0 = mb; m0 < me; m0 += U) {
      uint2 u[U];
      float vn[U];
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const int m = m0 + x;
        const int J = m < me ? sj[m] : sj[mb];
        u[x] = ldg_nc_v2(vbase + (size_t)J * kD);
        vn[x] = __ldg(vrow + J);
      }
#pragma unroll
      for (int x = 0; x < U; ++x) {          // accumulate in draw order
        if (m0 + x >= me) break;
        const float f = 1.0f / vn[x];
        acc[0] = fmaf(bf16lo(u[x].x), f, acc[0]);
        acc[1] = fmaf(bf16hi(u[x].x), f, acc[1]);
        acc[2] = fmaf(bf16lo(u[x].y), f, acc[2]);
        acc[3] = fmaf(bf16hi(u[x].y), f, acc[3]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) red[warp * kD + lane * 4 + e] = acc[e];
  __syncthreads();
  if (tid < kD) {
    float t = 0.f;
    for (int w = 0; w < kSmpWarps; ++w) t += red[w * kD + tid];
    const float scale = (C > 0.f && Z > 0.f && M > 0) ? (C / Z) / (float)M : 0.f;
    a.out[(size_t)row * kD + tid] = (uint16_t)f2bf_bits(t * scale);
  }
}

size_t sample_smem_bytes(int M) {
  int Mp2 = 1;
  while (Mp2 < M) Mp2 <<= 1;
  return (size_t)Mp2 * 8 + (size_t)M * 4 + (size_t)kSmpWarps * kD * 4;
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
  int Mp2 = 1;
  while (Mp2 < M) Mp2 <<= 1;
  a.Mp2 = Mp2;
  const size_t sm = sample_smem_bytes(M);
  cudaFuncSetAttribute(sample_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  sample_decode_kernel<<<rows, kSmpThreads, sm, st>>>(a);
  return check_launch("sample_decode_kernel");
}

}  // namespace sk
