// Alg. 1 PrecomputeKeyHashes and value norms.
//
// Codes are written in the key-tiled, bank-rotated layout documented in
// include/socket_b200.h.  The tensor-core (tcgen05) projection GEMM for large
// prefills lives in hash_tc.cu; this file holds the CUDA-core path used for
// small ranges (the per-step append of a decode step, n_count = 1) and for
// configurations the tcgen05 kernel does not tile, plus the layout converters.
#include "step_dev.cuh"

namespace sk {


// ----------------------------------------------------------------------------
// CUDA-core hash: one CTA = one 32-key tile of one (b, kv-head); warp w
// computes tables l = w, w+8, ... for the 32 keys (lane = key), each table
// being P dot products of length 128 accumulated in fp32, t ascending.
// ----------------------------------------------------------------------------
constexpr int kHashThreads = 256;

template <typename CT>   // code element: uint8_t (P <= 8) or uint16_t (P > 8)
__global__ void __launch_bounds__(kHashThreads)
hash_keys_simt_kernel(const uint16_t* __restrict__ K, const uint16_t* __restrict__ W,
                      CT* __restrict__ codes, int H_kv, int N_max, int L, int P, int Lp,
                      int n_begin, int n_end) {
  __shared__ float kt[kD][33];            // K tile transposed: kt[t][key]
  __shared__ CT cs[32][128 + 4];          // codes of the tile: cs[key][table]  (L <= 128)
  const int bh = blockIdx.y;
  const int tile = (n_begin >> 5) + blockIdx.x;
  const int j0 = tile * 32;
  const uint16_t* Kb = K + ((size_t)bh * N_max + j0) * kD;
  for (int i = threadIdx.x; i < 32 * kD; i += kHashThreads) {
    const int key = i / kD, t = i % kD;
    kt[t][key] = __uint_as_float((uint32_t)Kb[(size_t)key * kD + t] << 16);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int l = warp; l < L; l += kHashThreads / 32) {
    uint32_t code = 0;
    for (int i = 0; i < P; ++i) {
      const uint16_t* w = W + ((size_t)l * P + i) * kD;
      float x = 0.f;
#pragma unroll 8
      for (int t = 0; t < kD; ++t) x = fmaf(__uint_as_float((uint32_t)w[t] << 16), kt[t][lane], x);
      code |= (x >= 0.f ? 1u : 0u) << i;   // sign(0) = +1 (R-3); row i -> bit i (R-4)
    }
    cs[lane][l] = (CT)code;
  }
  __syncthreads();
  if (P > 8) {
    // packed wide codes: thread = (key, group, word) gathers the slots overlapping
    // word w of the group's 32P-bit string (internal.cuh, packed_word)
    const int G = Lp >> 5;
    uint32_t* cw = reinterpret_cast<uint32_t*>(codes) + (size_t)bh * N_max * Lp * P / 32;
    for (int i = threadIdx.x; i < 32 * G * P; i += kHashThreads) {
      const int key = i & 31, gw = i >> 5, g = gw / P, w = gw % P;
      const int j = j0 + key;
      if (j < n_begin || j >= n_end) continue;
      uint32_t word = 0;
      const int s_lo = (32 * w) / P, s_hi = min(31, (32 * w + 31) / P);
      for (int s = s_lo; s <= s_hi; ++s) {
        const int t = g * 32 + ((s + j) & 31);
        const uint32_t code = t < L ? (uint32_t)cs[key][t] : 0u;
        const int bp = s * P - 32 * w;          // slot's first bit relative to the word
        word |= bp >= 0 ? (code << bp) : (code >> -bp);
      }
      cw[packed_word(j, g, w, G, P)] = word;
    }
    return;
  }
  // write: thread = (key, chunk); CB contiguous code elements per (key, chunk)
  const int CB = Lp < 16 ? Lp : 16;
  const int nch = Lp / CB;
  CT* cb = codes + (size_t)bh * N_max * Lp;
  for (int i = threadIdx.x; i < 32 * nch; i += kHashThreads) {
    const int key = i & 31, ch = i >> 5;
    const int j = j0 + key;
    if (j < n_begin || j >= n_end) continue;
    __align__(16) CT buf[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      if (e < CB) {
        const int s = ch * CB + e;
        const int t = slot_table(s, j, Lp);
        buf[e] = t < L ? cs[key][t] : (CT)0;
      }
    }
    CT* dst = cb + code_off(j, ch * CB, Lp);
    const int nbytes = CB * (int)sizeof(CT);   // 8 or 16
    for (int o = 0; o < nbytes; o += 8)
      *reinterpret_cast<uint2*>(reinterpret_cast<char*>(dst) + o) =
          *reinterpret_cast<const uint2*>(reinterpret_cast<const char*>(buf) + o);
  }
}

// ||v_j||_2.  A warp handles 32 consecutive rows: lane t holds elements
// 4t .. 4t+3 of every row (same per-lane fma order as append_tile) and the 32
// lane partials of the 32 rows are summed by a recursive-halving
// reduce-scatter, which pairs lanes exactly like the xor butterfly of
// append_tile (bit 4 first) -- fp addition is commutative, so every norm is
// bit-identical to the per-step append's -- but costs ~1 shuffle per row
// instead of 5.  Afterwards lane r holds the sum of row r.
constexpr int kVnormRows = 32;

__global__ void __launch_bounds__(256) vnorm_kernel(const uint16_t* __restrict__ V,
                                                    float* __restrict__ vnorm, int N_max,
                                                    int n_begin, int n_count, int rows_total) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int row0 = warp * kVnormRows;
  if (row0 >= rows_total) return;
  // rows row0 .. row0 + 31 of the flattened (bh, j) space (may cross a bh boundary)
  int bh = row0 / n_count, jj = row0 - bh * n_count;
  float v[kVnormRows];
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint2 u[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int row = row0 + half * 16 + r;
      u[r] = make_uint2(0, 0);
      if (row < rows_total)
        u[r] = ldg_nc_v2(V + ((size_t)bh * N_max + n_begin + jj) * kD + lane * 4);
      if (++jj == n_count) { jj = 0; ++bh; }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const float a = bf16lo(u[r].x), b = bf16hi(u[r].x), c = bf16lo(u[r].y), e = bf16hi(u[r].y);
      v[half * 16 + r] = fmaf(a, a, fmaf(b, b, fmaf(c, c, e * e)));
    }
  }
  // recursive halving: at distance off, the lane with bit `off` set keeps the
  // upper half of its values and receives its partner's upper half
#pragma unroll
  for (int off = 16, nv = 32; off >= 1; off >>= 1, nv >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < nv / 2; ++i) {
      const float send = up ? v[i] : v[i + nv / 2];
      const float keep = up ? v[i + nv / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  // lane l now holds row l: bit k of the lane decided "upper half" at distance 2^k
  const int row = row0 + lane;
  if (row < rows_total) {
    const int bh = row / n_count, j = n_begin + row - bh * n_count;
    vnorm[(size_t)bh * N_max + j] = sqrtf(v[0]);
  }
}

// plain [bh][L][N_max] <-> tiled layout; one thread per (bh, j, slot)
template <typename CT>
__global__ void pack_codes_kernel(const CT* __restrict__ plain, CT* __restrict__ codes,
                                  int N_max, int L, int Lp, long long total, bool unpack) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int s = (int)(i % Lp);
  const long long r = i / Lp;
  const int j = (int)(r % N_max);
  const long long bh = r / N_max;
  const int t = slot_table(s, j, Lp);
  CT* cdst = codes + bh * (long long)N_max * Lp + code_off(j, s, Lp);
  if (!unpack) {
    *cdst = t < L ? plain[(bh * L + t) * N_max + j] : (CT)0;
  } else if (t < L) {
    const_cast<CT*>(plain)[(bh * L + t) * N_max + j] = *cdst;
  }
}

// plain [bh][L][N_max] int16 <-> packed wide layout (P > 8)
//   pack:   one thread per (bh, j, group, word): the slots overlapping the word
//   unpack: one thread per (bh, j, slot): the slot's P bits from one or two words
__global__ void pack_wide_kernel(const uint16_t* __restrict__ plain, uint32_t* __restrict__ codes, int N_max,
                                 int L, int Lp, int P, long long total) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int G = Lp >> 5;
  const int w = (int)(i % P);
  const long long r1 = i / P;
  const int g = (int)(r1 % G);
  const long long r2 = r1 / G;
  const int j = (int)(r2 % N_max);
  const long long bh = r2 / N_max;
  uint32_t word = 0;
  const int s_lo = (32 * w) / P, s_hi = min(31, (32 * w + 31) / P);
  for (int s = s_lo; s <= s_hi; ++s) {
    const int t = g * 32 + ((s + j) & 31);
    const uint32_t code = t < L ? (uint32_t)plain[(bh * L + t) * N_max + j] : 0u;
    const int bp = s * P - 32 * w;
    word |= bp >= 0 ? (code << bp) : (code >> -bp);
  }
  codes[bh * (long long)N_max * Lp * P / 32 + packed_word(j, g, w, G, P)] = word;
}

__global__ void unpack_wide_kernel(uint16_t* __restrict__ plain, const uint32_t* __restrict__ codes, int N_max,
                                   int L, int Lp, int P, long long total) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int G = Lp >> 5;
  const int slot = (int)(i % Lp);
  const long long r = i / Lp;
  const int j = (int)(r % N_max);
  const long long bh = r / N_max;
  const int g = slot >> 5, s = slot & 31;
  const int t = g * 32 + ((s + j) & 31);
  if (t >= L) return;
  const uint32_t* cw = codes + bh * (long long)N_max * Lp * P / 32;
  const int bp = s * P, w = bp >> 5, sh = bp & 31;
  uint64_t v = cw[packed_word(j, g, w, G, P)];
  if (sh + P > 32) v |= (uint64_t)cw[packed_word(j, g, w + 1, G, P)] << 32;
  plain[(bh * L + t) * N_max + j] = (uint16_t)((v >> sh) & ((1u << P) - 1u));
}

socket_status launch_hash_keys_simt(const socket_cfg& c, const void* K, const void* W,
                                    uint8_t* codes, int n_begin, int n_count, cudaStream_t st) {
  const int Lp = code_slots_p(c.L, c.P);
  const int t0 = n_begin >> 5, t1 = (n_begin + n_count - 1) >> 5;
  dim3 grid(t1 - t0 + 1, c.B * c.H_kv);
  if (c.P > 8)
    hash_keys_simt_kernel<uint16_t><<<grid, kHashThreads, 0, st>>>(
        (const uint16_t*)K, (const uint16_t*)W, reinterpret_cast<uint16_t*>(codes), c.H_kv, c.N_max,
        c.L, c.P, Lp, n_begin, n_begin + n_count);
  else
    hash_keys_simt_kernel<uint8_t><<<grid, kHashThreads, 0, st>>>(
        (const uint16_t*)K, (const uint16_t*)W, codes, c.H_kv, c.N_max, c.L, c.P, Lp, n_begin,
        n_begin + n_count);
  return check_launch("hash_keys_simt_kernel");
}

socket_status launch_hash_keys_tc(const socket_cfg& c, const void* K, const void* W,
                                  uint8_t* codes, int n_begin, int n_count, cudaStream_t st,
                                  bool* used);

socket_status launch_hash_keys(const socket_cfg& c, const void* K, const void* V, int n_begin,
                               int n_count, const void* W, uint8_t* codes, float* vnorm,
                               cudaStream_t st) {
  if (n_count == 0) return SOCKET_OK;
  socket_status s = SOCKET_OK;
  if (n_count <= 16) {
    const int total = c.B * c.H_kv * n_count;
    ProArgs a = {};
    a.W = (const uint16_t*)W;
    a.K = (const uint16_t*)K;
    a.V = (const uint16_t*)V;
    a.codes = codes;
    a.vnorm = vnorm;
    a.n_keys = total;
    a.n_begin = n_begin;
    a.n_count = n_count;
    a.append_last = 0;
    return launch_prologue(c, a, false, st);   // value norms written by the append tiles
  } else {
    bool used = false;
    s = launch_hash_keys_tc(c, K, W, codes, n_begin, n_count, st, &used);
    if (s == SOCKET_OK && !used) s = launch_hash_keys_simt(c, K, W, codes, n_begin, n_count, st);
  }
  if (s != SOCKET_OK) return s;
  if (V) {
    const int rows = c.B * c.H_kv * n_count;
    const int threads = 256;
    const long long warps = (rows + kVnormRows - 1) / kVnormRows;
    const int blocks = (int)((warps * 32 + threads - 1) / threads);
    vnorm_kernel<<<blocks, threads, 0, st>>>((const uint16_t*)V, vnorm, c.N_max, n_begin, n_count,
                                             rows);
    s = check_launch("vnorm_kernel");
  }
  return s;
}

socket_status launch_pack_codes(const socket_cfg& c, const uint8_t* plain, uint8_t* codes,
                                bool unpack, cudaStream_t st) {
  const int Lp = code_slots_p(c.L, c.P);
  const long long total = (long long)c.B * c.H_kv * c.N_max * Lp;
  if (total == 0) return SOCKET_OK;
  const int threads = 256;
  const unsigned blocks = (unsigned)((total + threads - 1) / threads);
  if (c.P > 8) {
    if (unpack) {
      unpack_wide_kernel<<<blocks, threads, 0, st>>>(reinterpret_cast<uint16_t*>(const_cast<uint8_t*>(plain)),
                                                     reinterpret_cast<const uint32_t*>(codes), c.N_max, c.L,
                                                     Lp, c.P, total);
    } else {
      const long long words = (long long)c.B * c.H_kv * c.N_max * (Lp / 32) * c.P;
      pack_wide_kernel<<<(unsigned)((words + threads - 1) / threads), threads, 0, st>>>(
          reinterpret_cast<const uint16_t*>(plain), reinterpret_cast<uint32_t*>(codes), c.N_max, c.L, Lp,
          c.P, words);
    }
    return check_launch("pack_wide_kernel");
  } else
    pack_codes_kernel<uint8_t><<<blocks, threads, 0, st>>>(plain, codes, c.N_max, c.L, Lp, total,
                                                            unpack);
  return check_launch("pack_codes_kernel");
}

}  // namespace sk
