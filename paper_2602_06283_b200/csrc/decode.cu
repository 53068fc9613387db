// Eq. 2 sparse attention over the selected rows with exact
// logits (l.271, l.309), as a split flash-decode with online softmax, and the
// log-sum-exp combine of partial states.  The dense variant (Eq. 1, every key
// j < seq_len) is the same kernel with an implicit contiguous index list.
//
// Work unit = (b, selection row, split).  A unit's NH query heads share the
// gathered K/V rows (NH = G in KV_SHARED and dense mode, 1 in PER_QHEAD mode).
// The split kernel (tensor-core mma.sync, decode_mma.cu) writes one partial
// (m, l, o) per (b, head, split); the last split CTA of each unit merges them
// (combine_kernel serves socket_lse_combine across sequence shards).
#include <cstdlib>

#include "internal.cuh"

namespace sk {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;


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

socket_status launch_decode_mma(const socket_cfg& c, const void* q, const void* K, const void* V,
                                const int32_t* idx, const int32_t* cnt, int k,
                                const int32_t* seq_lens, bool dense, int units, int NH,
                                int n_splits, int rps, float* part, int* tickets, void* out,
                                float* lse, float* part_out, cudaStream_t st, bool pdl);

// Split geometry: rows per split is a multiple of `gran` (rows one CTA consumes
// per round) and at most `max_rps` (index staging); the splits of a unit are
// balanced (equal up to one granule), and the grid aims at `target` CTAs.
static void pick_splits(int units, int max_rows, int gran, int max_rps, int target,
                        int& n_splits, int& rows_per_split) {
  int ns = (target + units - 1) / units;
  const int max_ns = (max_rows + 2 * gran - 1) / (2 * gran);   // >= 2 rounds per CTA
  if (ns > max_ns) ns = max_ns;
  const int min_ns = (max_rows + max_rps - 1) / max_rps;        // index staging limit
  if (ns < min_ns) ns = min_ns;
  if (ns < 1) ns = 1;
  int rps = (max_rows + ns - 1) / ns;
  rps = (rps + gran - 1) / gran * gran;
  if (rps < gran) rps = gran;
  n_splits = (max_rows + rps - 1) / rps;
  if (n_splits < 1) n_splits = 1;
  rows_per_split = rps;
}

constexpr int kMmaGran = 64, kMmaMaxRps = 2048;

static void decode_geometry(const socket_cfg& c, int k, bool dense, int& units, int& NH,
                            int& n_splits, int& rps) {
  const bool per_q = !dense && c.group_mode == SOCKET_GROUP_PER_QHEAD;
  const int H_sel = per_q ? c.H_q : c.H_kv;
  units = c.B * H_sel;
  NH = per_q ? 1 : c.H_q / c.H_kv;
  // ~0.86 of one wave at 2 CTAs per SM (256 CTAs on 148 SMs): a single wave of
  // balanced splits was the fastest geometry in tools/tune_step.py sweeps
  // (B 4-16, 5x-10x, 32K)
#ifdef SK_DECODE_TARGET_PCT   // experiments only (tools/variant_build.py)
  const int target = num_sms() * SK_DECODE_TARGET_PCT / 100;
#else
  const int target = num_sms() * 173 / 100;
#endif
  pick_splits(units, dense ? c.N_max : k, kMmaGran, kMmaMaxRps, target, n_splits, rps);
}

static size_t part_bytes(const socket_cfg& c, int ns) {
  return ((size_t)c.B * c.H_q * ns * (kD + 2) * sizeof(float) + 255) & ~(size_t)255;
}

size_t decode_workspace_bytes(const socket_cfg& c, int k, bool dense) {
  int units, NH, ns, rps;
  decode_geometry(c, k, dense, units, NH, ns, rps);
  return part_bytes(c, ns) + (size_t)units * sizeof(int);
}

socket_status launch_decode(const socket_cfg& c, const void* q, const void* K, const void* V,
                            const int32_t* idx, const int32_t* cnt, int k,
                            const int32_t* seq_lens, bool dense, void* out, float* lse,
                            float* partial, void* ws, size_t ws_bytes, cudaStream_t st) {
  int units, NH, ns, rps;
  decode_geometry(c, k, dense, units, NH, ns, rps);
  if (ws_bytes < part_bytes(c, ns) + (size_t)units * sizeof(int))
    return fail(SOCKET_EWORKSPACE, "decode: workspace too small");
  if (units == 0) return SOCKET_OK;
  if (NH > 8) return fail(SOCKET_EUNSUPPORTED, "decode: more than 8 query heads per selection row");
  int* tickets = reinterpret_cast<int*>(static_cast<char*>(ws) + part_bytes(c, ns));
  cudaError_t e = cudaMemsetAsync(tickets, 0, (size_t)units * sizeof(int), st);
  if (e != cudaSuccess) return fail(SOCKET_ECUDA, std::string("decode: memset: ") + cudaGetErrorString(e));
  return launch_decode_mma(c, q, K, V, idx, cnt, k, seq_lens, dense, units, NH, ns, rps, (float*)ws,
                           tickets, out, lse, partial, st, false);
}

// Sparse decode inside socket_decode_step: no ticket memset (the step prologue
// clears the tickets), PDL launch.  With tickets_out != nullptr it only
// reports where the tickets live and how many units there are (no launch).
socket_status launch_decode_pdl(const socket_cfg& c, const void* q, const void* K, const void* V,
                                const int32_t* idx, const int32_t* cnt, int k, void* out,
                                float* lse, void* ws, size_t ws_bytes, cudaStream_t st, bool pdl,
                                int** tickets_out, int* n_units) {
  int units, NH, ns, rps;
  decode_geometry(c, k, false, units, NH, ns, rps);
  if (ws_bytes < part_bytes(c, ns) + (size_t)units * sizeof(int))
    return fail(SOCKET_EWORKSPACE, "decode: workspace too small");
  if (NH > 8) return fail(SOCKET_EUNSUPPORTED, "decode: more than 8 query heads per selection row");
  int* tickets = reinterpret_cast<int*>(static_cast<char*>(ws) + part_bytes(c, ns));
  if (tickets_out) {
    *tickets_out = tickets;
    *n_units = units;
    return SOCKET_OK;
  }
  if (units == 0) return SOCKET_OK;
  return launch_decode_mma(c, q, K, V, idx, cnt, k, nullptr, false, units, NH, ns, rps, (float*)ws,
                           tickets, out, lse, nullptr, st, pdl);
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
