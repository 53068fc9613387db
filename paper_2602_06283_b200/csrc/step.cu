// One SOCKET decode step as a single library call (socket_decode_step):
//
//   prologue   one launch, two CTA roles running concurrently:
//                tables CTAs -> Alg. 2 LUT images of every selection row
//                append CTAs -> Alg. 1 on the newest key of every (b, kv head)
//                               (j = seq_lens[b] - 1) + its value norm
//              and it clears the decode tickets (no memset node);
//   score      Eq. 4 / Alg. 4 from the LUT images          (PDL-chained)
//   top-k      Alg. 3 l.244                                 (PDL-chained)
//   decode     Eq. 2 split flash-decode + fused LSE combine (PDL-chained)
//
// PDL (programmatic dependent launch): each dependent kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization and executes
// griddepcontrol.wait before it reads its predecessor's output, so its launch
// and prologue overlap the predecessor's tail.  Inside a CUDA graph the edges
// become programmatic dependencies.
#include "step_dev.cuh"

namespace sk {

#ifdef SK_TRACE
// reads this translation unit's copy (the decode-step prologue)
extern "C" int socket_debug_prologue_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_pro_trace, (size_t)n * sizeof(unsigned long long));
}
#endif

socket_status launch_score_pdl(const socket_cfg& c, const float* lut, const uint8_t* codes,
                               const float* vnorm, const int32_t* seq_lens, const uint8_t* mask,
                               float* scores, cudaStream_t st, bool pdl);
socket_status launch_topk_pdl(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                              int k, int sink, int window, int32_t* idx, int32_t* cnt,
                              float* sel_scores, cudaStream_t st, bool pdl);
socket_status launch_decode_pdl(const socket_cfg& c, const void* q, const void* K, const void* V,
                                const int32_t* idx, const int32_t* cnt, int k, void* out,
                                float* lse, void* ws, size_t ws_bytes, cudaStream_t st, bool pdl,
                                int** tickets_out, int* n_units);
size_t decode_workspace_bytes(const socket_cfg& c, int k, bool dense);

template <int NH>
__global__ void __launch_bounds__(kTabThreads)
step_prologue_kernel(const uint16_t* __restrict__ q, const uint16_t* __restrict__ W,
                     float* __restrict__ lut, const uint16_t* __restrict__ K,
                     const uint16_t* __restrict__ V, uint8_t* __restrict__ codes,
                     float* __restrict__ vnorm, const int32_t* __restrict__ seq_lens,
                     int* __restrict__ tickets, int n_tickets, int H_q, int H_sel, int H_kv,
                     int N_max, int L, int P, int Lp, float tau, int n_table_ctas, int tchunks) {
  extern __shared__ __align__(16) char tsm[];
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < n_tickets; i += blockDim.x) tickets[i] = 0;
  if ((int)blockIdx.x < n_table_ctas) {
    tables_cta<NH>(q, W, nullptr, lut, H_q, H_sel, L, P, Lp, tau, blockIdx.x / tchunks,
                   (blockIdx.x % tchunks) * kTabPerCta, tsm);
  } else {
    const int a = (int)blockIdx.x - n_table_ctas;
    append_cta(K, W, codes, V, vnorm, N_max, L, P, Lp, 0, 1, 1, seq_lens, H_kv, a / tchunks,
               (a % tchunks) * kTabPerCta, reinterpret_cast<float*>(tsm));
  }
}

size_t decode_step_workspace_bytes(const socket_cfg& c, int k) {
  const size_t lut = ((size_t)c.B * num_sel_rows(c) * lut_bytes_per_row(c.L) + 255) & ~(size_t)255;
  return lut + decode_workspace_bytes(c, k, false);
}

socket_status launch_decode_step(const socket_cfg& c, const void* q, const void* K, const void* V,
                                 const void* W, uint8_t* codes, float* vnorm,
                                 const int32_t* seq_lens, const uint8_t* mask, int do_append, int k,
                                 int sink, int window, float* scores, int32_t* idx, int32_t* cnt,
                                 void* out, float* lse, void* ws, size_t ws_bytes,
                                 cudaStream_t st) {
  const int Lp = code_slots(c.L);
  if (Lp > 64) return fail(SOCKET_EUNSUPPORTED, "decode step: L > 64 not supported");
  const int H_sel = num_sel_rows(c);
  const int NH = c.group_mode == SOCKET_GROUP_PER_QHEAD ? 1 : c.H_q / c.H_kv;
  if (NH != 1 && NH != 2 && NH != 4 && NH != 8)
    return fail(SOCKET_EUNSUPPORTED, "decode step: heads per selection row must be 1, 2, 4 or 8");
  const size_t lut_bytes = ((size_t)c.B * H_sel * lut_bytes_per_row(c.L) + 255) & ~(size_t)255;
  if (ws_bytes < decode_step_workspace_bytes(c, k))
    return fail(SOCKET_EWORKSPACE, "decode step: workspace too small");
  float* lut = static_cast<float*>(ws);
  void* dws = static_cast<char*>(ws) + lut_bytes;
  const size_t dws_bytes = ws_bytes - lut_bytes;
  // decode tickets live at the end of the decode workspace; find them without launching
  int* tickets = nullptr;
  int n_units = 0;
  socket_status s = launch_decode_pdl(c, q, K, V, idx, cnt, k, out, lse, dws, dws_bytes, st, false,
                                      &tickets, &n_units);   // query only (tickets_out != null)
  if (s != SOCKET_OK) return s;
  // ---- prologue ---------------------------------------------------------------
  const int tchunks = (Lp + kTabPerCta - 1) / kTabPerCta;
  const int n_table_ctas = c.B * H_sel * tchunks;
  const int n_keys = c.B * c.H_kv;
  const int n_append_ctas = do_append ? n_keys * tchunks : 0;
  const dim3 grid(n_table_ctas + n_append_ctas);
#define SK_PRO(N)                                                                                   \
  case N: {                                                                                         \
    const size_t sm = tables_smem_bytes(N);                                                         \
    cudaFuncSetAttribute(step_prologue_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    step_prologue_kernel<N><<<grid, kTabThreads, sm, st>>>(                                         \
        (const uint16_t*)q, (const uint16_t*)W, lut, (const uint16_t*)K, (const uint16_t*)V, codes, \
        vnorm, seq_lens, tickets, n_units, c.H_q, H_sel, c.H_kv, c.N_max, c.L, c.P, Lp, c.tau,     \
        n_table_ctas, tchunks);                                                                     \
    break;                                                                                          \
  }
  switch (NH) { SK_PRO(1) SK_PRO(2) SK_PRO(4) SK_PRO(8) }
#undef SK_PRO
  s = check_launch("step_prologue_kernel");
  if (s != SOCKET_OK) return s;
  // ---- score, top-k, decode (PDL chain) ----------------------------------------
  s = launch_score_pdl(c, lut, codes, vnorm, seq_lens, mask, scores, st, true);
  if (s != SOCKET_OK) return s;
  s = launch_topk_pdl(c, scores, seq_lens, k, sink, window, idx, cnt, nullptr, st, true);
  if (s != SOCKET_OK) return s;
  return launch_decode_pdl(c, q, K, V, idx, cnt, k, out, lse, dws, dws_bytes, st, true, nullptr,
                           nullptr);
}

}  // namespace sk
