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
#include <algorithm>

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
                              float* sel_scores, cudaStream_t st, bool pdl, void* ws, size_t ws_bytes);
socket_status launch_decode_pdl(const socket_cfg& c, const void* q, const void* K, const void* V,
                                const int32_t* idx, const int32_t* cnt, int k, void* out,
                                float* lse, void* ws, size_t ws_bytes, cudaStream_t st, bool pdl,
                                int** tickets_out, int* n_units);
size_t decode_workspace_bytes(const socket_cfg& c, int k, bool dense);
bool spread_geometry(const socket_cfg& c, int& C, int& S);
size_t spread_workspace_bytes(const socket_cfg& c);
socket_status launch_spread_step(const socket_cfg& c, const void* q, void* K, void* V,
                                 const void* W, uint8_t* codes, float* vnorm, const int32_t* seq_lens,
                                 const uint8_t* mask, int do_append, const void* k_new,
                                 const void* v_new, int k, int sink, int window,
                                 float* scores, int32_t* idx, int32_t* cnt, void* out, float* lse,
                                 void* ws, cudaStream_t st);

// one-launch row-spread step (spread.cu): by default up to 32 selection rows
// (measured against the chained kernels, DESIGN 4.5b: -21..24% at B = 2, -10% at
// B = 3 and -5% at B = 4 (32K); larger shapes fall back to the chained kernels by
// geometry); SOCKET_FLAG_ONE_LAUNCH whenever the shape allows
constexpr int kSpreadMaxRows = 32;
bool one_launch_step(const socket_cfg& c) {
  if (c.flags & SOCKET_FLAG_CHAINED_STEP) return false;
  int C, S;
  if (!spread_geometry(c, C, S)) return false;
  return (c.flags & SOCKET_FLAG_ONE_LAUNCH) || (long long)c.B * c.H_kv <= kSpreadMaxRows;
}

socket_status launch_prologue(const socket_cfg& c, ProArgs a, bool tables, cudaStream_t st) {
  const int NH = c.group_mode == SOCKET_GROUP_PER_QHEAD ? 1 : c.H_q / c.H_kv;
  if (tables && NH != 1 && NH != 2 && NH != 4 && NH != 8)
    return fail(SOCKET_EUNSUPPORTED, "tables: heads per selection row must be 1, 2, 4 or 8");
  a.B = c.B;
  a.H_q = c.H_q;
  a.H_sel = num_sel_rows(c);
  a.H_kv = c.H_kv;
  a.N_max = c.N_max;
  a.L = c.L;
  a.P = c.P;
  a.Lp = code_slots_p(c.L, c.P);
  a.tau = c.tau;
  a.hard = c.scoring == SOCKET_SCORING_HARD;
  a.tpt = c.P > 8 ? 64 / c.P : kTT;
  a.n_wtiles = (a.Lp + a.tpt - 1) / a.tpt;
  a.n_tab_ctas = tables ? (c.B * c.H_q + kTQ - 1) / kTQ * a.n_wtiles : 0;
  const int n_app = (a.n_keys + kAK - 1) / kAK * a.n_wtiles;
  const int grid = a.n_tab_ctas + n_app;
  if (grid == 0) return SOCKET_OK;
  const size_t sm = prologue_smem_bytes();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kPT);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
#define SK_PRO(N)                                                                              \
  case N:                                                                                      \
    cudaFuncSetAttribute(prologue_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    if (cudaLaunchKernelEx(&cfg, prologue_kernel<N>, a) != cudaSuccess)                        \
      return check_launch("prologue_kernel");                                                  \
    break;
  switch (tables ? NH : 1) { SK_PRO(1) SK_PRO(2) SK_PRO(4) SK_PRO(8) }
#undef SK_PRO
  return check_launch("prologue_kernel");
}

// Host-resident step inputs (pinned, UVA-mapped q / k_new / v_new): one copy
// kernel pulls them into the workspace before the prologue -- 16-B loads, all in
// flight at once, so the PCIe reads overlap (a DMA copy of the same 192 KB took
// ~16 us in tools/e2e_probe3.py).
size_t stage_bytes(const socket_cfg& c);
static size_t chained_ws_bytes(const socket_cfg& c, int k);
size_t stage_bytes(const socket_cfg& c) {
  return (((size_t)c.B * c.H_q * kD + 2 * (size_t)c.B * c.H_kv * kD) * 2 + 255) & ~(size_t)255;
}

constexpr int kStageThreads = 256;
__global__ void __launch_bounds__(256) stage_inputs_kernel(const uint4* q_h, const uint4* k_h,
                                                           const uint4* v_h, uint4* dst, int nq, int nk) {
  const int n = nq + 2 * nk;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint4* src = i < nq ? q_h + i : (i < nq + nk ? k_h + (i - nq) : v_h + (i - nq - nk));
    dst[i] = *src;
  }
}

static bool host_resident(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

static size_t chained_ws_bytes(const socket_cfg& c, int k) {
  const size_t lut = ((size_t)c.B * num_sel_rows(c) * lut_row_bytes(c) + 255) & ~(size_t)255;
  return lut + ((decode_workspace_bytes(c, k, false) + 255) & ~(size_t)255) + stage_bytes(c) +
         ((topk_workspace_bytes(c) + 255) & ~(size_t)255);
}
// [chained-path regions | row-spread control region]; the latter must be zero
// before the first step (every step leaves it zero) and no other path writes it
size_t decode_step_workspace_bytes(const socket_cfg& c, int k) {
  return chained_ws_bytes(c, k) + spread_workspace_bytes(c);
}

bool decode_step_stages_inputs(const socket_cfg& c, const void* q, const void* k_new, const void* v_new) {
  return !one_launch_step(c) && (host_resident(q) || host_resident(k_new) || host_resident(v_new));
}

socket_status launch_decode_step(const socket_cfg& c, const void* q, void* K, void* V,
                                 const void* W, uint8_t* codes, float* vnorm,
                                 const int32_t* seq_lens, const uint8_t* mask, int do_append,
                                 const void* k_new, const void* v_new, int k, int sink, int window,
                                 float* scores, int32_t* idx, int32_t* cnt, void* out, float* lse,
                                 void* ws, size_t ws_bytes, cudaStream_t st) {
  const int Lp = code_slots_p(c.L, c.P);
  if (Lp > 64) return fail(SOCKET_EUNSUPPORTED, "decode step: L > 64 not supported");
  const int H_sel = num_sel_rows(c);
  const int NH = c.group_mode == SOCKET_GROUP_PER_QHEAD ? 1 : c.H_q / c.H_kv;
  if (NH != 1 && NH != 2 && NH != 4 && NH != 8)
    return fail(SOCKET_EUNSUPPORTED, "decode step: heads per selection row must be 1, 2, 4 or 8");
  const size_t lut_bytes = ((size_t)c.B * H_sel * lut_row_bytes(c) + 255) & ~(size_t)255;
  if (ws_bytes < decode_step_workspace_bytes(c, k))
    return fail(SOCKET_EWORKSPACE, "decode step: workspace too small");
  // small batch: one launch over all SMs
  if (one_launch_step(c))
    return launch_spread_step(c, q, K, V, W, codes, vnorm, seq_lens, mask, do_append, k_new, v_new, k,
                              sink, window, scores, idx, cnt, out, lse,
                              static_cast<char*>(ws) + chained_ws_bytes(c, k), st);
  float* lut = static_cast<float*>(ws);
  void* dws = static_cast<char*>(ws) + lut_bytes;
  const size_t dws_bytes = (decode_workspace_bytes(c, k, false) + 255) & ~(size_t)255;
  // ---- host-resident inputs: stage them into the workspace first --------------
  const bool staged = decode_step_stages_inputs(c, q, k_new, v_new);
  if (staged) {
    const int nq = c.B * c.H_q * kD / 8, nk = c.B * c.H_kv * kD / 8;   // 16-B chunks
    uint16_t* stage = reinterpret_cast<uint16_t*>(static_cast<char*>(dws) + dws_bytes);
    const bool has_new = k_new != nullptr && v_new != nullptr;
    const int nk_used = has_new ? nk : 0;
    const int n = nq + 2 * nk_used;
    const int blocks = std::min((n + kStageThreads - 1) / kStageThreads, 2 * num_sms());
    stage_inputs_kernel<<<blocks, kStageThreads, 0, st>>>(static_cast<const uint4*>(q),
                                                static_cast<const uint4*>(k_new),
                                                static_cast<const uint4*>(v_new),
                                                reinterpret_cast<uint4*>(stage), nq, nk_used);
    socket_status s0 = check_launch("stage_inputs_kernel");
    if (s0 != SOCKET_OK) return s0;
    q = stage;
    if (has_new) {
      k_new = stage + (size_t)nq * 8;
      v_new = stage + (size_t)(nq + nk) * 8;
    }
  }
  // decode tickets live at the end of the decode workspace; find them without launching
  int* tickets = nullptr;
  int n_units = 0;
  socket_status s = launch_decode_pdl(c, q, K, V, idx, cnt, k, out, lse, dws, dws_bytes, st, false,
                                      &tickets, &n_units);   // query only (tickets_out != null)
  if (s != SOCKET_OK) return s;
  // ---- prologue: tables || append ---------------------------------------------
  ProArgs pa = {};
  pa.q = (const uint16_t*)q;
  pa.W = (const uint16_t*)W;
  pa.lut = lut;
  pa.K = (const uint16_t*)K;
  pa.V = (const uint16_t*)V;
  pa.k_new = (const uint16_t*)k_new;
  pa.v_new = (const uint16_t*)v_new;
  pa.K_w = (uint16_t*)K;
  pa.V_w = (uint16_t*)V;
  pa.codes = codes;
  pa.vnorm = vnorm;
  pa.seq_lens = seq_lens;
  pa.tickets = tickets;
  pa.n_tickets = n_units;
  pa.n_keys = do_append ? c.B * c.H_kv : 0;
  pa.n_begin = 0;
  pa.n_count = 1;
  pa.append_last = 1;
  pa.pdl = staged ? 1 : 0;           // PDL edge after the staging kernel
  s = launch_prologue(c, pa, true, st);
  if (s != SOCKET_OK) return s;
  // ---- score, top-k, decode (PDL chain) ----------------------------------------
  s = launch_score_pdl(c, lut, codes, vnorm, seq_lens, mask, scores, st, true);
  if (s != SOCKET_OK) return s;
  const size_t tws_bytes = topk_workspace_bytes(c);   // key slices of rows > 655360 keys
  void* tws = static_cast<char*>(dws) + dws_bytes + stage_bytes(c);
  s = launch_topk_pdl(c, scores, seq_lens, k, sink, window, idx, cnt, nullptr, st, true, tws, tws_bytes);
  if (s != SOCKET_OK) return s;
  return launch_decode_pdl(c, q, K, V, idx, cnt, k, out, lse, dws, dws_bytes, st, true, nullptr,
                           nullptr);
}

}  // namespace sk
