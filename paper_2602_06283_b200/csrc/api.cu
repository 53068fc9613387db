// extern "C" boundary of libsocket_b200: argument validation, workspace
// carving, launches.  See include/socket_b200.h for the contract.
#include <cmath>
#include <string>

#include "internal.cuh"

namespace sk {

bool one_launch_step(const socket_cfg& c);

static thread_local std::string g_last_error;

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

void set_error(const std::string& msg) { g_last_error = msg; }
socket_status fail(socket_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}
socket_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SOCKET_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return SOCKET_OK;
}

static socket_status validate(const socket_cfg* c) {
  if (!c) return fail(SOCKET_EINVAL, "cfg is NULL");
  if (c->B < 0 || c->H_q < 1 || c->H_kv < 1 || c->N_max < 0)
    return fail(SOCKET_EINVAL, "B, H_q, H_kv, N_max must be non-negative (heads >= 1)");
  if (c->H_q % c->H_kv != 0) return fail(SOCKET_EINVAL, "H_q % H_kv != 0");
  if (c->d != kD) {
    if (c->d <= 0) return fail(SOCKET_EINVAL, "d must be positive");
    return fail(SOCKET_EUNSUPPORTED, "only d = 128 is implemented");
  }
  if (c->N_max % 32 != 0) return fail(SOCKET_EINVAL, "N_max must be a multiple of 32");
  if (c->L < 1) return fail(SOCKET_EINVAL, "L must be >= 1");
  if (c->L > 128) return fail(SOCKET_EUNSUPPORTED, "L > 128 not implemented");
  if (c->P < 1 || c->P > 16) return fail(SOCKET_EINVAL, "P must be in [1, 16]");
  if (!(c->tau > 0.f) || !std::isfinite(c->tau)) return fail(SOCKET_EINVAL, "tau must be > 0");
  if (!std::isfinite(c->sm_scale)) return fail(SOCKET_EINVAL, "sm_scale must be finite");
  if (c->group_mode != SOCKET_GROUP_KV_SHARED && c->group_mode != SOCKET_GROUP_PER_QHEAD)
    return fail(SOCKET_EINVAL, "unknown group_mode");
  if (c->scoring != SOCKET_SCORING_SOFT && c->scoring != SOCKET_SCORING_HARD)
    return fail(SOCKET_EINVAL, "unknown scoring");
  if (c->flags & ~(SOCKET_FLAG_CHAINED_STEP | SOCKET_FLAG_ONE_LAUNCH)) return fail(SOCKET_EINVAL, "unknown flags");
  if (c->index_base < 0) return fail(SOCKET_EINVAL, "index_base must be >= 0");
  return SOCKET_OK;
}

#define SK_CHECK(x)                   \
  do {                                \
    socket_status _s = (x);           \
    if (_s != SOCKET_OK) return _s;   \
  } while (0)
#define SK_NONNULL(p) \
  if (!(p)) return fail(SOCKET_EINVAL, #p " is NULL")

static inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

static size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

}  // namespace sk

using namespace sk;

extern "C" {

int32_t socket_version(void) { return SOCKET_ABI_VERSION; }

const char* socket_last_error(void) { return g_last_error.c_str(); }

int32_t socket_code_slots(int32_t L) { return code_slots(L); }

size_t socket_codes_bytes(const socket_cfg* c) {
  if (!c) return 0;
  return (size_t)c->B * c->H_kv * c->N_max * code_bytes_per_key(c->L, c->P);
}

size_t socket_workspace_bytes(const socket_cfg* c, int32_t op, int32_t k) {
  if (validate(c) != SOCKET_OK) return 0;
  switch (op) {
    case SOCKET_OP_SCORE:
      return align16((size_t)c->B * num_sel_rows(*c) * lut_row_bytes(*c));
    case SOCKET_OP_SPARSE_DECODE:
      return align16(decode_workspace_bytes(*c, k > 0 ? k : 1, false));
    case SOCKET_OP_DENSE_DECODE:
      return align16(decode_workspace_bytes(*c, 1, true));
    case SOCKET_OP_DECODE_STEP:
      return align16(decode_step_workspace_bytes(*c, k > 0 ? k : 1));
    case SOCKET_OP_TOPK:
    case SOCKET_OP_RESOLVE:
      return align16(topk_workspace_bytes(*c));
    default:
      return 0;
  }
}

socket_status socket_hash_keys(const socket_cfg* cfg, const void* K, const void* V,
                               int32_t n_begin, int32_t n_count, const void* W, uint8_t* codes,
                               float* vnorm, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(K);
  SK_NONNULL(W);
  SK_NONNULL(codes);
  if ((V == nullptr) != (vnorm == nullptr)) return fail(SOCKET_EINVAL, "V and vnorm must both be set or both NULL");
  if (n_begin < 0 || n_count < 0 || (long long)n_begin + n_count > cfg->N_max)
    return fail(SOCKET_EINVAL, "bad [n_begin, n_begin + n_count) range");
  if (cfg->B == 0) return SOCKET_OK;
  return launch_hash_keys(*cfg, K, V, n_begin, n_count, W, codes, vnorm, S(stream));
}

socket_status socket_pack_codes(const socket_cfg* cfg, const uint8_t* plain, uint8_t* codes,
                                void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(plain);
  SK_NONNULL(codes);
  return launch_pack_codes(*cfg, plain, codes, false, S(stream));
}

socket_status socket_unpack_codes(const socket_cfg* cfg, const uint8_t* codes, uint8_t* plain,
                                  void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(plain);
  SK_NONNULL(codes);
  return launch_pack_codes(*cfg, plain, const_cast<uint8_t*>(codes), true, S(stream));
}

socket_status socket_query_tables(const socket_cfg* cfg, const void* q, const void* W,
                                  float* tables, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(q);
  SK_NONNULL(W);
  SK_NONNULL(tables);
  if (cfg->B == 0) return SOCKET_OK;
  return launch_query_tables(*cfg, q, W, tables, nullptr, S(stream));
}

socket_status socket_score(const socket_cfg* cfg, const void* q, const void* W,
                           const uint8_t* codes, const float* vnorm, const int32_t* seq_lens,
                           const uint8_t* mask, float* scores, void* ws, size_t ws_bytes,
                           void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(q);
  SK_NONNULL(W);
  SK_NONNULL(codes);
  SK_NONNULL(vnorm);
  SK_NONNULL(seq_lens);
  SK_NONNULL(scores);
  const size_t need = socket_workspace_bytes(cfg, SOCKET_OP_SCORE, 0);
  if (need && (!ws || ws_bytes < need)) return fail(SOCKET_EWORKSPACE, "score: workspace too small");
  if (cfg->B == 0 || cfg->N_max == 0) return SOCKET_OK;
  float* lut = static_cast<float*>(ws);
  SK_CHECK(launch_query_tables(*cfg, q, W, nullptr, lut, S(stream)));
  return launch_score(*cfg, lut, codes, vnorm, seq_lens, mask, scores, S(stream));
}

socket_status socket_build_lut(const socket_cfg* cfg, const void* q, const void* W, void* lut,
                               size_t lut_bytes, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(q);
  SK_NONNULL(W);
  SK_NONNULL(lut);
  if (lut_bytes < socket_workspace_bytes(cfg, SOCKET_OP_SCORE, 0))
    return fail(SOCKET_EWORKSPACE, "build_lut: buffer too small");
  if (cfg->B == 0) return SOCKET_OK;
  return launch_query_tables(*cfg, q, W, nullptr, static_cast<float*>(lut), S(stream));
}

socket_status socket_score_lut(const socket_cfg* cfg, const void* lut, const uint8_t* codes,
                               const float* vnorm, const int32_t* seq_lens, const uint8_t* mask,
                               float* scores, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(lut);
  SK_NONNULL(codes);
  SK_NONNULL(vnorm);
  SK_NONNULL(seq_lens);
  SK_NONNULL(scores);
  if (cfg->B == 0 || cfg->N_max == 0) return SOCKET_OK;
  return launch_score(*cfg, static_cast<const float*>(lut), codes, vnorm, seq_lens, mask, scores,
                      S(stream));
}

socket_status socket_decode_step(const socket_cfg* cfg, const void* q, void* K, void* V,
                                 const void* W, uint8_t* codes, float* vnorm,
                                 const int32_t* seq_lens, const uint8_t* mask,
                                 int32_t append_last, const void* k_new, const void* v_new,
                                 int32_t k, int32_t sink, int32_t window,
                                 float* scores, int32_t* idx, int32_t* cnt, void* out, float* lse,
                                 void* ws, size_t ws_bytes, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(q);
  SK_NONNULL(K);
  SK_NONNULL(V);
  SK_NONNULL(W);
  SK_NONNULL(codes);
  SK_NONNULL(vnorm);
  SK_NONNULL(seq_lens);
  SK_NONNULL(scores);
  SK_NONNULL(idx);
  SK_NONNULL(cnt);
  SK_NONNULL(out);
  SK_NONNULL(ws);
  if ((k_new == nullptr) != (v_new == nullptr)) return fail(SOCKET_EINVAL, "k_new and v_new must both be set or both NULL");
  if (k_new && !append_last) return fail(SOCKET_EINVAL, "k_new / v_new need append_last");
  if (cfg->index_base != 0) return fail(SOCKET_EUNSUPPORTED, "decode step: index_base must be 0");
  if (k <= 0) return fail(SOCKET_EINVAL, "k must be >= 1");
  if (k > cfg->N_max) return fail(SOCKET_EINVAL, "k > N_max");
  if (sink < 0 || window < 0 || (long long)sink + window > k)
    return fail(SOCKET_EINVAL, "need 0 <= sink, window and sink + window <= k");
  if (cfg->B == 0 || cfg->N_max == 0) return SOCKET_OK;
  return launch_decode_step(*cfg, q, K, V, W, codes, vnorm, seq_lens, mask, append_last != 0,
                            k_new, v_new, k, sink, window, scores, idx, cnt, out, lse, ws, ws_bytes,
                            S(stream));
}

int32_t socket_decode_step_launches(const socket_cfg* cfg) {
  if (validate(cfg) != SOCKET_OK) return 0;
  return one_launch_step(*cfg) ? 1 : 4;
}

static socket_status check_topk_args(int32_t k, int32_t sink, int32_t window) {
  if (k <= 0) return fail(SOCKET_EINVAL, "k must be >= 1");
  if (sink < 0 || window < 0 || (long long)sink + window > k)
    return fail(SOCKET_EINVAL, "need 0 <= sink, window and sink + window <= k");
  return SOCKET_OK;
}

socket_status socket_topk(const socket_cfg* cfg, const float* scores, const int32_t* seq_lens,
                          int32_t k, int32_t sink, int32_t window, int32_t* idx, int32_t* cnt,
                          float* sel_scores, void* ws, size_t ws_bytes, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(scores);
  SK_NONNULL(seq_lens);
  SK_NONNULL(idx);
  SK_NONNULL(cnt);
  SK_CHECK(check_topk_args(k, sink, window));
  if (k > cfg->N_max) return fail(SOCKET_EINVAL, "k > N_max");
  if (cfg->B == 0) return SOCKET_OK;
  return launch_topk(*cfg, scores, seq_lens, k, sink, window, idx, cnt, sel_scores, ws, ws_bytes,
                     S(stream));
}

socket_status socket_topk_digest(const socket_cfg* cfg, const float* scores, const int32_t* seq_lens,
                                 int32_t k, int32_t sink, int32_t window, int32_t shards, int32_t Q,
                                 uint32_t* digest, void* ws, size_t ws_bytes, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(scores);
  SK_NONNULL(seq_lens);
  SK_NONNULL(digest);
  SK_CHECK(check_topk_args(k, sink, window));
  if (shards < 1 || shards > SOCKET_MAX_SHARDS) return fail(SOCKET_EINVAL, "shards must be in [1, 64]");
  if (Q < 4 || Q > 1024) return fail(SOCKET_EINVAL, "Q must be in [4, 1024]");
  if (cfg->B == 0) return SOCKET_OK;
  return launch_topk_digest(*cfg, scores, seq_lens, k, sink, window, shards, Q, digest, ws, ws_bytes,
                            S(stream));
}

socket_status socket_topk_bracket(const socket_cfg* cfg, const uint32_t* all_digests, int32_t G,
                                  int32_t Q, int32_t k, uint32_t* state, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(all_digests);
  SK_NONNULL(state);
  if (G < 1 || G > SOCKET_MAX_SHARDS) return fail(SOCKET_EINVAL, "G must be in [1, 64]");
  if (Q < 4 || Q > 1024 || (size_t)2 * G * Q * 4 > 200 * 1024)
    return fail(SOCKET_EINVAL, "Q must be in [4, 1024] and G * Q <= 25600");
  if (k <= 0) return fail(SOCKET_EINVAL, "k must be >= 1");
  if (cfg->B == 0) return SOCKET_OK;
  return launch_topk_bracket(*cfg, all_digests, G, Q, k, state, S(stream));
}

socket_status socket_topk_window(const socket_cfg* cfg, const float* scores, const int32_t* seq_lens,
                                 int32_t sink, int32_t window, const uint32_t* state, uint32_t* msg,
                                 void* ws, size_t ws_bytes, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(scores);
  SK_NONNULL(seq_lens);
  SK_NONNULL(state);
  SK_NONNULL(msg);
  if (sink < 0 || window < 0) return fail(SOCKET_EINVAL, "need 0 <= sink, window");
  if (cfg->B == 0) return SOCKET_OK;
  return launch_topk_window(*cfg, scores, seq_lens, sink, window, state, msg, ws, ws_bytes, S(stream));
}

socket_status socket_topk_resolve(const socket_cfg* cfg, const uint32_t* all_msgs, int32_t G,
                                  int32_t rank, uint32_t* state, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(all_msgs);
  SK_NONNULL(state);
  if (G < 1 || G > SOCKET_MAX_SHARDS || rank < 0 || rank >= G)
    return fail(SOCKET_EINVAL, "need 1 <= G <= 64 and 0 <= rank < G");
  if (cfg->B == 0) return SOCKET_OK;
  return launch_topk_resolve(*cfg, all_msgs, G, rank, state, S(stream));
}

socket_status socket_topk_emit(const socket_cfg* cfg, const float* scores, const int32_t* seq_lens,
                               int32_t k, int32_t sink, int32_t window, const uint32_t* state,
                               int32_t* idx, int32_t* cnt, float* sel_scores, void* ws,
                               size_t ws_bytes, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(scores);
  SK_NONNULL(seq_lens);
  SK_NONNULL(state);
  SK_NONNULL(idx);
  SK_NONNULL(cnt);
  SK_CHECK(check_topk_args(k, sink, window));
  if (cfg->B == 0) return SOCKET_OK;
  return launch_topk_emit(*cfg, scores, seq_lens, k, sink, window, state, idx, cnt, sel_scores, ws,
                          ws_bytes, S(stream));
}

socket_status socket_sparse_decode(const socket_cfg* cfg, const void* q, const void* K,
                                   const void* V, const int32_t* idx, const int32_t* cnt,
                                   int32_t k, void* out, float* lse, float* partial, void* ws,
                                   size_t ws_bytes, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(q);
  SK_NONNULL(K);
  SK_NONNULL(V);
  SK_NONNULL(idx);
  SK_NONNULL(cnt);
  SK_NONNULL(ws);
  if (!out && !partial) return fail(SOCKET_EINVAL, "out and partial are both NULL");
  if (lse && !out) return fail(SOCKET_EINVAL, "lse requires out");
  if (k <= 0) return fail(SOCKET_EINVAL, "k must be >= 1");
  if (cfg->B == 0) return SOCKET_OK;
  return launch_decode(*cfg, q, K, V, idx, cnt, k, nullptr, false, out, lse, partial, ws,
                       ws_bytes, S(stream));
}

socket_status socket_dense_decode(const socket_cfg* cfg, const void* q, const void* K,
                                  const void* V, const int32_t* seq_lens, void* out, float* lse,
                                  void* ws, size_t ws_bytes, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(q);
  SK_NONNULL(K);
  SK_NONNULL(V);
  SK_NONNULL(seq_lens);
  SK_NONNULL(out);
  SK_NONNULL(ws);
  if (cfg->B == 0) return SOCKET_OK;
  return launch_decode(*cfg, q, K, V, nullptr, nullptr, 1, seq_lens, true, out, lse, nullptr, ws,
                       ws_bytes, S(stream));
}

socket_status socket_sample_decode(const socket_cfg* cfg, const float* scores, const float* vnorm,
                                   const void* V, const int32_t* seq_lens, const float* uniforms,
                                   int32_t M, int32_t* samples, void* out, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(scores);
  SK_NONNULL(vnorm);
  SK_NONNULL(V);
  SK_NONNULL(seq_lens);
  SK_NONNULL(uniforms);
  SK_NONNULL(out);
  if (cfg->index_base != 0) return fail(SOCKET_EUNSUPPORTED, "sample decode: index_base must be 0");
  return launch_sample_decode(*cfg, scores, vnorm, V, seq_lens, uniforms, M, samples, out, S(stream));
}

socket_status socket_lse_combine(const socket_cfg* cfg, const float* partials, int32_t G,
                                 void* out, float* lse, void* stream) {
  SK_CHECK(validate(cfg));
  SK_NONNULL(partials);
  SK_NONNULL(out);
  if (G < 1) return fail(SOCKET_EINVAL, "G must be >= 1");
  return launch_lse_combine(*cfg, partials, G, out, lse, S(stream));
}

}  // extern "C"
