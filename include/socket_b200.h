/*
 * socket_b200.h -- C ABI of the B200-native SOCKET decode hot path.
 *
 * SOCKET (arxiv 2602.06283) scores every cached key by a soft collision of
 * L SimHash buckets, keeps the top-k keys and runs exact attention over them.
 * Citations "P:L" are lines of the paper's text.
 *
 *   stage                      paper                                  entry point
 *   key hashing (prefill)      Alg. 1, P:194-209, P:263               socket_hash_keys
 *   query soft hashing         Alg. 2, P:211-225                      socket_query_tables
 *   soft-collision scoring     Eq. 4, Alg. 4 P:1485-1506    socket_score
 *   top-k selection            Alg. 3 l.244, P:686            socket_topk
 *   sparse flash-decode        Eq. 2 P:169-174, P:271, P:309, P:701   socket_sparse_decode
 *   LSE combine of partials    (Flash-Decode split merge)      socket_lse_combine
 *   dense decode (k = n)       Eq. 1 P:16-22                          socket_dense_decode
 *   whole decode step          P:259-271                              socket_decode_step
 *   sequence-shard top-k       exact global top-k over shards         socket_topk_digest,
 *                                                                     _bracket, _window,
 *                                                                     _resolve, _emit
 *
 * Conventions (all entry points)
 *  - Every pointer argument is DEVICE memory owned by the caller, except the
 *    `socket_cfg*` (host).  The library never allocates, frees or copies
 *    host<->device; temporary storage is the caller's `ws` buffer of at least
 *    socket_workspace_bytes(cfg, op, k) bytes (16-byte aligned).
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream).  No call synchronizes or reads device data
 *    on the host.
 *  - bf16 arrays are passed as `const void*` holding IEEE bfloat16 values.
 *  - Errors: host-side validation returns SOCKET_EINVAL (null required pointer,
 *    P not in [1,16], L < 1, d <= 0, tau <= 0, k <= 0, sink+window > k,
 *    H_q % H_kv != 0, N_max not a multiple of 32, index_base < 0, bad
 *    ranges);
 *    SOCKET_EUNSUPPORTED for valid but not implemented shapes;
 *    SOCKET_EWORKSPACE if ws_bytes is too small; SOCKET_ECUDA if a launch
 *    fails.  The message of the last non-OK status of the calling thread is
 *    returned by socket_last_error().  Nothing aborts, throws or prints.
 *  - Data-dependent conditions are not errors: k > #valid keys gives
 *    cnt = #valid; a row with no valid key gives cnt = 0, a zero output and
 *    lse = -inf.
 *  - Determinism: identical inputs give bit-identical outputs (no
 *    order-dependent atomics; top-k compaction is stable).
 */
#ifndef SOCKET_B200_H
#define SOCKET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SOCKET_ABI_VERSION 4

typedef enum {
  SOCKET_OK = 0,
  SOCKET_EINVAL = 1,
  SOCKET_EUNSUPPORTED = 2,
  SOCKET_ECUDA = 3,
  SOCKET_EWORKSPACE = 4
} socket_status;

/* How query heads of one GQA group share a selection (reading R-14;
 * the paper is single-query).
 *  KV_SHARED: one top-k per (b, KV head) from s_g(j) = ||v_j|| * sum_{h in g} w_hat_h(j);
 *             H_sel = H_kv selection rows; all G = H_q/H_kv query heads attend
 *             over the same selected rows.
 *  PER_QHEAD: one top-k per (b, query head) from s_h(j) = ||v_j|| * w_hat_h(j);
 *             H_sel = H_q selection rows (the paper's literal single-query form). */
typedef enum { SOCKET_GROUP_KV_SHARED = 0, SOCKET_GROUP_PER_QHEAD = 1 } socket_group_mode;

/* Which bucket weights the tables hold.
 *  SOFT: Alg. 2 soft bucket probabilities p_tau(r | q) -- SOCKET, Eq. 4;
 *  HARD: the indicator [r == b_q^(l)] of the query's own bucket (b_q by the key
 *        rule of Alg. 1, sign(0) = +1) -- traditional LSH, Eq. 3, so that the
 *        score is the collision count sum_l [b_j^(l) == b_q^(l)] (times ||v_j||,
 *        or a caller-supplied all-ones vnorm for the plain Eq. 3 count). */
typedef enum { SOCKET_SCORING_SOFT = 0, SOCKET_SCORING_HARD = 1 } socket_scoring;

typedef struct {
  int32_t B;          /* batch                                                     */
  int32_t H_q;        /* query heads                                               */
  int32_t H_kv;       /* key/value heads; H_q % H_kv == 0                          */
  int32_t d;          /* head dim; must be 128                                     */
  int32_t N_max;      /* token capacity = row stride of K/V/vnorm/scores; %32 == 0 */
  int32_t L;          /* hash tables, >= 1 (Alg. 1 "#tables L")                    */
  int32_t P;          /* hyperplanes per table, 1..16 (Alg. 1 "#hyperplanes P");    *
                       * P <= 8: one code byte per table slot; P = 9..16: P-bit  *
                       * codes tightly packed (socket_codes_bytes)              */
  float tau;          /* temperature > 0 (Alg. 2)                                  */
  float sm_scale;     /* softmax scale on q.k (reading R-2; usually 1/sqrt(d))     */
  int32_t group_mode; /* socket_group_mode                                         */
  int32_t scoring;    /* socket_scoring; 0 = soft scores (SOCKET, Eq. 4)           */
  int32_t flags;      /* SOCKET_FLAG_* bits; 0 = defaults                          */
  int64_t index_base; /* global token position of local row 0 of this buffer      *
                       * (sequence shards); 0 otherwise.   *
                       * Keys are at global positions index_base + j, and key j  *
                       * is valid iff index_base + j < seq_lens[b] (seq_lens are *
                       * always the sequences' TOTAL lengths).                   */
} socket_cfg;

/* socket_cfg.flags */
enum {
  /* socket_decode_step: never use the one-launch kernel, always the
   * PDL-chained kernels (both give bit-identical codes, scores and selections) */
  SOCKET_FLAG_CHAINED_STEP = 1,
  /* socket_decode_step: use the one-launch row-spread kernel whenever the shape
   * allows it (KV_SHARED, P <= 8, L <= 64, 2 B H_kv <= #SMs), not only for the
   * small grids where it is the default */
  SOCKET_FLAG_ONE_LAUNCH = 2
};

/* ------------------------------------------------------------------------ *
 * Data layouts (all row-major, innermost last)
 *   q       [B][H_q][d]            bf16
 *   K, V    [B][H_kv][N_max][d]    bf16   (256-byte rows for d = 128)
 *   W       [L][P][d]              bf16   projections W^(l) (Alg. 1 l.201);
 *                                         one W shared by every b and head
 *   vnorm   [B][H_kv][N_max]       fp32   ||v_j||_2
 *   seq_lens[B]                    int32  total length n_b of sequence b; local key j
 *                                         is valid iff index_base + j < n_b (so with
 *                                         index_base = 0: j < seq_lens[b]).  The
 *                                         contract is seq_lens[b] - index_base <= N_max
 *                                         for the calls that append (decode step);
 *                                         the others clamp to N_max.
 *   mask    [B][N_max]             uint8  optional; 0 = invalid key (Alg. 4 m_j)
 *   scores  [B][H_sel][N_max]      fp32   -inf for invalid keys (Alg. 4)
 *   idx     [B][H_sel][k]          int32  selected keys, ascending; -1 past cnt
 *   cnt     [B][H_sel]             int32
 *   out     [B][H_q][d]            bf16
 *   lse     [B][H_q]               fp32   natural-log sum of exp(sm_scale q.k) over S
 *   partial [B][H_q][d+2]          fp32   (m, l, o[d]): m = max logit, l = sum e^{z-m},
 *                                         o = sum e^{z-m} v  (unnormalised)
 *
 * Codes (the "index", Alg. 1 output b_j^(l)):  one byte per (key, table), in a
 * key-tiled, bank-rotated layout chosen for the score kernel:
 *   Lp  = socket_code_slots(L) = 8, 16, 32, or L rounded up to a multiple of 32
 *   M   = min(Lp, 32) - 1
 *   slot s of key j holds the bucket id of table  t(s, j) = (s & ~M) | ((s + j) & M)
 *   (slots with t >= L are padding and hold 0)
 *   CB  = min(Lp, 16)  bytes per chunk
 *   byte offset of (b, h, j, s) =
 *        ((b*H_kv + h) * N_max) * Lp
 *      + ((j >> 5) * (Lp / CB) + s / CB) * (32 * CB) + (j & 31) * CB + (s % CB)
 * Rotating each key's slots by j mod 32 makes the 32 lanes of a warp (lane =
 * key j mod 32) look up 32 different tables at every step, i.e. 32 different
 * shared-memory banks.
 *
 * Wide codes (P = 9..16, NEXT-2): the same slots and rotation with Lp =
 * max(32, socket_code_slots(L)), tightly packed -- Lp * P bits per key (640
 * bits for the 600 useful at L = 60, P = 10).  Per (b, h) region, 32-key tiles;
 * per tile and 32-slot group g (G = Lp / 32), the group's 32 slot codes form
 * one 32P-bit string, slot s at bits [s P, s P + P) LSB first, stored as P
 * uint32 words interleaved across the tile's keys:
 *   uint32 index of word w of group g of key j = (((j >> 5) * G + g) * P + w) * 32 + (j & 31)
 * (in units of uint32 from the start of the (b, h) region, which is
 * N_max * Lp * P / 8 bytes).
 * socket_pack_codes / socket_unpack_codes convert from / to the plain
 * [B][H_kv][L][N_max] layout (uint8 for P <= 8, uint16 for P > 8).
 * ------------------------------------------------------------------------ */

/* Slots per key of the byte-code layout (see above); 0 if L < 1. */
int32_t socket_code_slots(int32_t L);
/* Bytes of the codes buffer for cfg: B*H_kv*N_max*socket_code_slots(L) for
 * P <= 8, B*H_kv*N_max*Lp*P/8 (packed) for P > 8. */
size_t socket_codes_bytes(const socket_cfg* cfg);

/* Workspace requirement of an entry point (op = SOCKET_OP_*), for budget k. */
enum {
  SOCKET_OP_HASH = 0,
  SOCKET_OP_TABLES = 1,
  SOCKET_OP_SCORE = 2,
  SOCKET_OP_TOPK = 3,
  SOCKET_OP_SPARSE_DECODE = 4,
  SOCKET_OP_DENSE_DECODE = 5,
  SOCKET_OP_RESOLVE = 6,
  SOCKET_OP_DECODE_STEP = 7
};
size_t socket_workspace_bytes(const socket_cfg* cfg, int32_t op, int32_t k);

/* Alg. 1 PrecomputeKeyHashes, applied to token rows
 * [n_begin, n_begin + n_count) of every (b, kv head):
 *   x_{l,i}(j) = sum_t W[l][i][t] * K[b][h][j][t]   (fp32 accumulation)
 *   bit_i = (x_{l,i} >= 0)        -- sign(0) = +1, reading R-3
 *   b_j^(l) = sum_i bit_i << i    -- row i = bit i, LSB first, reading R-4
 * Writes those keys' codes (layout above) and, if V != NULL, vnorm[j] =
 * sqrt(sum_t V[j][t]^2) (fp32).  The per-step append of a decode step is the
 * call with n_count = 1.  V == NULL requires vnorm == NULL.
 * Requires 0 <= n_begin, n_begin + n_count <= N_max. */
socket_status socket_hash_keys(const socket_cfg* cfg, const void* K, const void* V,
                               int32_t n_begin, int32_t n_count, const void* W,
                               uint8_t* codes, float* vnorm, void* stream);

/* Layout converters for codes: plain [B][H_kv][L][N_max] uint8 <-> tiled layout. */
socket_status socket_pack_codes(const socket_cfg* cfg, const uint8_t* plain, uint8_t* codes,
                                void* stream);
socket_status socket_unpack_codes(const socket_cfg* cfg, const uint8_t* codes, uint8_t* plain,
                                  void* stream);

/* Alg. 2 SoftBucketProbs for every (b, selection row):
 *   u_{l,i} = tanh(W[l][i] . q) / sqrt(d)
 *   p_h^(l)(r) = softmax_r(u^(l) . c_r / tau),  c_{r,i} = +1 iff bit i of r (R-5),
 * evaluated in the exact product form prod_i sigma(2 u_i c_{r,i} / tau).
 * tables[b][row][l][r] (fp32, R = 2^P) = p_h (PER_QHEAD) or sum_{h in group} p_h
 * (KV_SHARED). */
socket_status socket_query_tables(const socket_cfg* cfg, const void* q, const void* W,
                                  float* tables, void* stream);

/* Eq. 4 + Alg. 4: for every (b, row) and key j < N_max
 *   w_hat(j) = sum_{l=0}^{L-1} T_row^(l)(b_j^(l))      (T from Alg. 2 as above)
 *   scores[b][row][j] = vnorm[b][g][j] * w_hat(j)        if j < seq_lens[b] and mask != 0
 *                     = -inf                             otherwise
 * (g = kv head of the row).  Computes the tables itself (into ws). */
socket_status socket_score(const socket_cfg* cfg, const void* q, const void* W,
                           const uint8_t* codes, const float* vnorm, const int32_t* seq_lens,
                           const uint8_t* mask, float* scores, void* ws, size_t ws_bytes,
                           void* stream);

/* The two halves of socket_score, for callers that schedule them separately:
 * socket_build_lut writes the Alg. 2 tables of every (b, selection row) as the
 * score kernel's shared-memory image (opaque layout) into `lut`, which must
 * hold socket_workspace_bytes(cfg, SOCKET_OP_SCORE, 0) bytes; socket_score_lut
 * computes Eq. 4 + Alg. 4 scores from it (same semantics as socket_score). */
socket_status socket_build_lut(const socket_cfg* cfg, const void* q, const void* W, void* lut,
                               size_t lut_bytes, void* stream);
socket_status socket_score_lut(const socket_cfg* cfg, const void* lut, const uint8_t* codes,
                               const float* vnorm, const int32_t* seq_lens, const uint8_t* mask,
                               float* scores, void* stream);

/* One whole SOCKET decode step, as one call with internal fusion:
 *   if append_last != 0: Alg. 1 on the newest key j = seq_lens[b] - 1 of every
 *     (b, kv head) (codes + vnorm; the new key is a candidate, reading R-18),
 *     in the same launch as the Alg. 2 table build.  If k_new / v_new are
 *     non-NULL ([B][H_kv][d] bf16, the new token's K and V rows), the step also
 *     stores them into K / V at row j (the caller need not write the cache);
 *     otherwise the caller has written row j already;
 *   then scores (Eq. 4 / Alg. 4, written to `scores`), TopK with sink/window
 *   (idx, cnt as socket_topk) and sparse attention (out, lse as
 *   socket_sparse_decode).  Up to 32 selection rows (KV_SHARED, P <= 8, and
 *   every selection row spread over >= 2 SMs) run as ONE cooperative launch
 *   over all SMs (the row-spread kernel; SOCKET_FLAG_ONE_LAUNCH: whenever the
 *   shape allows); otherwise 4 launches chained with programmatic dependent
 *   launch.  Requires L <= 64.
 *   q, k_new and v_new may be device pointers or pinned, UVA-mapped host
 *   pointers (cudaHostAlloc / cudaHostRegister); out may be either too.  On the
 *   chained path host-resident inputs are first pulled into the workspace by
 *   one copy kernel (a 5th launch); the one-launch kernel reads them in place.
 *   ws: socket_workspace_bytes(cfg, SOCKET_OP_DECODE_STEP, k) bytes, ZERO-FILLED
 *   before its first use with a given cfg (e.g. one cudaMemsetAsync after
 *   allocation): it holds the one-launch kernel's row barrier counters, which
 *   every step leaves at zero again.  (A workspace whose counters are not zero
 *   makes the kernel trap after 2 s instead of hanging.) */
socket_status socket_decode_step(const socket_cfg* cfg, const void* q, void* K, void* V,
                                 const void* W, uint8_t* codes, float* vnorm,
                                 const int32_t* seq_lens, const uint8_t* mask,
                                 int32_t append_last, const void* k_new, const void* v_new,
                                 int32_t k, int32_t sink, int32_t window,
                                 float* scores, int32_t* idx, int32_t* cnt, void* out, float* lse,
                                 void* ws, size_t ws_bytes, void* stream);

/* Number of kernel launches socket_decode_step issues for cfg with device
 * inputs: 1 (the one-launch row-spread kernel, small batches) or 4 (PDL-chained
 * kernels; 5 when q / k_new / v_new are host-resident); 0 if cfg is invalid. */
int32_t socket_decode_step_launches(const socket_cfg* cfg);

/* Alg. 3 l.244 TopK with forced sink / local window: per (b, row),
 * with n = seq_lens[b], position p(j) = index_base + j and
 * valid = (scores != -inf) & (p(j) < n) & (j < N_max):
 *   k_eff = min(k, #valid); forced F = valid & (p(j) < sink | n - window <= p(j));
 *   S = F plus the (k_eff - |F|) best remaining keys under the total order
 *   (score descending, index ascending) -- ties to the smaller index (R-15).
 * Writes idx[b][row][0..cnt) ascending, -1 after, cnt[b][row] = k_eff, and if
 * sel_scores != NULL, sel_scores[b][row][i] = scores[idx[i]] (-inf past cnt).
 * Positions (sink, window) are global (index_base + j).  Requires k <= N_max,
 * sink + window <= k.  ws: socket_workspace_bytes(cfg, SOCKET_OP_TOPK, k)
 * bytes -- 0 unless rows exceed 655360 keys (one cluster's shared memory), in
 * which case the key slices live in ws (4 B per key). */
socket_status socket_topk(const socket_cfg* cfg, const float* scores, const int32_t* seq_lens,
                          int32_t k, int32_t sink, int32_t window, int32_t* idx, int32_t* cnt,
                          float* sel_scores, void* ws, size_t ws_bytes, void* stream);

/* Eq. 2 with exact logits (reading R-1): for every
 * (b, query head h) with selection row r(h) (= h // G for KV_SHARED, h for PER_QHEAD)
 *   z_j = sm_scale * q_h . k_j,  j in S = idx[b][r][0..cnt)
 *   y = sum_j softmax(z)_j v_j,  lse = log sum_j exp(z_j)
 * idx rows have stride k.  Writes out (bf16, round-to-nearest) and lse if
 * non-NULL, and/or the unnormalised partial state (m, l, o) if partial != NULL
 * (used by sequence sharding; combine with socket_lse_combine). */
socket_status socket_sparse_decode(const socket_cfg* cfg, const void* q, const void* K,
                                   const void* V, const int32_t* idx, const int32_t* cnt,
                                   int32_t k, void* out, float* lse, float* partial, void* ws,
                                   size_t ws_bytes, void* stream);

/* Merge G partial states (m, l, o) over disjoint key sets (flash-decode split
 * merge): M = max_s m_s, w_s = e^{m_s - M}, y = sum w_s o_s / sum w_s l_s,
 * lse = M + log sum w_s l_s.  partials [G][B][H_q][d+2]; all-empty gives y = 0,
 * lse = -inf. */
socket_status socket_lse_combine(const socket_cfg* cfg, const float* partials, int32_t G,
                                 void* out, float* lse, void* stream);

/* Value-aware sampling decode, Eq. 6: for every query row (b, h)
 * (requires PER_QHEAD, so that `scores` holds that head's own s_j), with the
 * masked value scores s_j = ||v_j|| w_hat_j of socket_score (-inf = invalid):
 *   p_j = s_j / sum_i s_i                    (= a~_j ||v_j|| / sum_i a~_i ||v_i||)
 *   J_m = min{ j < seq_lens[b] : sum_{i<=j} s_i > u_m sum_i s_i }   (inverse CDF)
 *   out = (1/M) sum_m (a~_J / p_J) v_J = (sum s / sum w_hat) / M * sum_m v_J / ||v_J||
 * where a~_j = w_hat_j / sum_i w_hat_i and w_hat_j = s_j / ||v_j|| (0 if ||v_j|| = 0,
 * DESIGN.md R-24).  uniforms [B][H_q][M] fp32 in [0, 1) are the caller's draws;
 * samples [B][H_q][M] (nullable) receives J_m in the order of the uniforms
 * (-1 for a row without mass, whose output is 0).  out [B][H_q][d] bf16.
 * 1 <= M <= 8192.  No workspace. */
socket_status socket_sample_decode(const socket_cfg* cfg, const float* scores, const float* vnorm,
                                   const void* V, const int32_t* seq_lens, const float* uniforms,
                                   int32_t M, int32_t* samples, void* out, void* stream);

/* Eq. 1 (with sm_scale): dense flash-decode over every key
 * j < seq_lens[b] of the kv head of each query head; the k = n baseline. */
socket_status socket_dense_decode(const socket_cfg* cfg, const void* q, const void* K,
                                  const void* V, const int32_t* seq_lens, void* out, float* lse,
                                  void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ *
 * Sequence sharding: exact global top-k over G shards (DESIGN.md "Multi-GPU",
 * SURVEY 8(e) v2).  Shard s (rank s of G) holds the keys at global positions
 * [index_base_s, index_base_s + N_max) with index_base_s = s * N_max (shards
 * in rank order), scores from socket_score with the same cfg.index_base, and
 * seq_lens = the sequences' TOTAL lengths.  The selection equals socket_topk
 * over the concatenated rows (Alg. 3 l.244, ties to the smaller GLOBAL index,
 * reading R-15; sink / window on global positions).  Protocol, with an
 * all-gather (rank order) of each call's output across the shards:
 *   1. socket_topk_digest  -> digest [B][H_sel][Q][2]             all-gather
 *   2. socket_topk_bracket (all digests)      -> state [B][H_sel][SOCKET_TOPK_STATE_WORDS]
 *   3. socket_topk_window  (state)            -> msg   [B][H_sel][SOCKET_TOPK_MSG_WORDS]
 *                                                                 all-gather
 *   4. socket_topk_resolve (all msgs, rank)   -> state (resolved or a narrower bracket)
 *      repeat 3-4 while some row is unresolved (state word 3 == 0); at most 3
 *      rounds are ever needed, so a fixed 3 rounds is always exact (extra
 *      rounds on resolved rows are no-ops)
 *   5. socket_topk_emit    (state)            -> idx (local indices, ascending), cnt
 * The state and all messages are identical on every rank except the own-shard
 * quota words, so every rank resolves the same threshold.  Bytes per shard and
 * row: digest Q*8, message SOCKET_TOPK_MSG_WORDS*4.  ws: as socket_topk.
 * ------------------------------------------------------------------------ */
#define SOCKET_MAX_SHARDS 64
#define SOCKET_TOPK_STATE_WORDS 8
#define SOCKET_TOPK_MSG_WORDS (8 + 2048)

/* Digest of this shard's row (k = the GLOBAL budget, shards = G): Q pairs
 * (edge key, #keys with key >= edge), every count exact, on the monotone u32
 * key image of the scores (invalid 0, forced sink / window 0xFFFFFFFF):
 *   (1, #valid), (0xFFFFFFFF, #forced), (max regular key + 1, #forced), then
 *   the lower edges of the 2048-bin histogram bins that hold local ranks
 *   spread over (0, 2 ceil(k / shards)] and (.., min(k, #valid)].
 * Unused pairs are (0, 0).  4 <= Q <= 1024. */
socket_status socket_topk_digest(const socket_cfg* cfg, const float* scores, const int32_t* seq_lens,
                                 int32_t k, int32_t sink, int32_t window, int32_t shards, int32_t Q,
                                 uint32_t* digest, void* ws, size_t ws_bytes, void* stream);
/* Bracket [T_lo, T_hi) holding the global threshold key T of every row, from
 * the G all-gathered digests [G][B][H_sel][Q][2]; writes the initial state. */
socket_status socket_topk_bracket(const socket_cfg* cfg, const uint32_t* all_digests, int32_t G,
                                  int32_t Q, int32_t k, uint32_t* state, void* stream);
/* Window message of this shard for each unresolved row: header (lo, hi,
 * #keys >= hi, #keys in [lo, hi), mode, shift) and either the bracket's keys
 * (mode 0, when they fit 2048) or their 2048-bin histogram (mode 1). */
socket_status socket_topk_window(const socket_cfg* cfg, const float* scores, const int32_t* seq_lens,
                                 int32_t sink, int32_t window, const uint32_t* state, uint32_t* msg,
                                 void* ws, size_t ws_bytes, void* stream);
/* Resolve from the G all-gathered messages [G][B][H_sel][SOCKET_TOPK_MSG_WORDS]:
 * T exact (state word 3 = 1, word 4 = T, word 5 = this rank's quota of keys
 * == T, word 7 = this rank's #keys > T) or a narrower bracket. */
socket_status socket_topk_resolve(const socket_cfg* cfg, const uint32_t* all_msgs, int32_t G,
                                  int32_t rank, uint32_t* state, void* stream);
/* This shard's share of the selection: keys > T plus its quota of keys == T,
 * local indices ascending in idx[b][row][0..cnt) (-1 after; row stride k),
 * sel_scores optional.  A row whose state is unresolved gets cnt = -1. */
socket_status socket_topk_emit(const socket_cfg* cfg, const float* scores, const int32_t* seq_lens,
                               int32_t k, int32_t sink, int32_t window, const uint32_t* state,
                               int32_t* idx, int32_t* cnt, float* sel_scores, void* ws,
                               size_t ws_bytes, void* stream);

/* Message of the calling thread's last non-OK status ("" if none). */
const char* socket_last_error(void);
/* SOCKET_ABI_VERSION of the loaded library. */
int32_t socket_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SOCKET_B200_H */
