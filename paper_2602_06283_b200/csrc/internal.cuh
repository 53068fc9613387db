// Internal helpers of libsocket_b200 (sm_100a).  Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/socket_b200.h"

namespace sk {

// ----------------------------------------------------------------------------
// error reporting (thread-local last error; the C ABI never throws)
// ----------------------------------------------------------------------------
void set_error(const std::string& msg);
socket_status fail(socket_status st, const std::string& msg);
socket_status check_launch(const char* what);

constexpr int kD = 128;           // head dim supported by every kernel
// SM count of the current device (queried once per device; MIG / green
// contexts report their own count)
int num_sms();
constexpr int kLutPanelCols = 64; // LUT row = 64 fp32 columns = 256 B
constexpr int kLutRows = 256;     // 2^P rows for P <= 8

inline int code_slots(int L) {
  if (L < 1) return 0;
  if (L <= 8) return 8;
  if (L <= 16) return 16;
  if (L <= 32) return 32;
  return (L + 31) / 32 * 32;
}
inline int lut_panels(int Lp) { return Lp <= 64 ? 1 : (Lp + 63) / 64; }
inline int num_sel_rows(const socket_cfg& c) {
  return c.group_mode == SOCKET_GROUP_PER_QHEAD ? c.H_q : c.H_kv;
}
inline size_t lut_bytes_per_row(int L) {
  return (size_t)lut_panels(code_slots(L)) * kLutRows * kLutPanelCols * sizeof(float);
}
// P > 8 ("wide" codes, NEXT-2): one uint16 per (key, table); the score kernel's
// LUT holds per query head the two factor half-tables A(lo), B(hi) of the
// exact product form p(r) = A(r mod 2^Pl) B(r >> Pl), Pl = P / 2.
// Code slots of the stored layout for (L, P): byte codes (P <= 8) use
// code_slots(L); packed wide codes (P > 8) need whole 32-slot groups.
inline int code_slots_p(int L, int P) {
  const int lp = code_slots(L);
  return (P > 8 && lp < 32) ? 32 : lp;
}
// Stored code bytes per key: Lp bytes (P <= 8) or Lp * P bits, tightly packed (P > 8)
inline size_t code_bytes_per_key(int L, int P) {
  const int lp = code_slots_p(L, P);
  return P > 8 ? (size_t)lp * P / 8 : (size_t)lp;
}
inline int wide_lo_bits(int P) { return P / 2; }
inline int wide_entries(int P) { return 1 << (P - P / 2); }   // rows per half-table image
inline int heads_per_row(const socket_cfg& c) {
  return c.group_mode == SOCKET_GROUP_PER_QHEAD ? 1 : c.H_q / c.H_kv;
}
// LUT image bytes of one selection row for cfg (P <= 8: the [256][64] table
// panels; P > 8: [NH][2][2^(P - P/2)][64] half-table panels)
inline size_t lut_row_bytes(const socket_cfg& c) {
  if (c.P <= 8) return lut_bytes_per_row(c.L);
  return (size_t)heads_per_row(c) * 2 * wide_entries(c.P) * kLutPanelCols * sizeof(float);
}
constexpr size_t kWideLutMax = 160 * 1024;   // shared-memory budget of the wide score kernel

// ----------------------------------------------------------------------------
// launchers (defined in the kernel .cu files)
// ----------------------------------------------------------------------------
socket_status launch_hash_keys(const socket_cfg& c, const void* K, const void* V, int n_begin,
                               int n_count, const void* W, uint8_t* codes, float* vnorm,
                               cudaStream_t st);
socket_status launch_pack_codes(const socket_cfg& c, const uint8_t* plain, uint8_t* codes,
                                bool unpack, cudaStream_t st);
socket_status launch_query_tables(const socket_cfg& c, const void* q, const void* W,
                                  float* tables_plain, float* lut, cudaStream_t st);
socket_status launch_score(const socket_cfg& c, const float* lut, const uint8_t* codes,
                           const float* vnorm, const int32_t* seq_lens, const uint8_t* mask,
                           float* scores, cudaStream_t st);
socket_status launch_topk(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                          int k, int sink, int window, int32_t* idx, int32_t* cnt,
                          float* sel_scores, void* ws, size_t ws_bytes, cudaStream_t st);
size_t topk_workspace_bytes(const socket_cfg& c);
socket_status launch_topk_digest(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                                 int k, int sink, int window, int shards, int Q, uint32_t* digest,
                                 void* ws, size_t ws_bytes, cudaStream_t st);
socket_status launch_topk_bracket(const socket_cfg& c, const uint32_t* digests, int G, int Q, int k,
                                  uint32_t* state, cudaStream_t st);
socket_status launch_topk_window(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                                 int sink, int window, const uint32_t* state, uint32_t* msg,
                                 void* ws, size_t ws_bytes, cudaStream_t st);
socket_status launch_topk_resolve(const socket_cfg& c, const uint32_t* msgs, int G, int rank,
                                  uint32_t* state, cudaStream_t st);
socket_status launch_topk_emit(const socket_cfg& c, const float* scores, const int32_t* seq_lens,
                               int k, int sink, int window, const uint32_t* state, int32_t* idx,
                               int32_t* cnt, float* sel_scores, void* ws, size_t ws_bytes,
                               cudaStream_t st);
size_t decode_workspace_bytes(const socket_cfg& c, int k, bool dense);
socket_status launch_decode(const socket_cfg& c, const void* q, const void* K, const void* V,
                            const int32_t* idx, const int32_t* cnt, int k,
                            const int32_t* seq_lens, bool dense, void* out, float* lse,
                            float* partial, void* ws, size_t ws_bytes, cudaStream_t st);
size_t decode_step_workspace_bytes(const socket_cfg& c, int k);
socket_status launch_decode_step(const socket_cfg& c, const void* q, void* K, void* V,
                                 const void* W, uint8_t* codes, float* vnorm,
                                 const int32_t* seq_lens, const uint8_t* mask, int do_append,
                                 const void* k_new, const void* v_new, int k, int sink, int window,
                                 float* scores, int32_t* idx, int32_t* cnt, void* out, float* lse,
                                 void* ws, size_t ws_bytes, cudaStream_t st);
socket_status launch_sample_decode(const socket_cfg& c, const float* scores, const float* vnorm,
                                   const void* V, const int32_t* seq_lens, const float* uniforms,
                                   int M, int32_t* samples, void* out, cudaStream_t st);
socket_status launch_lse_combine(const socket_cfg& c, const float* partials, int G,
                                 void* out, float* lse, cudaStream_t st);

}  // namespace sk

// ----------------------------------------------------------------------------
// device helpers
// ----------------------------------------------------------------------------
#ifdef __CUDACC__
namespace sk {

__device__ __forceinline__ float bf16lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

// round-to-nearest-even fp32 -> bf16 bits (finite inputs)
__device__ __forceinline__ uint32_t f2bf_bits(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7F800000u) == 0x7F800000u) return (u >> 16) | ((u & 0xFFFFu) ? 0x40u : 0u);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return u >> 16;
}

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// L2 cache policies: streamed-once operands (evict_first) and results the next
// kernel of the step reads back (evict_last)
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ldg_nc_v4_hint(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint2 ldg_nc_v2_hint(const void* p, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint32_t ldg_nc_u32_hint(const void* p, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_f32_hint(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint2 ldg_nc_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}

// keys of a buffer at global positions index_base + j are valid iff
// index_base + j < seq_len (socket_cfg.index_base); local valid count:
__device__ __forceinline__ int local_len(int seq_len, long long index_base, int N_max) {
  const long long n = (long long)seq_len - index_base;
  return n < 0 ? 0 : (n > N_max ? N_max : (int)n);
}

// Packed wide codes (P > 8, NEXT-2): per (b, kv head) region, 32-key tiles;
// per tile and 32-slot group g (G = Lp / 32 groups), the group's 32 P-bit slot
// codes form one 32P-bit string (slot s at bits [sP, sP + P), LSB first), kept
// as P u32 words, word-interleaved across the tile's 32 keys.  u32 index of
// word w of group g of key j:
__device__ __forceinline__ size_t packed_word(int j, int g, int w, int G, int P) {
  return ((size_t)((j >> 5) * G + g) * P + w) * 32 + (j & 31);
}

// monotone map fp32 -> u32 (larger float <=> larger key)
__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

}  // namespace sk
#endif
