// tcgen05 projection GEMM for Alg. 1 (placeholder until the tensor-core kernel lands).
#include "internal.cuh"

namespace sk {

socket_status launch_hash_keys_tc(const socket_cfg& c, const void* K, const void* W,
                                  uint8_t* codes, int n_begin, int n_count, cudaStream_t st,
                                  bool* used) {
  (void)c; (void)K; (void)W; (void)codes; (void)n_begin; (void)n_count; (void)st;
  *used = false;
  return SOCKET_OK;
}

}  // namespace sk
