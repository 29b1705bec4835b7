// Causal multi-head attention over packed qkv [b, s, 3, heads, d]: the C ABI entry points and
// the kernel preload.  Every path is tcgen05 / TMEM / TMA (sm_100a):
//   forward   attention_fwd2_tc.cu  two 128-query tiles per CTA (seq % 256 == 0)
//             attention_tc.cu       one 128-query tile per CTA   (seq % 128 == 0, e.g. s = 128)
//   backward  attention_bwd_tc.cu   dQ kernel (+ delta) then dK/dV kernel, deterministic
#include <cuda_runtime.h>
#include <stdint.h>

#include "zpp_internal.h"

namespace zpp {

template <int D>
int attn_fwd_tc_launch(const void* qkv, void* out, float* lse, int B, int T, int H, cudaStream_t s);
template <int D>
int attn_fwd2_tc_launch(const void* qkv, void* out, float* lse, int B, int T, int H, cudaStream_t s);
template <int D>
int attn_bwd_tc_launch(const void* qkv, const void* out, const float* lse, const void* dout, void* dqkv, float* ws,
                       int B, int T, int H, cudaStream_t s);

int attention_tc_preload();
int attention_fwd2_preload();
int attention_bwd_tc_preload();
int gemm_preload();
int kernels_preload();

}  // namespace zpp

using namespace zpp;

// Force-load every kernel of the library (CUDA lazy loading would otherwise load a
// kernel at its first launch, which needs a context-wide synchronisation: that
// deadlocks against NCCL kernels spinning on a peer rank).
extern "C" int zpp_preload_kernels(void) {
  int rc = gemm_preload();
  if (!rc) rc = attention_tc_preload();
  if (!rc) rc = attention_bwd_tc_preload();
  if (!rc) rc = attention_fwd2_preload();
  if (!rc) rc = kernels_preload();
  return rc;
}

extern "C" int zpp_attn_fwd(const void* qkv, void* out, float* lse, int batch, int seq, int heads, int head_dim,
                            uintptr_t stream) {
  if (seq % 128) return set_error(ZPP_ERR_ARG, "attn: seq must be a multiple of 128");
  if (head_dim != 64 && head_dim != 128) return set_error(ZPP_ERR_ARG, "attn: head_dim must be 64 or 128");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (seq % 256 == 0)
    return head_dim == 128 ? attn_fwd2_tc_launch<128>(qkv, out, lse, batch, seq, heads, s)
                           : attn_fwd2_tc_launch<64>(qkv, out, lse, batch, seq, heads, s);
  return head_dim == 128 ? attn_fwd_tc_launch<128>(qkv, out, lse, batch, seq, heads, s)
                         : attn_fwd_tc_launch<64>(qkv, out, lse, batch, seq, heads, s);
}

extern "C" long long zpp_attn_bwd_workspace_floats(int batch, int seq, int heads, int head_dim) {
  (void)head_dim;
  return 2LL * batch * heads * seq;  // delta | lse * log2(e)
}

extern "C" int zpp_attn_bwd(const void* qkv, const void* out, const float* lse, const void* dout, void* dqkv,
                            float* workspace, int batch, int seq, int heads, int head_dim, uintptr_t stream) {
  if (seq % 128) return set_error(ZPP_ERR_ARG, "attn_bwd: seq must be a multiple of 128");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (head_dim == 128) return attn_bwd_tc_launch<128>(qkv, out, lse, dout, dqkv, workspace, batch, seq, heads, s);
  if (head_dim == 64) return attn_bwd_tc_launch<64>(qkv, out, lse, dout, dqkv, workspace, batch, seq, heads, s);
  return set_error(ZPP_ERR_ARG, "attn_bwd: head_dim must be 64 or 128");
}
