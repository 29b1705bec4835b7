// Causal flash-attention FORWARD on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// One CTA per (128-query block, batch*head); q-blocks scheduled latest-first.
//   warp 0     TMA producer: Q once, then K 128-key tiles through a 2-stage ring
//   warp 3     TMA producer: V tiles through their own 2-stage ring.  K_i's slot frees as
//              soon as S_i is computed, so K_{i+2} streams in while PV_i / softmax run
//              (a joint K/V slot would put PV_i + the TMA latency on the S critical path)
//   warp 1     MMA issuer (one lane):  S_i = Q K_i^T   (M=128, N=128, K=d)  -> TMEM S[i%2]
//                                      O  += P_i V_i    (M=128, N=d,  K=128) -> TMEM O
//              S_{i+1} is issued before O += P_i V_i so the tensor core works while
//              the softmax warps process S_i.
//   warps 4-7  softmax: thread t owns query row t (= TMEM lane t).  tcgen05.ld S row,
//              running max in the log2 domain, P = exp2(s - m) -> bf16 P tile in
//              smem (128B-swizzled K-major, the A operand of the PV MMA).  O is
//              rescaled in TMEM (tcgen05.ld/st) only when the row max grows by more
//              than 2^8 (exact: l and O always share the same reference max).
// TMEM: S double buffer 2 x 128 columns + O d columns.  smem (d=128): Q 32 KB,
// K/V 2 x 64 KB, P 32 KB.  Output O (bf16) and lse (natural log) like attn_fwd.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "ptx.cuh"
#include "zpp_internal.h"

namespace zpp {

typedef __nv_bfloat16 bf16;

template <int D>
struct TcFwdCfg {
  static constexpr int ATOM = 128 * 128;       // one [128 rows][64 bf16] swizzled atom = 16 KB
  static constexpr int TILE = (D / 64) * ATOM;  // [128][D] tile
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + TILE;
  static constexpr int V_OFF = K_OFF + 2 * TILE;
  static constexpr int P_OFF = V_OFF + 2 * TILE;
  static constexpr int BAR_OFF = P_OFF + 2 * ATOM;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(256, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, bf16* __restrict__ out, float* __restrict__ lse,
                       int T, int H, float scale_log2) {
  using C = TcFwdCfg<D>;
  constexpr int NA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bars = base + C::BAR_OFF;
  const uint32_t q_full = bars, k_full0 = bars + 8, k_empty0 = bars + 24, s_full0 = bars + 40;
  const uint32_t p_full = bars + 56, o_done = bars + 64, v_full0 = bars + 72, v_empty0 = bars + 88;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + C::BAR_OFF + 128);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int qblk = gridDim.x - 1 - blockIdx.x;
  const int q0 = qblk * 128;
  const int nkb = qblk + 1;
  const int row_base = b * T;  // row index of token 0 of this sequence in [b*T, 3HD]

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_qkv);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(k_full0 + 8 * s, 1);
      mbar_init(k_empty0 + 8 * s, 1);
      mbar_init(v_full0 + 8 * s, 1);
      mbar_init(v_empty0 + 8 * s, 1);
      mbar_init(s_full0 + 8 * s, 1);
    }
    mbar_init(p_full, 128);
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, C::TILE);
      for (int a = 0; a < NA; ++a) tma_load_2d(base + C::Q_OFF + a * C::ATOM, &tm_qkv, q_full, h * D + 64 * a, row_base + q0);
      for (int i = 0; i < nkb; ++i) {
        const int st = i & 1;
        mbar_wait(k_empty0 + 8 * st, ((i >> 1) & 1) ^ 1);
        const uint32_t fb = k_full0 + 8 * st;
        mbar_arrive_expect_tx(fb, C::TILE);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(base + C::K_OFF + st * C::TILE + a * C::ATOM, &tm_qkv, fb, H * D + h * D + 64 * a, row_base + i * 128);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int st = i & 1;
        mbar_wait(v_empty0 + 8 * st, ((i >> 1) & 1) ^ 1);
        const uint32_t fb = v_full0 + 8 * st;
        mbar_arrive_expect_tx(fb, C::TILE);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(base + C::V_OFF + st * C::TILE + a * C::ATOM, &tm_qkv, fb, 2 * H * D + h * D + 64 * a,
                      row_base + i * 128);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, D, false, true);
      auto issue_s = [&](int i) {
        const int st = i & 1;
        mbar_wait(k_full0 + 8 * st, (i >> 1) & 1);
        tc_fence_after();
        const uint32_t kb = base + C::K_OFF + st * C::TILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::ATOM + (kk & 3) * 32;
          mma_bf16(tmem + st * 128, make_sdesc(base + C::Q_OFF + off, 16, 1024), make_sdesc(kb + off, 16, 1024), idesc_s,
                   kk > 0 ? 1u : 0u);
        }
        mma_commit(s_full0 + 8 * st);
        mma_commit(k_empty0 + 8 * st);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      for (int i = 0; i < nkb; ++i) {
        if (i + 1 < nkb) issue_s(i + 1);
        mbar_wait(p_full, i & 1);
        mbar_wait(v_full0 + 8 * (i & 1), (i >> 1) & 1);
        tc_fence_after();
        const uint32_t vb = base + C::V_OFF + (i & 1) * C::TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = make_sdesc(base + C::P_OFF + (kk >> 2) * C::ATOM + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = make_sdesc(vb + kk * 2048, C::ATOM, 1024);
          mma_bf16(tmem + 256, ad, bd, idesc_o, (i > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(o_done);
        mma_commit(v_empty0 + 8 * (i & 1));
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int r = q * 32 + lane;  // query row within the block == TMEM lane
    const uint32_t tl = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float m_run = -INFINITY, l = 0.f;
    for (int i = 0; i < nkb; ++i) {
      mbar_wait(s_full0 + 8 * (i & 1), (i >> 1) & 1);
      tc_fence_after();
      float x[128];  // raw scores (scale folded into the exp2 FFMA below)
      {
        uint32_t v0[32], v1[32], v2[32], v3[32];
        const uint32_t sb = tl + (i & 1) * 128;
        tmem_ld32(sb, v0);
        tmem_ld32(sb + 32, v1);
        tmem_ld32(sb + 64, v2);
        tmem_ld32(sb + 96, v3);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          x[j] = __uint_as_float(v0[j]);
          x[32 + j] = __uint_as_float(v1[j]);
          x[64 + j] = __uint_as_float(v2[j]);
          x[96 + j] = __uint_as_float(v3[j]);
        }
      }
      if (i == nkb - 1) {  // diagonal block: keys after the query are masked
#pragma unroll
        for (int j = 0; j < 128; ++j)
          if (j > r) x[j] = -INFINITY;
      }
      float pm[8];  // 8 independent max chains
#pragma unroll
      for (int k = 0; k < 8; ++k) pm[k] = x[k];
#pragma unroll
      for (int j = 8; j < 128; ++j) pm[j & 7] = fmaxf(pm[j & 7], x[j]);
      const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                             fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7]))) * scale_log2;
      const float m_new = fmaxf(m_run, mx);
      // tcgen05.ld/st below are warp-collective (.sync.aligned): the rescale decision
      // must be warp-uniform.  Any lane needing it makes every lane move to its own max.
      const bool rescale = __any_sync(0xffffffffu, m_new > m_run + 8.f);
      const float m_use = rescale ? m_new : m_run;
      float ps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 8 independent sum chains
#pragma unroll
      for (int j = 0; j < 128; ++j) {
        x[j] = fast_exp2(fmaf(x[j], scale_log2, -m_use));
        ps[j & 7] += x[j];
      }
      const float rs = ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
      if (i > 0) {
        mbar_wait(o_done, (i - 1) & 1);  // PV_{i-1} finished: P buffer free, O stable
        tc_fence_after();
        if (rescale) {
          const float f = fast_exp2(m_run - m_use);
          l *= f;
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t v[32];
            tmem_ld32(tl + 256 + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * f);
            tmem_st32(tl + 256 + c * 32, v);
          }
          tmem_wait_st();
        }
      }
      m_run = m_use;
      l += rs;
      // P row -> smem (two 64-key K-major atoms, 128B swizzle)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const uint32_t rowp = base + C::P_OFF + a * C::ATOM + r * 128;
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          const float* s = &x[a * 64 + c8 * 8];
          st_shared_v4(rowp + ((c8 ^ (r & 7)) << 4), pack_bf16(s[0], s[1]), pack_bf16(s[2], s[3]),
                       pack_bf16(s[4], s[5]), pack_bf16(s[6], s[7]));
        }
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(o_done, (nkb - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    bf16* orow = out + ((long long)row_base + q0 + r) * H * D + (long long)h * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tl + 256 + c * 32, v);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; j += 8)
        *reinterpret_cast<uint4*>(orow + c * 32 + j) =
            make_uint4(pack_bf16(__uint_as_float(v[j]) * inv, __uint_as_float(v[j + 1]) * inv),
                       pack_bf16(__uint_as_float(v[j + 2]) * inv, __uint_as_float(v[j + 3]) * inv),
                       pack_bf16(__uint_as_float(v[j + 4]) * inv, __uint_as_float(v[j + 5]) * inv),
                       pack_bf16(__uint_as_float(v[j + 6]) * inv, __uint_as_float(v[j + 7]) * inv));
    }
    lse[(long long)bh * T + q0 + r] = (m_run + log2f(l)) * 0.6931471805599453f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int D>
int attn_fwd_tc_launch(const void* qkv, void* out, float* lse, int B, int T, int H, cudaStream_t s) {
  using C = TcFwdCfg<D>;
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)3 * H * D, (cuuint64_t)B * T};
  cuuint64_t strides[1] = {(cuuint64_t)3 * H * D * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  int rc = encode_tensor_map(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims, strides, box, estr,
                             CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_fwd_tc attr");
    set = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  attn_fwd_tc_kernel<D><<<dim3(T / 128, B * H), 256, C::SMEM, s>>>(m, (bf16*)out, lse, T, H, scale_log2);
  return check_launch("attn_fwd_tc");
}

template int attn_fwd_tc_launch<64>(const void*, void*, float*, int, int, int, cudaStream_t);
template int attn_fwd_tc_launch<128>(const void*, void*, float*, int, int, int, cudaStream_t);

int attention_tc_preload() {
  cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       TcFwdCfg<64>::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(attn_fwd_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             TcFwdCfg<128>::SMEM);
  return e == cudaSuccess ? ZPP_OK : set_cuda_error(e, "attention_tc preload");
}

}  // namespace zpp
