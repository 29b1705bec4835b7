// Causal flash-attention FORWARD, two query tiles per CTA (tcgen05 + TMEM + TMA).
//
// One CTA per (pair of 128-query blocks, batch*head): tiles t = 0, 1 cover queries
// [256p, 256p+128) and [256p+128, 256p+256) and share every K / V tile the TMA brings in.
// CTAs are issued heaviest pair first (causal work grows with p).
//   warp 0      TMA: Q_0, Q_1 once, K_j through a 2-stage ring
//   warp 3      TMA: V_j through its own 2-stage ring
//   warp 1      MMA issuer (one lane), per key block j:
//                 O_0 += P_0 V_j ; S_0 = Q_0 K_{j+1}^T ; O_1 += P_1 V_j ; S_1 = Q_1 K_{j+1}^T
//               P_t is read straight from TMEM (it overwrites S_t as packed bf16), so while
//               softmax warpgroup t works on S_t the tensor core runs tile 1-t's pair of MMAs
//               (ping-pong).  Because S_t(j+1) is issued after O_t += P_t(j) V_j on the same
//               in-order pipe, S_t(j+1) landing implies O_t is stable: the softmax warps may
//               rescale O_t without another barrier.
//   warps 4-7   softmax of tile 0, warps 8-11 softmax of tile 1: thread = query row = TMEM
//               lane.  tcgen05.ld the S row, causal mask on the diagonal block, running max in
//               the log2 domain, P = exp2(s*scale - m) -> bf16 pairs -> tcgen05.st over S.
//               O is rescaled in TMEM only when the row max grows by > 2^8 (l and O always
//               share one reference max, so the result is exact).
// TMEM (512 columns): S_0 [0,128) S_1 [128,256) O_0 [256,256+D) O_1 [256+D,256+2D).
// smem (D=128): Q 2 x 32 KB, K 2 x 32 KB, V 2 x 32 KB.
// Output O (bf16 [B*T, H*D]) and lse (natural log, [B, H, T]) exactly like attn_fwd_tc.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "ptx.cuh"
#include "zpp_internal.h"

namespace zpp {

typedef __nv_bfloat16 bf16;


template <int D>
struct Fwd2Cfg {
  static constexpr int ATOM = 128 * 128;       // [128 rows][64 bf16], 128B swizzle = 16 KB
  static constexpr int TILE = (D / 64) * ATOM;  // [128][D]
  static constexpr int Q_OFF = 0;               // 2 tiles
  static constexpr int K_OFF = Q_OFF + 2 * TILE;
  static constexpr int V_OFF = K_OFF + 2 * TILE;
  static constexpr int BAR_OFF = V_OFF + 2 * TILE;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static_assert(SMEM <= 232448, "smem budget");
};

template <int D>
__global__ void __launch_bounds__(384, 1)
    attn_fwd2_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, bf16* __restrict__ out, float* __restrict__ lse,
                        int T, int H, int BH, float scale_log2) {
  using C = Fwd2Cfg<D>;
  constexpr int NA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bars = base + C::BAR_OFF;
  // barrier map (8 B each)
  const uint32_t q_full = bars;
  const uint32_t k_full0 = bars + 8, k_empty0 = bars + 24, v_full0 = bars + 40, v_empty0 = bars + 56;
  const uint32_t s_full0 = bars + 72, p_full0 = bars + 88, o_final0 = bars + 104;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + C::BAR_OFF + 192);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npairs = T / 256;
  const int pair = npairs - 1 - static_cast<int>(blockIdx.x) / BH;  // heaviest first
  const int bh = static_cast<int>(blockIdx.x) % BH;
  const int b = bh / H, h = bh % H;
  const int nkb = 2 * pair + 2;  // key blocks 0 .. 2p+1 (tile 0 stops at 2p)
  const int row_base = b * T;

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_qkv);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(k_full0 + 8 * s, 1);
      mbar_init(k_empty0 + 8 * s, 1);
      mbar_init(v_full0 + 8 * s, 1);
      mbar_init(v_empty0 + 8 * s, 1);
      mbar_init(s_full0 + 8 * s, 1);
      mbar_init(p_full0 + 8 * s, 128);
      mbar_init(o_final0 + 8 * s, 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * C::TILE);
      for (int t = 0; t < 2; ++t)
        for (int a = 0; a < NA; ++a)
          tma_load_2d(base + C::Q_OFF + t * C::TILE + a * C::ATOM, &tm_qkv, q_full, h * D + 64 * a,
                      row_base + pair * 256 + t * 128);
      for (int j = 0; j < nkb; ++j) {
        const int st = j & 1;
        mbar_wait(k_empty0 + 8 * st, ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(k_full0 + 8 * st, C::TILE);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(base + C::K_OFF + st * C::TILE + a * C::ATOM, &tm_qkv, k_full0 + 8 * st, H * D + h * D + 64 * a,
                      row_base + j * 128);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (lane == 0) {
      for (int j = 0; j < nkb; ++j) {
        const int st = j & 1;
        mbar_wait(v_empty0 + 8 * st, ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(v_full0 + 8 * st, C::TILE);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(base + C::V_OFF + st * C::TILE + a * C::ATOM, &tm_qkv, v_full0 + 8 * st,
                      2 * H * D + h * D + 64 * a, row_base + j * 128);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, D, false, true);
      auto wait_k = [&](int j) {
        mbar_wait(k_full0 + 8 * (j & 1), (j >> 1) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int t, int j) {  // S_t = Q_t K_j^T
        const uint32_t kb = base + C::K_OFF + (j & 1) * C::TILE;
        const uint32_t qb = base + C::Q_OFF + t * C::TILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::ATOM + (kk & 3) * 32;
          mma_bf16(tmem + t * 128, make_sdesc(qb + off, 16, 1024), make_sdesc(kb + off, 16, 1024), idesc_s,
                   kk > 0 ? 1u : 0u);
        }
        mma_commit(s_full0 + 8 * t);
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P_t V_j  (P_t: TMEM columns [128t, 128t+64))
        const uint32_t vb = base + C::V_OFF + (j & 1) * C::TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_bf16_ts(tmem + 256 + t * D, tmem + t * 128 + kk * 8, make_sdesc(vb + kk * 2048, C::ATOM, 1024),
                      idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
      };
      mbar_wait(q_full, 0);
      wait_k(0);
      issue_s(0, 0);
      issue_s(1, 0);
      mma_commit(k_empty0);
      const int last0 = 2 * pair;  // tile 0's diagonal block
      for (int j = 0; j < nkb; ++j) {
        bool k_waited = false;
        mbar_wait(v_full0 + 8 * (j & 1), (j >> 1) & 1);
        if (j <= last0) {
          mbar_wait(p_full0, j & 1);
          tc_fence_after();
          issue_pv(0, j);
          if (j == last0) {
            mma_commit(o_final0);
          } else {
            wait_k(j + 1);
            k_waited = true;
            issue_s(0, j + 1);
          }
        }
        mbar_wait(p_full0 + 8, j & 1);
        tc_fence_after();
        issue_pv(1, j);
        mma_commit(v_empty0 + 8 * (j & 1));
        if (j == nkb - 1) {
          mma_commit(o_final0 + 8);
        } else {
          if (!k_waited) wait_k(j + 1);
          issue_s(1, j + 1);
          mma_commit(k_empty0 + 8 * ((j + 1) & 1));
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int t = (warp - 4) >> 2;
    const int q = warp & 3;
    const int r = q * 32 + lane;  // query row within the tile == TMEM lane
    const uint32_t lo = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t tS = tmem + lo + t * 128, tO = tmem + lo + 256 + t * D;
    const int diag = 2 * pair + t;
    const uint32_t s_full = s_full0 + 8 * t, p_full = p_full0 + 8 * t;
    float m_run = -INFINITY, l = 0.f;
    for (int j = 0; j <= diag; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      float x[128];
      {
        uint32_t v0[32], v1[32], v2[32], v3[32];
        tmem_ld32(tS, v0);
        tmem_ld32(tS + 32, v1);
        tmem_ld32(tS + 64, v2);
        tmem_ld32(tS + 96, v3);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          x[c] = __uint_as_float(v0[c]);
          x[32 + c] = __uint_as_float(v1[c]);
          x[64 + c] = __uint_as_float(v2[c]);
          x[96 + c] = __uint_as_float(v3[c]);
        }
      }
      if (j == diag) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c > r) x[c] = -INFINITY;
      }
      float pm[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pm[k] = x[k];
#pragma unroll
      for (int c = 8; c < 128; ++c) pm[c & 7] = fmaxf(pm[c & 7], x[c]);
      const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                             fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7]))) * scale_log2;
      const float m_new = fmaxf(m_run, mx);
      // tcgen05.ld/st are warp-collective: the rescale decision is warp-uniform
      const bool rescale = __any_sync(0xffffffffu, m_new > m_run + 8.f);
      const float m_use = rescale ? m_new : m_run;
      if (rescale && j > 0) {  // O_t is stable here (see header)
        const float f = fast_exp2(m_run - m_use);
        l *= f;
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(tO + c * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(__uint_as_float(v[k]) * f);
          tmem_st32(tO + c * 32, v);
        }
      }
      m_run = m_use;
      float ps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        uint32_t pk[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float a0 = fmaf(x[c4 * 32 + 2 * k], scale_log2, -m_use);
          const float a1 = fmaf(x[c4 * 32 + 2 * k + 1], scale_log2, -m_use);
          const float e0 = fast_exp2(a0);
          const float e1 = fast_exp2(a1);
          ps[(2 * k) & 7] += e0;
          ps[(2 * k + 1) & 7] += e1;
          pk[k] = pack_bf16(e0, e1);
        }
        tmem_st16(tS + c4 * 16, pk);  // P keys [32 c4, 32 c4 + 32) -> columns [16 c4, 16 c4 + 16)
      }
      l += ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(o_final0 + 8 * t, 0);
    tc_fence_after();
    const float inv = 1.f / l;
    const int qrow = pair * 256 + t * 128 + r;
    bf16* orow = out + ((long long)row_base + qrow) * H * D + (long long)h * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tO + c * 32, v);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; k += 8)
        *reinterpret_cast<uint4*>(orow + c * 32 + k) =
            make_uint4(pack_bf16(__uint_as_float(v[k]) * inv, __uint_as_float(v[k + 1]) * inv),
                       pack_bf16(__uint_as_float(v[k + 2]) * inv, __uint_as_float(v[k + 3]) * inv),
                       pack_bf16(__uint_as_float(v[k + 4]) * inv, __uint_as_float(v[k + 5]) * inv),
                       pack_bf16(__uint_as_float(v[k + 6]) * inv, __uint_as_float(v[k + 7]) * inv));
    }
    lse[(long long)bh * T + qrow] = (m_run + log2f(l)) * 0.6931471805599453f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int D>
static cudaError_t fwd2_attr() {
  return cudaFuncSetAttribute(attn_fwd2_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Cfg<D>::SMEM);
}

template <int D>
int attn_fwd2_tc_launch(const void* qkv, void* out, float* lse, int B, int T, int H, cudaStream_t s) {
  using C = Fwd2Cfg<D>;
  if (T % 256) return set_error(ZPP_ERR_ARG, "attn_fwd2: seq must be a multiple of 256");
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
    cudaError_t e = fwd2_attr<D>();
    if (e != cudaSuccess) return set_cuda_error(e, "attn_fwd2_tc attr");
    set = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  const int BH = B * H;
  attn_fwd2_tc_kernel<D><<<dim3((T / 256) * BH), 384, C::SMEM, s>>>(m, (bf16*)out, lse, T, H, BH, scale_log2);
  return check_launch("attn_fwd2_tc");
}

template int attn_fwd2_tc_launch<64>(const void*, void*, float*, int, int, int, cudaStream_t);
template int attn_fwd2_tc_launch<128>(const void*, void*, float*, int, int, int, cudaStream_t);

int attention_fwd2_preload() {
  cudaError_t e = fwd2_attr<64>();
  if (e == cudaSuccess) e = fwd2_attr<128>();
  return e == cudaSuccess ? ZPP_OK : set_cuda_error(e, "attention_fwd2 preload");
}

}  // namespace zpp
