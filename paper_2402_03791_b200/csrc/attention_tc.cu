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
                       int T, int H, float scale_log2, unsigned long long* __restrict__ trace) {
  using C = TcFwdCfg<D>;
  // optional phase timeline of CTA (0, 0) (ZPP_ATTN_TRACE; trace == nullptr in production)
  const bool tr = trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0;
  auto mark = [&](int slot) {
    if (tr) trace[slot] = clock64();
  };
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
        mark(16 * i + 0);
        if (i + 1 < nkb) issue_s(i + 1);
        mark(16 * i + 1);
        mbar_wait(p_full, i & 1);
        mark(16 * i + 2);
        mbar_wait(v_full0 + 8 * (i & 1), (i >> 1) & 1);
        mark(16 * i + 3);
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
    const bool tl0 = threadIdx.x == 128;
    for (int i = 0; i < nkb; ++i) {
      if (tl0) mark(16 * i + 8);
      mbar_wait(s_full0 + 8 * (i & 1), (i >> 1) & 1);
      if (tl0) mark(16 * i + 9);
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
      if (tl0) mark(16 * i + 10);
      if (i > 0) {
        mbar_wait(o_done, (i - 1) & 1);  // PV_{i-1} finished: P buffer free, O stable
        if (tl0) mark(16 * i + 11);
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
      if (tl0) mark(16 * i + 12);
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
  static int want_trace = -1;
  if (want_trace < 0) want_trace = getenv("ZPP_ATTN_TRACE") ? 1 : 0;
  unsigned long long* trace = nullptr;
  if (want_trace) {
    cudaMalloc(&trace, 16 * 32 * sizeof(unsigned long long));
    cudaMemset(trace, 0, 16 * 32 * sizeof(unsigned long long));
  }
  attn_fwd_tc_kernel<D><<<dim3(T / 128, B * H), 256, C::SMEM, s>>>(m, (bf16*)out, lse, T, H, scale_log2, trace);
  if (trace) {
    unsigned long long hbuf[16 * 32];
    cudaMemcpy(hbuf, trace, sizeof(hbuf), cudaMemcpyDeviceToHost);
    const int nkb = T / 128;
    const unsigned long long t0 = hbuf[0];
    for (int i = 0; i < nkb; ++i) {
      const unsigned long long* x = hbuf + 16 * i;
      printf("fwd it %2d | mma: top %7lld s_next %7lld pfull %7lld vfull %7lld | sm: top %7lld sfull %7lld exp %7lld"
             " odone %7lld parrive %7lld\n", i, (long long)(x[0] - t0), (long long)(x[1] - t0), (long long)(x[2] - t0),
             (long long)(x[3] - t0), (long long)(x[8] - t0), (long long)(x[9] - t0), (long long)(x[10] - t0),
             (long long)(i ? x[11] - t0 : 0), (long long)(x[12] - t0));
    }
    cudaFree(trace);
  }
  return check_launch("attn_fwd_tc");
}

template int attn_fwd_tc_launch<64>(const void*, void*, float*, int, int, int, cudaStream_t);
template int attn_fwd_tc_launch<128>(const void*, void*, float*, int, int, int, cudaStream_t);

// ===========================================================================
// Causal flash-attention BACKWARD on tcgen05.
//
// One CTA per (128-key block j, batch*head); loop over query blocks i >= j.
//   warp 0     TMA: K_j, V_j once; Q_i / dO_i through a 2-stage ring
//   warp 1     MMA: S^T = K Q_i^T, dP^T = V dO_i^T                (TMEM cols 256 / 384)
//                   dV += P^T dO_i  (A = P^T from TMEM, bf16)      (TMEM cols 0..)
//                   dK += dS^T Q_i  (A = dS^T smem, K-major)       (TMEM cols 128..)
//                   dQ  = dS K_j    (A = dS^T smem read MN-major)  (TMEM cols 384.., over dP^T)
//   warps 4-7  thread t owns key row t: P^T = exp2(S^T*scale*log2e - lse*log2e) (causal mask
//              on the diagonal block), dS^T = P^T (dP^T - delta) * scale; P^T -> TMEM
//              (over S^T), dS^T -> smem.  Then dQ rows (thread = query row) are read from
//              TMEM into registers and the dP columns released at once (the next dP^T
//              does not wait for the reduction), then staged in the free dS^T smem and
//              TMA reduce-added into the fp32 dQ workspace.
// smem (d=128): K 32 KB, V 32 KB, Q/dO 2 x 64 KB, dS^T 32 KB (+ lse/delta 1 KB).
template <int D>
struct TcBwdCfg {
  static constexpr int ATOM = 128 * 128;
  static constexpr int TILE = (D / 64) * ATOM;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + TILE;
  static constexpr int Q_OFF = V_OFF + TILE;    // 2 stages
  static constexpr int DO_OFF = Q_OFF + 2 * TILE;  // 2 stages
  static constexpr int DS_OFF = DO_OFF + 2 * TILE;  // 2 atoms (128 keys x 128 queries bf16)
  static constexpr int L_OFF = DS_OFF + 2 * ATOM;   // lse*log2e [128], delta [128]
  static constexpr int BAR_OFF = L_OFF + 1024;
  static constexpr int SMEM = BAR_OFF + 128 + 1024;
  static_assert(SMEM <= 232448, "smem budget");
};

template <int D>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_dq, const float* __restrict__ lse,
                       const float* __restrict__ delta, bf16* __restrict__ dqkv, float* __restrict__ dq_acc,
                       int T, int H, float scale, unsigned long long* __restrict__ trace) {
  using C = TcBwdCfg<D>;
  // optional phase timeline of CTA (0, 0) for performance analysis (trace == nullptr in production)
  const bool tr = trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0;
  auto mark = [&](int slot) {
    if (tr) trace[slot] = clock64();
  };
  constexpr int NA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  float* sL = reinterpret_cast<float*>(gbase + C::L_OFF);
  float* sDl = sL + 128;
  const uint32_t bars = base + C::BAR_OFF;
  const uint32_t kv_full = bars, qd_full0 = bars + 8, qd_empty0 = bars + 24, sp_full = bars + 40;
  const uint32_t ds_full = bars + 48, mm_done = bars + 56, dq_free = bars + 64;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + C::BAR_OFF + 96);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int kblk = blockIdx.x;
  const int k0 = kblk * 128;
  const int nq = T / 128 - kblk;
  const int row_base = b * T;
  const float LOG2E_ = 1.4426950408889634f;

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_dq);
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(qd_full0 + 8 * s, 1);
      mbar_init(qd_empty0 + 8 * s, 1);
    }
    mbar_init(sp_full, 1);
    mbar_init(ds_full, 256);
    mbar_init(mm_done, 1);
    mbar_init(dq_free, 256);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t T_DV = tmem, T_DK = tmem + 128, T_S = tmem + 256, T_DP = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * C::TILE);
      for (int a = 0; a < NA; ++a) {
        tma_load_2d(base + C::K_OFF + a * C::ATOM, &tm_qkv, kv_full, H * D + h * D + 64 * a, row_base + k0);
        tma_load_2d(base + C::V_OFF + a * C::ATOM, &tm_qkv, kv_full, 2 * H * D + h * D + 64 * a, row_base + k0);
      }
      for (int it = 0; it < nq; ++it) {
        const int st = it & 1;
        const int q0 = (kblk + it) * 128;
        mbar_wait(qd_empty0 + 8 * st, ((it >> 1) & 1) ^ 1);
        const uint32_t fb = qd_full0 + 8 * st;
        mbar_arrive_expect_tx(fb, 2 * C::TILE);
        for (int a = 0; a < NA; ++a) {
          tma_load_2d(base + C::Q_OFF + st * C::TILE + a * C::ATOM, &tm_qkv, fb, h * D + 64 * a, row_base + q0);
          tma_load_2d(base + C::DO_OFF + st * C::TILE + a * C::ATOM, &tm_do, fb, h * D + 64 * a, row_base + q0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_kk = make_idesc_bf16(128, 128, false, false);  // S^T, dP^T (N = 128 queries)
      constexpr uint32_t id_kmn = make_idesc_bf16(128, D, false, true);    // dV, dK (B MN-major, N = d)
      constexpr uint32_t id_mnmn = make_idesc_bf16(128, D, true, true);    // dQ (A and B MN-major)
      mbar_wait(kv_full, 0);
      auto issue_st = [&](int it) {  // S^T = K Q^T into the S columns (in-order after dV read P^T)
        const int st = it & 1;
        mbar_wait(qd_full0 + 8 * st, (it >> 1) & 1);
        tc_fence_after();
        const uint32_t qs = base + C::Q_OFF + st * C::TILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::ATOM + (kk & 3) * 32;
          mma_bf16(T_S, make_sdesc(base + C::K_OFF + off, 16, 1024), make_sdesc(qs + off, 16, 1024), id_kk,
                   kk > 0 ? 1u : 0u);
        }
      };
      issue_st(0);
      for (int it = 0; it < nq; ++it) {
        const int st = it & 1;
        mark(16 * it + 0);
        if (it > 0) mbar_wait(dq_free, (it - 1) & 1);  // dQ_{it-1} read out of the dP columns
        mark(16 * it + 1);
        tc_fence_after();
        const uint32_t qs = base + C::Q_OFF + st * C::TILE, ds_ = base + C::DO_OFF + st * C::TILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::ATOM + (kk & 3) * 32;
          mma_bf16(T_DP, make_sdesc(base + C::V_OFF + off, 16, 1024), make_sdesc(ds_ + off, 16, 1024), id_kk,
                   kk > 0 ? 1u : 0u);
        }
        mma_commit(sp_full);
        mark(16 * it + 2);
        mbar_wait(ds_full, it & 1);
        mark(16 * it + 3);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K = 128 queries
          // dV += P^T dO : A = P^T (TMEM, 8 columns per k16), B = dO (MN-major: n = d)
          mma_bf16_ts(T_DV, T_S + (kk >> 2) * 64 + (kk & 3) * 8, make_sdesc(ds_ + kk * 2048, C::ATOM, 1024), id_kmn,
                      (it > 0 || kk > 0) ? 1u : 0u);
          // dK += dS^T Q : A = dS^T (smem K-major), B = Q (MN-major)
          mma_bf16(T_DK, make_sdesc(base + C::DS_OFF + (kk >> 2) * C::ATOM + (kk & 3) * 32, 16, 1024),
                   make_sdesc(qs + kk * 2048, C::ATOM, 1024), id_kmn, (it > 0 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K = 128 keys
          // dQ = dS K : A = dS (dS^T smem read MN-major, m = query), B = K (MN-major: n = d)
          mma_bf16(T_DP, make_sdesc(base + C::DS_OFF + kk * 2048, C::ATOM, 1024),
                   make_sdesc(base + C::K_OFF + kk * 2048, C::ATOM, 1024), id_mnmn, kk > 0 ? 1u : 0u);
        }
        mma_commit(mm_done);
        mma_commit(qd_empty0 + 8 * st);
        mark(16 * it + 4);
        if (it + 1 < nq) issue_st(it + 1);  // overlaps the dQ readout of this block
        mark(16 * it + 5);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // 8 warps: warp (q, hh) owns TMEM lane quarter q and column half hh of every tile
    const int q = warp & 3;
    const int hh = (warp - 4) >> 2;
    const int r = q * 32 + lane;  // key row for softmax-bwd; query row for the dQ readout
    const uint32_t lo = static_cast<uint32_t>(q * 32) << 16;
    const float sl2 = scale * LOG2E_;

    // lse/delta of the next query block are prefetched into registers one iteration ahead
    float nl = lse[(long long)bh * T + kblk * 128 + r] * LOG2E_;
    float nd = delta[(long long)bh * T + kblk * 128 + r];
    for (int it = 0; it < nq; ++it) {
      const int q0 = (kblk + it) * 128;
      if (r == 0 && hh == 0) mark(16 * it + 8);
      named_bar_sync(1, 256);  // previous iteration's lse/delta reads and staging TMA reads are done
      if (hh == 0) {
        sL[r] = nl;
        sDl[r] = nd;
      }
      named_bar_sync(1, 256);
      if (it + 1 < nq) {
        nl = lse[(long long)bh * T + q0 + 128 + r] * LOG2E_;
        nd = delta[(long long)bh * T + q0 + 128 + r];
      }
      if (r == 0 && hh == 0) mark(16 * it + 9);
      mbar_wait(sp_full, it & 1);
      if (r == 0 && hh == 0) mark(16 * it + 10);
      tc_fence_after();
#pragma unroll 1
      for (int c = 2 * hh; c < 2 * hh + 2; ++c) {  // 32 queries per chunk, this warp's half
        uint32_t sv[32], pv[32];
        tmem_ld32(T_S + lo + c * 32, sv);
        tmem_ld32(T_DP + lo + c * 32, pv);
        tmem_wait_ld();
        float p[32], ds[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int qi = c * 32 + j;
          float pj = fast_exp2(__uint_as_float(sv[j]) * sl2 - sL[qi]);
          if (it == 0 && r > qi) pj = 0.f;  // diagonal block: key after query
          p[j] = pj;
          ds[j] = pj * (__uint_as_float(pv[j]) - sDl[qi]) * scale;
        }
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(p[2 * j], p[2 * j + 1]);
        // P^T bf16 over S^T columns this warp has already consumed (each column half packs
        // into its own first 32 columns, so the other half's scores are never overwritten)
        tmem_st16(T_S + lo + (c >> 1) * 64 + (c & 1) * 16, pk);
        const uint32_t rowp = base + C::DS_OFF + (c >> 1) * C::ATOM + r * 128;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int c8 = (c & 1) * 4 + t;
          const float* s = &ds[t * 8];
          st_shared_v4(rowp + ((c8 ^ (r & 7)) << 4), pack_bf16(s[0], s[1]), pack_bf16(s[2], s[3]),
                       pack_bf16(s[4], s[5]), pack_bf16(s[6], s[7]));
        }
      }
      tmem_wait_st();
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(ds_full);
      if (r == 0 && hh == 0) mark(16 * it + 11);
      // dQ rows of this query block: thread r owns query q0 + r; this warp reads its column half
      mbar_wait(mm_done, it & 1);
      if (r == 0 && hh == 0) mark(16 * it + 12);
      tc_fence_after();
      constexpr int NCH = D / 64;  // 32-column chunks per warp
      uint32_t dqv[NCH][32];
#pragma unroll
      for (int cc = 0; cc < NCH; ++cc) tmem_ld32(T_DP + lo + (hh * NCH + cc) * 32, dqv[cc]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(dq_free);  // dQ is in registers: the dP columns may receive the next dP^T now
      if (r == 0 && hh == 0) mark(16 * it + 13);
      // stage each 32x32 fp32 chunk in this warp's 4 KB slice of the (free) dS^T tile and
      // TMA reduce-add it into the dQ workspace; runs while the next dP^T computes
      const uint32_t buf = base + C::DS_OFF + (warp - 4) * 4096;
#pragma unroll
      for (int cc = 0; cc < NCH; ++cc) {
        const int c = hh * NCH + cc;
        const uint32_t* v = dqv[cc];
        if (cc > 0) {
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          st_shared_v4(buf + lane * 128 + ((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_reduce_add_2d(&tm_dq, buf, h * D + c * 32, row_base + q0 + q * 32);
          bulk_commit();
        }
      }
      if (lane == 0) bulk_wait_read<0>();  // the staging slice is rewritten as dS^T next iteration
      __syncwarp();
      if (r == 0 && hh == 0) mark(16 * it + 14);
    }
    // final dK / dV rows (thread = key row)
    mbar_wait(mm_done, (nq - 1) & 1);
    tc_fence_after();
    bf16* dk = dqkv + ((long long)row_base + k0 + r) * 3 * H * D + (long long)H * D + (long long)h * D;
    bf16* dv = dk + (long long)H * D;
#pragma unroll 1
    for (int c = hh * (D / 64); c < (hh + 1) * (D / 64); ++c) {
      uint32_t a[32], bb[32];
      tmem_ld32(T_DK + lo + c * 32, a);
      tmem_ld32(T_DV + lo + c * 32, bb);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        *reinterpret_cast<uint4*>(dk + c * 32 + j) = make_uint4(
            pack_bf16(__uint_as_float(a[j]), __uint_as_float(a[j + 1])), pack_bf16(__uint_as_float(a[j + 2]), __uint_as_float(a[j + 3])),
            pack_bf16(__uint_as_float(a[j + 4]), __uint_as_float(a[j + 5])), pack_bf16(__uint_as_float(a[j + 6]), __uint_as_float(a[j + 7])));
        *reinterpret_cast<uint4*>(dv + c * 32 + j) = make_uint4(
            pack_bf16(__uint_as_float(bb[j]), __uint_as_float(bb[j + 1])), pack_bf16(__uint_as_float(bb[j + 2]), __uint_as_float(bb[j + 3])),
            pack_bf16(__uint_as_float(bb[j + 4]), __uint_as_float(bb[j + 5])), pack_bf16(__uint_as_float(bb[j + 6]), __uint_as_float(bb[j + 7])));
      }
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int D>
int attn_bwd_tc_launch(const void* qkv, const void* dout, const float* lse, const float* delta, void* dqkv,
                       float* dq_acc, int B, int T, int H, cudaStream_t s) {
  using C = TcBwdCfg<D>;
  CUtensorMap mq, mdo, mdq;
  cuuint32_t estr[2] = {1, 1};
  {
    cuuint64_t dims[2] = {(cuuint64_t)3 * H * D, (cuuint64_t)B * T};
    cuuint64_t strides[1] = {(cuuint64_t)3 * H * D * 2};
    cuuint32_t box[2] = {64, 128};
    int rc = encode_tensor_map(&mq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims, strides, box,
                               estr, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)H * D, (cuuint64_t)B * T};
    cuuint64_t strides[1] = {(cuuint64_t)H * D * 2};
    cuuint32_t box[2] = {64, 128};
    int rc = encode_tensor_map(&mdo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(dout), dims, strides, box,
                               estr, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)H * D, (cuuint64_t)B * T};
    cuuint64_t strides[1] = {(cuuint64_t)H * D * 4};
    cuuint32_t box[2] = {32, 32};
    int rc = encode_tensor_map(&mdq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dq_acc, dims, strides, box, estr,
                               CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_bwd_tc attr");
    set = true;
  }
  static int want_trace = -1;
  if (want_trace < 0) want_trace = getenv("ZPP_ATTN_TRACE") ? 1 : 0;
  unsigned long long* trace = nullptr;
  if (want_trace) cudaMalloc(&trace, 16 * 32 * sizeof(unsigned long long));
  attn_bwd_tc_kernel<D><<<dim3(T / 128, B * H), 384, C::SMEM, s>>>(mq, mdo, mdq, lse, delta, (bf16*)dqkv, dq_acc,
                                                                    T, H, 1.f / sqrtf((float)D), trace);
  if (trace) {
    unsigned long long h[16 * 32];
    cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
    const int nq = T / 128;
    const unsigned long long t0 = h[0];
    for (int it = 0; it < nq; ++it) {
      const unsigned long long* x = h + 16 * it;
      printf("it %2d | mma: start %7lld dqfree %7lld spcommit %7lld dsfull %7lld mmcommit %7lld st_next %7lld |"
             " sm: bar %7lld spwait %7lld spfull %7lld dsarrive %7lld mmdone %7lld readout %7lld bulk %7lld\n", it,
             (long long)(x[0] - t0), (long long)(x[1] - t0), (long long)(x[2] - t0), (long long)(x[3] - t0),
             (long long)(x[4] - t0), (long long)(x[5] - t0), (long long)(x[8] - t0), (long long)(x[9] - t0),
             (long long)(x[10] - t0), (long long)(x[11] - t0), (long long)(x[12] - t0), (long long)(x[13] - t0),
             (long long)(x[14] - t0));
    }
    cudaFree(trace);
  }
  return check_launch("attn_bwd_tc");
}

template int attn_bwd_tc_launch<64>(const void*, const void*, const float*, const float*, void*, float*, int, int,
                                    int, cudaStream_t);
template int attn_bwd_tc_launch<128>(const void*, const void*, const float*, const float*, void*, float*, int, int,
                                     int, cudaStream_t);

int attention_tc_preload() {
  cudaError_t e = cudaSuccess;
  e = (cudaError_t)(e | cudaFuncSetAttribute(attn_fwd_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcFwdCfg<64>::SMEM));
  e = (cudaError_t)(e | cudaFuncSetAttribute(attn_fwd_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcFwdCfg<128>::SMEM));
  e = (cudaError_t)(e | cudaFuncSetAttribute(attn_bwd_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcBwdCfg<64>::SMEM));
  e = (cudaError_t)(e | cudaFuncSetAttribute(attn_bwd_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcBwdCfg<128>::SMEM));
  return e == cudaSuccess ? ZPP_OK : set_cuda_error(e, "attention_tc preload");
}

}  // namespace zpp
