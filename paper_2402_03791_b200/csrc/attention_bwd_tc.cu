// Causal flash-attention BACKWARD on tcgen05, split into two kernels so that no partial
// dQ ever leaves the SM (the fused key-outer kernel in attention_tc.cu reduce-adds a
// 128x128 fp32 dQ partial per (key block, query block) pair through L2 -- 64 KB per pair
// -- and that reduction, not the tensor core, set its pace).
//
//   attn_bwd_dkdv_tc_kernel  one CTA per (128-key block j, batch*head), loop over query
//                            blocks i >= j:  S^T = K Q_i^T, dP^T = V dO_i^T,
//                            dV += P^T dO_i (A = P^T from TMEM), dK += dS^T Q_i (A = dS^T smem)
//   attn_bwd_dq_tc_kernel    one CTA per (128-query block i, batch*head), loop over key
//                            blocks j <= i:  S = Q K_j^T, dP = dO V_j^T,
//                            dQ += dS K_j (A = dS from TMEM, written over S)
//
// The dQ kernel recomputes S and dP (2 of its 3 MMAs), i.e. 7 MMAs per (i, j) pair instead
// of 5, but both kernels now keep the tensor pipe fed: every MMA that a softmax phase does
// not depend on is issued ahead of it.
//
// Shared conventions (as attention_tc.cu): qkv [B*T, 3*H*D] bf16, dout [B*T, H*D],
// lse [B, H, T] natural log, delta [B, H, T] = rowsum(O * dO); dqkv [B*T, 3*H*D] bf16.
// 128B-swizzled [128 rows][64 cols] bf16 smem atoms loaded by 2-D TMA boxes {64, 128}.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ptx.cuh"
#include "zpp_internal.h"

namespace zpp {

typedef __nv_bfloat16 bf16;

namespace {
constexpr float kLog2e = 1.4426950408889634f;
}

// ---------------------------------------------------------------------------------------
// dK / dV.  warp 0: TMA (K_j, V_j once; Q_i / dO_i ring of 2), warp 1: MMA issuer,
// warp 2: TMEM owner, warps 4..11: softmax-bwd (warp (q, hh) = TMEM lane quarter q,
// query-column half hh; thread = key row).
// TMEM: dV [0,128) dK [128,256) S^T / P^T [256,384) dP^T [384,512).
// MMA order per query block i (after ds_full(i)):  dV(i), S^T(i+1), dP^T(i+1), dK(i)
// -> the softmax of block i+1 starts after three MMAs while dK(i) still runs.
template <int D>
struct DkdvCfg {
  static constexpr int ATOM = 128 * 128;
  static constexpr int TILE = (D / 64) * ATOM;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + TILE;
  static constexpr int Q_OFF = V_OFF + TILE;        // 2 stages
  static constexpr int DO_OFF = Q_OFF + 2 * TILE;   // 2 stages
  static constexpr int DS_OFF = DO_OFF + 2 * TILE;  // dS^T: 2 atoms (128 keys x 128 queries)
  static constexpr int L_OFF = DS_OFF + 2 * ATOM;   // lse*log2e [128], delta [128]
  static constexpr int BAR_OFF = L_OFF + 1024;
  static constexpr int SMEM = BAR_OFF + 128 + 1024;
  static_assert(SMEM <= 232448, "smem budget");
};

template <int D>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                            const float* __restrict__ lse, const float* __restrict__ delta, bf16* __restrict__ dqkv,
                            int T, int H, float scale) {
  using C = DkdvCfg<D>;
  constexpr int NA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  float* sL = reinterpret_cast<float*>(gbase + C::L_OFF);
  float* sDl = sL + 128;
  const uint32_t bars = base + C::BAR_OFF;
  const uint32_t kv_full = bars, qd_full0 = bars + 8, qd_empty0 = bars + 24, sp_full = bars + 40;
  const uint32_t ds_full = bars + 48, ds_free = bars + 56, mm_done = bars + 64;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + C::BAR_OFF + 96);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int kblk = blockIdx.x;  // longest (most query blocks) first
  const int k0 = kblk * 128;
  const int nq = T / 128 - kblk;
  const int row_base = b * T;

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(qd_full0 + 8 * s, 1);
      mbar_init(qd_empty0 + 8 * s, 1);
    }
    mbar_init(sp_full, 1);
    mbar_init(ds_full, 256);
    mbar_init(ds_free, 1);
    mbar_init(mm_done, 1);
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
      mbar_wait(kv_full, 0);
      auto issue_sp = [&](int it) {  // S^T = K Q^T and dP^T = V dO^T of query block it
        const int st = it & 1;
        mbar_wait(qd_full0 + 8 * st, (it >> 1) & 1);
        tc_fence_after();
        const uint32_t qs = base + C::Q_OFF + st * C::TILE, ds_ = base + C::DO_OFF + st * C::TILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::ATOM + (kk & 3) * 32;
          mma_bf16(T_S, make_sdesc(base + C::K_OFF + off, 16, 1024), make_sdesc(qs + off, 16, 1024), id_kk,
                   kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::ATOM + (kk & 3) * 32;
          mma_bf16(T_DP, make_sdesc(base + C::V_OFF + off, 16, 1024), make_sdesc(ds_ + off, 16, 1024), id_kk,
                   kk > 0 ? 1u : 0u);
        }
        mma_commit(sp_full);
      };
      issue_sp(0);
      for (int it = 0; it < nq; ++it) {
        const int st = it & 1;
        const uint32_t qs = base + C::Q_OFF + st * C::TILE, ds_ = base + C::DO_OFF + st * C::TILE;
        mbar_wait(ds_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dV += P^T dO : A = P^T (TMEM, 8 packed columns per k16)
          mma_bf16_ts(T_DV, T_S + (kk >> 2) * 64 + (kk & 3) * 8, make_sdesc(ds_ + kk * 2048, C::ATOM, 1024), id_kmn,
                      (it > 0 || kk > 0) ? 1u : 0u);
        if (it + 1 < nq) issue_sp(it + 1);  // S^T over P^T after dV read it (in-order pipe)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dK += dS^T Q : A = dS^T (smem K-major), B = Q (MN-major)
          mma_bf16(T_DK, make_sdesc(base + C::DS_OFF + (kk >> 2) * C::ATOM + (kk & 3) * 32, 16, 1024),
                   make_sdesc(qs + kk * 2048, C::ATOM, 1024), id_kmn, (it > 0 || kk > 0) ? 1u : 0u);
        mma_commit(ds_free);
        mma_commit(qd_empty0 + 8 * st);
      }
      mma_commit(mm_done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int hh = (warp - 4) >> 2;
    const int r = q * 32 + lane;  // key row
    const uint32_t lo = static_cast<uint32_t>(q * 32) << 16;
    const float sl2 = scale * kLog2e;
    float nl = lse[(long long)bh * T + kblk * 128 + r] * kLog2e;
    float nd = delta[(long long)bh * T + kblk * 128 + r];
    for (int it = 0; it < nq; ++it) {
      const int q0 = (kblk + it) * 128;
      named_bar_sync(1, 256);  // everyone is done reading the previous block's lse / delta
      if (hh == 0) {
        sL[r] = nl;
        sDl[r] = nd;
      }
      named_bar_sync(1, 256);
      if (it + 1 < nq) {
        nl = lse[(long long)bh * T + q0 + 128 + r] * kLog2e;
        nd = delta[(long long)bh * T + q0 + 128 + r];
      }
      mbar_wait(sp_full, it & 1);
      tc_fence_after();
      if (it > 0) mbar_wait(ds_free, (it - 1) & 1);  // dK(it-1) finished reading dS^T smem
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
        // P^T bf16 over the S^T columns this warp already consumed (each column half packs into
        // its own first 32 columns, so the other half's scores are never overwritten)
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
    }
    // final dK / dV rows (thread = key row)
    mbar_wait(mm_done, 0);
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
            pack_bf16(__uint_as_float(a[j]), __uint_as_float(a[j + 1])),
            pack_bf16(__uint_as_float(a[j + 2]), __uint_as_float(a[j + 3])),
            pack_bf16(__uint_as_float(a[j + 4]), __uint_as_float(a[j + 5])),
            pack_bf16(__uint_as_float(a[j + 6]), __uint_as_float(a[j + 7])));
        *reinterpret_cast<uint4*>(dv + c * 32 + j) = make_uint4(
            pack_bf16(__uint_as_float(bb[j]), __uint_as_float(bb[j + 1])),
            pack_bf16(__uint_as_float(bb[j + 2]), __uint_as_float(bb[j + 3])),
            pack_bf16(__uint_as_float(bb[j + 4]), __uint_as_float(bb[j + 5])),
            pack_bf16(__uint_as_float(bb[j + 6]), __uint_as_float(bb[j + 7])));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------------------
// dQ.  warp 0: TMA (Q_i, dO_i once; K_j ring of 3 -- K is read by S_j and dQ_j), warp 3:
// TMA V_j ring of 2, warp 1: MMA issuer, warp 2: TMEM owner, warps 4..11: thread = query
// row, warp (q, hh) takes key-column half hh (2 softmax warps per SM sub-partition).
// TMEM: S_j double buffer [0,256) (dS_j bf16: each 64-key half packed over the first 32 of
// its own S columns), dP [256,384), dQ [384,512).
// Per key block j the row threads compute P = exp2(S*scale*log2e - lse*log2e) as soon as
// S_j lands, then wait for dP_j, form dS = P (dP - delta) * scale into TMEM and signal; the
// MMA warp then issues dP_{j+1} (dP's columns are free) and dQ += dS_j K_j, with S_{j+1}
// already issued one block ahead.
template <int D>
struct DqCfg {
  static constexpr int ATOM = 128 * 128;
  static constexpr int TILE = (D / 64) * ATOM;
  static constexpr int KST = 3;
  static constexpr int Q_OFF = 0;
  static constexpr int DO_OFF = Q_OFF + TILE;
  static constexpr int K_OFF = DO_OFF + TILE;      // KST stages
  static constexpr int V_OFF = K_OFF + KST * TILE;  // 2 stages
  static constexpr int BAR_OFF = V_OFF + 2 * TILE;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static_assert(SMEM <= 232448, "smem budget");
};

template <int D>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                          const float* __restrict__ lse, const float* __restrict__ delta, bf16* __restrict__ dqkv,
                          int T, int H, float scale) {
  using C = DqCfg<D>;
  constexpr int NA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bars = base + C::BAR_OFF;
  const uint32_t qd_full = bars, k_full0 = bars + 8, k_empty0 = bars + 32, v_full0 = bars + 56;
  const uint32_t v_empty0 = bars + 72, s_full0 = bars + 88, dp_full = bars + 104, ds_full = bars + 112;
  const uint32_t dq_done = bars + 120;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + C::BAR_OFF + 192);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int qblk = gridDim.x - 1 - blockIdx.x;  // longest (most key blocks) first
  const int q0 = qblk * 128;
  const int nkb = qblk + 1;
  const int row_base = b * T;

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    mbar_init(qd_full, 1);
    for (int s = 0; s < C::KST; ++s) {
      mbar_init(k_full0 + 8 * s, 1);
      mbar_init(k_empty0 + 8 * s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(v_full0 + 8 * s, 1);
      mbar_init(v_empty0 + 8 * s, 1);
      mbar_init(s_full0 + 8 * s, 1);
    }
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 256);
    mbar_init(dq_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t T_S = tmem, T_DP = tmem + 256, T_DQ = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(qd_full, 2 * C::TILE);
      for (int a = 0; a < NA; ++a) {
        tma_load_2d(base + C::Q_OFF + a * C::ATOM, &tm_qkv, qd_full, h * D + 64 * a, row_base + q0);
        tma_load_2d(base + C::DO_OFF + a * C::ATOM, &tm_do, qd_full, h * D + 64 * a, row_base + q0);
      }
      for (int j = 0; j < nkb; ++j) {
        const int st = j % C::KST;
        mbar_wait(k_empty0 + 8 * st, ((j / C::KST) & 1) ^ 1);
        const uint32_t fb = k_full0 + 8 * st;
        mbar_arrive_expect_tx(fb, C::TILE);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(base + C::K_OFF + st * C::TILE + a * C::ATOM, &tm_qkv, fb, H * D + h * D + 64 * a,
                      row_base + j * 128);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (lane == 0) {
      for (int j = 0; j < nkb; ++j) {
        const int st = j & 1;
        mbar_wait(v_empty0 + 8 * st, ((j >> 1) & 1) ^ 1);
        const uint32_t fb = v_full0 + 8 * st;
        mbar_arrive_expect_tx(fb, C::TILE);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(base + C::V_OFF + st * C::TILE + a * C::ATOM, &tm_qkv, fb, 2 * H * D + h * D + 64 * a,
                      row_base + j * 128);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = make_idesc_bf16(128, 128, false, false);  // S, dP (N = 128 keys)
      constexpr uint32_t id_q = make_idesc_bf16(128, D, false, true);     // dQ (B = K MN-major, N = d)
      auto issue_s = [&](int j) {
        const int st = j % C::KST;
        mbar_wait(k_full0 + 8 * st, (j / C::KST) & 1);
        tc_fence_after();
        const uint32_t kb = base + C::K_OFF + st * C::TILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::ATOM + (kk & 3) * 32;
          mma_bf16(T_S + (j & 1) * 128, make_sdesc(base + C::Q_OFF + off, 16, 1024), make_sdesc(kb + off, 16, 1024),
                   id_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(s_full0 + 8 * (j & 1));
      };
      auto issue_dp = [&](int j) {
        const int st = j & 1;
        mbar_wait(v_full0 + 8 * st, (j >> 1) & 1);
        tc_fence_after();
        const uint32_t vb = base + C::V_OFF + st * C::TILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::ATOM + (kk & 3) * 32;
          mma_bf16(T_DP, make_sdesc(base + C::DO_OFF + off, 16, 1024), make_sdesc(vb + off, 16, 1024), id_s,
                   kk > 0 ? 1u : 0u);
        }
        mma_commit(dp_full);
        mma_commit(v_empty0 + 8 * st);
      };
      mbar_wait(qd_full, 0);
      issue_s(0);
      issue_dp(0);
      for (int j = 0; j < nkb; ++j) {
        if (j + 1 < nkb) issue_s(j + 1);  // S buffer (j+1)&1 was consumed by block j-1
        mbar_wait(ds_full, j & 1);
        tc_fence_after();
        if (j + 1 < nkb) issue_dp(j + 1);  // the row threads have read dP_j
        const uint32_t kb = base + C::K_OFF + (j % C::KST) * C::TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dQ += dS K : A = dS (TMEM; each 64-key half packed in its first 32 columns)
          mma_bf16_ts(T_DQ, T_S + (j & 1) * 128 + (kk >> 2) * 64 + (kk & 3) * 8,
                      make_sdesc(kb + kk * 2048, C::ATOM, 1024), id_q, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(k_empty0 + 8 * (j % C::KST));
      }
      mma_commit(dq_done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // 8 warps: warp (q, hh) owns TMEM lane quarter q (query rows) and key-column half hh
    const int q = warp & 3;
    const int hh = (warp - 4) >> 2;
    const int r = q * 32 + lane;  // query row == TMEM lane
    const uint32_t lo = static_cast<uint32_t>(q * 32) << 16;
    const float sl2 = scale * kLog2e;
    const float lse_r = lse[(long long)bh * T + q0 + r] * kLog2e;
    const float del_r = delta[(long long)bh * T + q0 + r];
    for (int j = 0; j < nkb; ++j) {
      const uint32_t ts = T_S + lo + (j & 1) * 128 + hh * 64;
      mbar_wait(s_full0 + 8 * (j & 1), (j >> 1) & 1);
      tc_fence_after();
      float p[64];
      {
        uint32_t v0[32], v1[32];
        tmem_ld32(ts, v0);
        tmem_ld32(ts + 32, v1);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          p[k] = fast_exp2(__uint_as_float(v0[k]) * sl2 - lse_r);
          p[32 + k] = fast_exp2(__uint_as_float(v1[k]) * sl2 - lse_r);
        }
      }
      if (j == nkb - 1) {  // diagonal block: keys after the query
#pragma unroll
        for (int k = 0; k < 64; ++k)
          if (hh * 64 + k > r) p[k] = 0.f;
      }
      mbar_wait(dp_full, j & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t v[32];
        tmem_ld32(T_DP + lo + hh * 64 + c * 32, v);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float d0 = p[c * 32 + 2 * k] * (__uint_as_float(v[2 * k]) - del_r) * scale;
          const float d1 = p[c * 32 + 2 * k + 1] * (__uint_as_float(v[2 * k + 1]) - del_r) * scale;
          pk[k] = pack_bf16(d0, d1);
        }
        // dS of this half's 64 keys packed into the half's first 32 columns, over S values
        // this warp has already read (the other half's columns are never touched)
        tmem_st16(ts + c * 16, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    mbar_wait(dq_done, 0);
    tc_fence_after();
    bf16* dq = dqkv + ((long long)row_base + q0 + r) * 3 * H * D + (long long)h * D;
#pragma unroll 1
    for (int c = hh * (D / 64); c < (hh + 1) * (D / 64); ++c) {
      uint32_t v[32];
      tmem_ld32(T_DQ + lo + c * 32, v);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; k += 8)
        *reinterpret_cast<uint4*>(dq + c * 32 + k) =
            make_uint4(pack_bf16(__uint_as_float(v[k]), __uint_as_float(v[k + 1])),
                       pack_bf16(__uint_as_float(v[k + 2]), __uint_as_float(v[k + 3])),
                       pack_bf16(__uint_as_float(v[k + 4]), __uint_as_float(v[k + 5])),
                       pack_bf16(__uint_as_float(v[k + 6]), __uint_as_float(v[k + 7])));
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int D>
int attn_bwd_split_tc_launch(const void* qkv, const void* dout, const float* lse, const float* delta, void* dqkv,
                             int B, int T, int H, cudaStream_t s) {
  CUtensorMap mq, mdo;
  cuuint32_t estr[2] = {1, 1};
  cuuint32_t box[2] = {64, 128};
  {
    cuuint64_t dims[2] = {(cuuint64_t)3 * H * D, (cuuint64_t)B * T};
    cuuint64_t strides[1] = {(cuuint64_t)3 * H * D * 2};
    int rc = encode_tensor_map(&mq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims, strides, box,
                               estr, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)H * D, (cuuint64_t)B * T};
    cuuint64_t strides[1] = {(cuuint64_t)H * D * 2};
    int rc = encode_tensor_map(&mdo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(dout), dims, strides, box,
                               estr, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_dkdv_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         DkdvCfg<D>::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dq_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, DqCfg<D>::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_bwd_split attr");
    set = true;
  }
  const float scale = 1.f / sqrtf((float)D);
  attn_bwd_dkdv_tc_kernel<D><<<dim3(T / 128, B * H), 384, DkdvCfg<D>::SMEM, s>>>(mq, mdo, lse, delta, (bf16*)dqkv, T,
                                                                                   H, scale);
  int rc = check_launch("attn_bwd_dkdv_tc");
  if (rc) return rc;
  attn_bwd_dq_tc_kernel<D><<<dim3(T / 128, B * H), 384, DqCfg<D>::SMEM, s>>>(mq, mdo, lse, delta, (bf16*)dqkv, T, H,
                                                                             scale);
  return check_launch("attn_bwd_dq_tc");
}

template int attn_bwd_split_tc_launch<64>(const void*, const void*, const float*, const float*, void*, int, int, int,
                                          cudaStream_t);
template int attn_bwd_split_tc_launch<128>(const void*, const void*, const float*, const float*, void*, int, int, int,
                                           cudaStream_t);

int attention_bwd_tc_preload() {
  cudaError_t e = cudaSuccess;
  e = (cudaError_t)(e | cudaFuncSetAttribute(attn_bwd_dkdv_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             DkdvCfg<64>::SMEM));
  e = (cudaError_t)(e | cudaFuncSetAttribute(attn_bwd_dkdv_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             DkdvCfg<128>::SMEM));
  e = (cudaError_t)(e | cudaFuncSetAttribute(attn_bwd_dq_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             DqCfg<64>::SMEM));
  e = (cudaError_t)(e | cudaFuncSetAttribute(attn_bwd_dq_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             DqCfg<128>::SMEM));
  return e == cudaSuccess ? ZPP_OK : set_cuda_error(e, "attention_bwd_tc preload");
}

}  // namespace zpp
