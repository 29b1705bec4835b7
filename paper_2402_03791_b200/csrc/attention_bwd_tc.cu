// Causal flash-attention BACKWARD on tcgen05 — two deterministic kernels, fully double-buffered
// in TMEM by working on 64-wide tiles of the loop dimension.
//
//   attn_bwd_dq_kernel    (launched first) one CTA per (128-query block i, b*h).
//       Prologue: delta_i = rowsum(O_i * dO_i) (fp32, fixed order) and lse2 = lse*log2(e) for
//       its 128 rows, both written to the workspace for the dK/dV kernel -- this replaces the
//       separate delta pass (one read of O, and dO is already in smem).
//       Loop over 64-key tiles j (keys <= last query):
//         S_j = Q K_j^T, dP_j = dO V_j^T                (M=128 queries, N=64 keys)
//         dS  = exp2(S*scale*log2e - lse2) (dP - delta) * scale   -> bf16 over S_j in TMEM
//         dQ += dS K_j                                    (A = dS from TMEM, M=128, N=d)
//   attn_bwd_dkdv_kernel  one CTA per (128-key block, b*h), loop over 64-query tiles:
//         S^T = K Q^T, dP^T = V dO^T                      (M=128 keys, N=64 queries)
//         P^T -> bf16 over S^T in TMEM, dS^T -> smem (128B-swizzled, K-major)
//         dV += P^T dO (A from TMEM), dK += dS^T Q        (M=128 keys, N=d)
//
// Why 64-wide tiles: with d = 128 the two 128x128 fp32 accumulators (dK, dV) take 256 of the
// 512 TMEM columns.  A 64-query S^T / dP^T pair is 128 columns, so BOTH can be double
// buffered: the softmax of tile t+1 runs while the tensor core executes dV(t), dK(t),
// S^T(t+2), dP^T(t+2) -- the pipe never waits for the exp2 phase.  Same in the dQ kernel
// (S and dP double-buffered, 256 columns, + dQ).
// No partial gradient leaves the SM and there are no atomics: every output is a fixed-order
// fp32 sum, so the backward is bit-reproducible run to run.
//
// Conventions: qkv [B*T, 3*H*D] bf16, out/dout [B*T, H*D], lse [B, H, T] natural log;
// workspace = delta [B*H*T] | lse2 [B*H*T] fp32; dqkv [B*T, 3*H*D] bf16.  T % 128 == 0.
// smem tiles are [rows][64 bf16] 128B-swizzled atoms loaded by 2-D TMA boxes {64, rows}.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ptx.cuh"
#include "zpp_internal.h"

namespace zpp {

typedef __nv_bfloat16 bf16;

#ifdef ZPP_TRACE
// Debug build only (make trace): clock64 stamps of CTA 0, [kernel][slot][tile], read by tools/attn_trace.py
__device__ unsigned long long g_attn_trace[2][8][64];
#ifndef ZPP_TRACE_CTA
#define ZPP_TRACE_CTA 0  // which CTA is traced (e.g. -DZPP_TRACE_CTA=640: a CTA of the 5th wave)
#endif
#define ZTRACE(k, slot, t) \
  do {                     \
    if (blockIdx.x == ZPP_TRACE_CTA && (t) < 64) g_attn_trace[k][slot][t] = clock64(); \
  } while (0)
#else
#define ZTRACE(k, slot, t) \
  do {                     \
  } while (0)
#endif

namespace {
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float dot8(uint4 a, uint4 b) {
  float s = bf16lo(a.x) * bf16lo(b.x);
  s = fmaf(bf16hi(a.x), bf16hi(b.x), s);
  s = fmaf(bf16lo(a.y), bf16lo(b.y), s);
  s = fmaf(bf16hi(a.y), bf16hi(b.y), s);
  s = fmaf(bf16lo(a.z), bf16lo(b.z), s);
  s = fmaf(bf16hi(a.z), bf16hi(b.z), s);
  s = fmaf(bf16lo(a.w), bf16lo(b.w), s);
  return fmaf(bf16hi(a.w), bf16hi(b.w), s);
}

// One arrival per warp on an mbarrier initialised with the number of arriving warps: a
// 256/512-thread barrier takes every lane's arrive as a serialised shared-memory atomic, which
// cost ~200 cycles of tensor-core idle per tile (measured).  Each lane's own prior TMEM
// accesses are complete (tcgen05.wait::*) and its smem stores fenced before the __syncwarp.
__device__ __forceinline__ void warp_arrive(uint32_t bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}

// Epilogue staging: thread = TMEM lane r of a 128-row fp32 accumulator, columns [c0, c0 + W)
// -> bf16 into a 128B-swizzled smem tile of [128 rows][64 cols] atoms (the TMA box layout), so
// one thread can then TMA-store the whole tile: each warp writing 32 different rows straight
// to global memory cost ~4k cycles of uncoalesced stores per tile (measured, dK/dV epilogue).
template <int W>
__device__ __forceinline__ void stage_acc(uint32_t tacc, uint32_t lo, int r, int c0, uint32_t tile) {
  uint32_t v[32];
  if constexpr (W == 32) {
    tmem_ld32(tacc + lo + c0, v);
  } else {
    tmem_ld16(tacc + lo + c0, *reinterpret_cast<uint32_t(*)[16]>(v));
  }
  tmem_wait_ld();
#pragma unroll
  for (int k = 0; k < W; k += 8) {
    const int col = c0 + k;  // multiple of 8: one 16-byte chunk
    const uint32_t atom = tile + (col >> 6) * (128 * 128), chunk = (col & 63) >> 3;
    st_shared_v4(atom + r * 128 + ((chunk ^ (r & 7)) << 4),
                 pack_bf16(__uint_as_float(v[k]), __uint_as_float(v[k + 1])),
                 pack_bf16(__uint_as_float(v[k + 2]), __uint_as_float(v[k + 3])),
                 pack_bf16(__uint_as_float(v[k + 4]), __uint_as_float(v[k + 5])),
                 pack_bf16(__uint_as_float(v[k + 6]), __uint_as_float(v[k + 7])));
  }
}

}  // namespace

// ---------------------------------------------------------------------------------------
// dQ (+ delta, lse2).  warp 0: TMA Q, dO once, K_j ring of 5 (K_j is read by S_j and dQ_j);
// warp 3: TMA V_j ring of 4; warp 1: MMA issuer; warp 2: TMEM owner; warps 4..11: thread =
// query row (TMEM lane), warp (quarter q, half hh) takes keys [32hh, 32hh+32) of each tile.
// TMEM: S/dS [0,128) (2 x 64), dP [128,256) (2 x 64), dQ [256, 256+D).
template <int D>
struct BwdDqCfg {
  static constexpr int QATOM = 128 * 128;  // [128 rows][64 bf16]
  static constexpr int QTILE = (D / 64) * QATOM;
  static constexpr int KATOM = 64 * 128;   // [64 rows][64 bf16]
  static constexpr int KTILE = (D / 64) * KATOM;
  // deep K / V rings: the load of K_{j+KST} can only start when dQ(j) retires, and at the
  // tensor core's rate one 64-key tile takes ~0.5 us -- an L2 TMA round trip is about as long
  static constexpr int KST = 5, VST = 4;
  static constexpr int Q_OFF = 0;
  static constexpr int DO_OFF = Q_OFF + QTILE;
  static constexpr int K_OFF = DO_OFF + QTILE;
  static constexpr int V_OFF = K_OFF + KST * KTILE;
  static constexpr int RED_OFF = V_OFF + VST * KTILE;  // float [2][128] delta halves
  static constexpr int BAR_OFF = RED_OFF + 1024;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static_assert(SMEM <= 232448, "smem budget");
};

template <int D>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                       const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_st,
                       const bf16* __restrict__ out,
                       const float* __restrict__ lse, float* __restrict__ delta_out, float* __restrict__ lse2_out,
                       bf16* __restrict__ dqkv, int T, int H, int BH, float scale) {
  using C = BwdDqCfg<D>;
  constexpr int NA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  float* red = reinterpret_cast<float*>(gbase + C::RED_OFF);
  const uint32_t bars = base + C::BAR_OFF;
  const uint32_t qd_full = bars, k_full0 = bars + 8, k_empty0 = k_full0 + 8 * C::KST;
  const uint32_t v_full0 = k_empty0 + 8 * C::KST, v_empty0 = v_full0 + 8 * C::VST;
  const uint32_t s_full0 = v_empty0 + 8 * C::VST, dp_full0 = s_full0 + 16, ds_full0 = dp_full0 + 16;
  const uint32_t dq_done = ds_full0 + 16, qt_full = dq_done + 8;
  static_assert(8 * (1 + 2 * C::KST + 2 * C::VST + 8) <= 240, "barrier area");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + C::BAR_OFF + 240);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 128) ZTRACE(0, 0, 63);
  // programmatic dependent launch: once every dQ CTA is resident, dK/dV CTAs may take the SMs
  // the dQ tail frees (they wait for our delta / lse2 with griddepcontrol.wait)
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // 1-D grid, heaviest query blocks first across ALL heads
  const int nqb = T / 128;
  const int bh = blockIdx.x % BH, b = bh / H, h = bh % H;
  const int qblk = nqb - 1 - static_cast<int>(blockIdx.x) / BH;
  const int q0 = qblk * 128;
  const int nkt = 2 * (qblk + 1);  // 64-key tiles up to the diagonal
  const int row_base = b * T;

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_kv);
    tma_prefetch(&tm_do);
    mbar_init(qd_full, 1);
    for (int s = 0; s < C::KST; ++s) {
      mbar_init(k_full0 + 8 * s, 1);
      mbar_init(k_empty0 + 8 * s, 1);
    }
    for (int s = 0; s < C::VST; ++s) {
      mbar_init(v_full0 + 8 * s, 1);
      mbar_init(v_empty0 + 8 * s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(s_full0 + 8 * s, 1);
      mbar_init(dp_full0 + 8 * s, 1);
      mbar_init(ds_full0 + 8 * s, 8);  // one arrival per row warp
    }
    mbar_init(dq_done, 1);
    mbar_init(qt_full, 8);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Q and dO live in TMEM as the A operands of S and dP (TS-mode MMAs: an SS MMA with N = 64
  // is bound by the smem read of its 128-row A operand, 48 instead of 32 cycles per K16)
  const uint32_t T_S = tmem, T_DP = tmem + 128, T_DQ = tmem + 256, T_Q = T_DQ + D, T_DO = T_Q + D / 2;
  if (threadIdx.x == 128) ZTRACE(0, 1, 63);

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(qd_full, 2 * C::QTILE);
      for (int a = 0; a < NA; ++a) {
        tma_load_2d(base + C::Q_OFF + a * C::QATOM, &tm_q, qd_full, h * D + 64 * a, row_base + q0);
        tma_load_2d(base + C::DO_OFF + a * C::QATOM, &tm_do, qd_full, h * D + 64 * a, row_base + q0);
      }
      for (int j = 0; j < nkt; ++j) {
        const int st = j % C::KST;
        mbar_wait(k_empty0 + 8 * st, ((j / C::KST) & 1) ^ 1);
        const uint32_t fb = k_full0 + 8 * st;
        mbar_arrive_expect_tx(fb, C::KTILE);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(base + C::K_OFF + st * C::KTILE + a * C::KATOM, &tm_kv, fb, H * D + h * D + 64 * a,
                      row_base + j * 64);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (lane == 0) {
      for (int j = 0; j < nkt; ++j) {
        const int st = j % C::VST;
        mbar_wait(v_empty0 + 8 * st, ((j / C::VST) & 1) ^ 1);
        const uint32_t fb = v_full0 + 8 * st;
        mbar_arrive_expect_tx(fb, C::KTILE);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(base + C::V_OFF + st * C::KTILE + a * C::KATOM, &tm_kv, fb, 2 * H * D + h * D + 64 * a,
                      row_base + j * 64);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {  // whole warp: uniform descriptors, elect.sync issues
      constexpr uint32_t id_s = make_idesc_bf16(128, 64, false, false);  // S, dP: N = 64 keys
      constexpr uint32_t id_q = make_idesc_bf16(128, D, false, true);    // dQ: B = K_j N-major (N = d)
      auto issue_s = [&](int j) {
        const int st = j % C::KST;
        mbar_wait(k_full0 + 8 * st, (j / C::KST) & 1);
        tc_fence_after();
        const uint32_t kb = base + C::K_OFF + st * C::KTILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16_ts_w(T_S + (j & 1) * 64, T_Q + kk * 8,
                        make_sdesc(kb + (kk >> 2) * C::KATOM + (kk & 3) * 32, 16, 1024), id_s, kk > 0 ? 1u : 0u);
        mma_commit_w(s_full0 + 8 * (j & 1));
      };
      auto issue_dp = [&](int j) {
        const int st = j % C::VST;
        mbar_wait(v_full0 + 8 * st, (j / C::VST) & 1);
        tc_fence_after();
        const uint32_t vb = base + C::V_OFF + st * C::KTILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16_ts_w(T_DP + (j & 1) * 64, T_DO + kk * 8,
                        make_sdesc(vb + (kk >> 2) * C::KATOM + (kk & 3) * 32, 16, 1024), id_s, kk > 0 ? 1u : 0u);
        mma_commit_w(dp_full0 + 8 * (j & 1));
        mma_commit_w(v_empty0 + 8 * st);
      };
      mbar_wait(qt_full, 0);  // Q, dO copied into TMEM by the row threads
      tc_fence_after();
      issue_s(0);
      issue_dp(0);
      if (nkt > 1) {
        issue_s(1);
        issue_dp(1);
      }
      for (int j = 0; j < nkt; ++j) {
        ZTRACE(0, 0, j);
        mbar_wait(ds_full0 + 8 * (j & 1), (j >> 1) & 1);
        ZTRACE(0, 1, j);
        tc_fence_after();
        const uint32_t kb = base + C::K_OFF + (j % C::KST) * C::KTILE;
        // dQ += dS K_j: A = dS in TMEM (each 32-key half packed into its first 16 columns)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16_ts_w(T_DQ, T_S + (j & 1) * 64 + (kk >> 1) * 32 + (kk & 1) * 8,
                      make_sdesc(kb + kk * 2048, C::KATOM, 1024), id_q, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit_w(k_empty0 + 8 * (j % C::KST));
        if (j + 2 < nkt) {  // buffers (j & 1): dS_j read by the dQ MMA above (in-order pipe)
          issue_s(j + 2);
          ZTRACE(0, 2, j);
          issue_dp(j + 2);
        }
        ZTRACE(0, 3, j);
      }
      mma_commit_w(dq_done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int hh = (warp - 4) >> 2;
    const int r = q * 32 + lane;  // query row == TMEM lane
    const uint32_t lo = static_cast<uint32_t>(q * 32) << 16;
    const float sl2 = scale * kLog2e;
    const float lse2_r = lse[(long long)bh * T + q0 + r] * kLog2e;
    // delta = rowsum(O * dO): this thread sums half hh of the row's D columns (O from global,
    // read once here; dO from the swizzled smem tile)
    constexpr int CH = D / 16;  // 16-byte chunks per half row
    uint4 ov[CH];
    const uint4* orow = reinterpret_cast<const uint4*>(out + ((long long)row_base + q0 + r) * H * D + h * D) + hh * CH;
#pragma unroll
    for (int i = 0; i < CH; ++i) ov[i] = __ldg(orow + i);
    mbar_wait(qd_full, 0);
    if (threadIdx.x == 128) ZTRACE(0, 2, 63);
    float acc = 0.f;
    {
      // this thread's half row of Q and dO -> TMEM (lane r, packed bf16 pairs), and delta
      uint32_t qv[4 * CH], dv[4 * CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int cg = hh * CH + i;  // global chunk index along D
        const uint32_t off = (cg >> 3) * C::QATOM + r * 128 + (((cg & 7) ^ (r & 7)) << 4);
        const uint4 d4 = ld_shared_v4(base + C::DO_OFF + off);
        const uint4 q4 = ld_shared_v4(base + C::Q_OFF + off);
        acc += dot8(ov[i], d4);
        dv[4 * i] = d4.x, dv[4 * i + 1] = d4.y, dv[4 * i + 2] = d4.z, dv[4 * i + 3] = d4.w;
        qv[4 * i] = q4.x, qv[4 * i + 1] = q4.y, qv[4 * i + 2] = q4.z, qv[4 * i + 3] = q4.w;
      }
      if constexpr (CH == 8) {
        tmem_st32(T_Q + lo + hh * 32, qv);
        tmem_st32(T_DO + lo + hh * 32, dv);
      } else {
        tmem_st16(T_Q + lo + hh * 16, qv);
        tmem_st16(T_DO + lo + hh * 16, dv);
      }
      tmem_wait_st();
      tc_fence_before();
      warp_arrive(qt_full);
    }
    red[hh * 128 + r] = acc;
    named_bar_sync(1, 256);
    const float delta_r = red[r] + red[128 + r];
    if (hh == 0) {
      delta_out[(long long)bh * T + q0 + r] = delta_r;
      lse2_out[(long long)bh * T + q0 + r] = lse2_r;
    }
    for (int j = 0; j < nkt; ++j) {
      const int buf = j & 1;
      const uint32_t par = (j >> 1) & 1;
      const uint32_t ts = T_S + lo + buf * 64 + hh * 32;
#ifdef ZPP_TRACE_NOSM  // debug experiment: MMA pipeline alone (softmax warps only hand over)
      mbar_wait(s_full0 + 8 * buf, par);
      mbar_wait(dp_full0 + 8 * buf, par);
      tc_fence_before();
      warp_arrive(ds_full0 + 8 * buf);
      if (threadIdx.x == 128) ZTRACE(0, 7, j);
      continue;
#endif
      if (threadIdx.x == 128) ZTRACE(0, 4, j);
      mbar_wait(s_full0 + 8 * buf, par);
      if (threadIdx.x == 128) ZTRACE(0, 5, j);
      tc_fence_after();
      float p[32];
      {
        uint32_t v[32];
        tmem_ld32(ts, v);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 32; ++k) p[k] = fast_exp2(fmaf(__uint_as_float(v[k]), sl2, -lse2_r));
      }
      if (j >= nkt - 2) {  // the two tiles that straddle the diagonal: keys after the query
        const int kq = j * 64 + hh * 32 - q0 - r;
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (kq + k > 0) p[k] = 0.f;
      }
      if (threadIdx.x == 128) ZTRACE(0, 6, j);
      mbar_wait(dp_full0 + 8 * buf, par);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(T_DP + lo + buf * 64 + hh * 32, v);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int k = 0; k < 16; ++k)
        pk[k] = pack_bf16(p[2 * k] * (__uint_as_float(v[2 * k]) - delta_r) * scale,
                          p[2 * k + 1] * (__uint_as_float(v[2 * k + 1]) - delta_r) * scale);
      tmem_st16(ts, pk);  // over S columns this warp has already read
      tmem_wait_st();
      tc_fence_before();
      warp_arrive(ds_full0 + 8 * buf);
      if (threadIdx.x == 128) ZTRACE(0, 7, j);
    }
    mbar_wait(dq_done, 0);
    if (threadIdx.x == 128) ZTRACE(0, 4, 63);
    tc_fence_after();
    // dQ -> swizzled smem (the Q tile's slot: Q lives in TMEM now) -> TMA store
    for (int c = hh * (D / 2); c < (hh + 1) * (D / 2); c += 32) stage_acc<32>(T_DQ, lo, r, c, base + C::Q_OFF);
    fence_proxy_async();
    named_bar_sync(1, 256);
    if (threadIdx.x == 128) {
      for (int a = 0; a < NA; ++a) tma_store_2d(&tm_st, base + C::Q_OFF + a * C::QATOM, h * D + 64 * a, row_base + q0);
      bulk_commit();
      bulk_wait_all();
    }
    if (threadIdx.x == 128) ZTRACE(0, 5, 63);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------------------
// dK / dV.  warp 0: TMA K, V once, then Q_t / dO_t (+ lse2_t, delta_t) through a ring of 3;
// warp 1: MMA issuer; warp 2: TMEM owner; warps 4..19: thread = key row (TMEM lane), warp
// (quarter q, part) takes queries [16 part, 16 part + 16) of each 64-query tile.
// K and V are copied into TMEM once (the A operands of S^T / dP^T: TS-mode MMAs run at the
// tensor core's rate for N = 64, the SS form is bound by re-reading the 128-row A from smem).
// S^T / dP^T are single-buffered but released as soon as the row threads have loaded them,
// so S^T(t+1), dP^T(t+1) run while the exp2 phase of tile t does; P^T and dS^T go to smem
// (the A operands of dV += P^T dO and dK += dS^T Q, N = d = 128: full rate from smem).
// TMEM: dV [0,D) dK [D,2D) K [2D,2D+D/2) V [2D+D/2,3D) S^T [3D,3D+64) dP^T [3D+64,3D+128).
template <int D>
struct BwdDkdvCfg {
  static constexpr int KATOM = 128 * 128;  // [128 rows][64 bf16]
  static constexpr int KTILE = (D / 64) * KATOM;
  static constexpr int QATOM = 64 * 128;   // [64 rows][64 bf16]
  static constexpr int QTILE = (D / 64) * QATOM;
  static constexpr int QST = 3;
  static constexpr int PT_BYTES = 128 * 128;  // P^T or dS^T: [128 keys][64 queries] bf16
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + KTILE;
  static constexpr int Q_OFF = V_OFF + KTILE;
  static constexpr int DO_OFF = Q_OFF + QST * QTILE;
  static constexpr int PT_OFF = DO_OFF + QST * QTILE;
  static constexpr int DS_OFF = PT_OFF + PT_BYTES;
  static constexpr int L_OFF = DS_OFF + PT_BYTES;  // per stage: lse2 [64] | delta [64]
  static constexpr int BAR_OFF = L_OFF + QST * 512;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static_assert(SMEM <= 232448, "smem budget");
  static_assert(2 * KTILE <= 2 * QST * QTILE, "dK / dV staging reuses the Q / dO ring");
};

template <int D>
__global__ void __launch_bounds__(640, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_st,
                         const float* __restrict__ lse2,
                         const float* __restrict__ delta, bf16* __restrict__ dqkv, int T, int H, int BH,
                         float scale) {
  using C = BwdDkdvCfg<D>;
  constexpr int NA = D / 64;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bars = base + C::BAR_OFF;
  const uint32_t kv_full = bars, qd_full0 = bars + 8, qd_empty0 = qd_full0 + 8 * C::QST;
  const uint32_t kv_tmem = qd_empty0 + 8 * C::QST, sp_full = kv_tmem + 8, sp_free = sp_full + 8;
  const uint32_t ds_full = sp_free + 8, ds_free = ds_full + 8, mm_done = ds_free + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + C::BAR_OFF + 240);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 128) ZTRACE(1, 0, 63);
  const int bh = blockIdx.x % BH, b = bh / H, h = bh % H;
  const int kblk = static_cast<int>(blockIdx.x) / BH;  // block 0 has the most query tiles: first
  const int k0 = kblk * 128;
  const int nq = 2 * (T / 128 - kblk);  // 64-query tiles from the diagonal on
  const int row_base = b * T;

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_kv);
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    mbar_init(kv_full, 1);
    for (int s = 0; s < C::QST; ++s) {
      mbar_init(qd_full0 + 8 * s, 1);
      mbar_init(qd_empty0 + 8 * s, 1);
    }
    mbar_init(kv_tmem, 16);  // one arrival per row warp
    mbar_init(sp_full, 1);
    mbar_init(sp_free, 16);
    mbar_init(ds_full, 16);
    mbar_init(ds_free, 1);
    mbar_init(mm_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t T_DV = tmem, T_DK = tmem + D, T_K = tmem + 2 * D, T_V = T_K + D / 2, T_S = tmem + 3 * D,
                 T_DP = T_S + 64;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * C::KTILE);
      for (int a = 0; a < NA; ++a) {
        tma_load_2d(base + C::K_OFF + a * C::KATOM, &tm_kv, kv_full, H * D + h * D + 64 * a, row_base + k0);
        tma_load_2d(base + C::V_OFF + a * C::KATOM, &tm_kv, kv_full, 2 * H * D + h * D + 64 * a, row_base + k0);
      }
      for (int it = 0; it < nq; ++it) {
        const int st = it % C::QST;
        const int q0 = k0 + it * 64;
        mbar_wait(qd_empty0 + 8 * st, ((it / C::QST) & 1) ^ 1);
        const uint32_t fb = qd_full0 + 8 * st;
        mbar_arrive_expect_tx(fb, 2 * C::QTILE + 512);
        for (int a = 0; a < NA; ++a) {
          tma_load_2d(base + C::Q_OFF + st * C::QTILE + a * C::QATOM, &tm_q, fb, h * D + 64 * a, row_base + q0);
          tma_load_2d(base + C::DO_OFF + st * C::QTILE + a * C::QATOM, &tm_do, fb, h * D + 64 * a, row_base + q0);
        }
        if (it == 0) asm volatile("griddepcontrol.wait;" ::: "memory");  // delta / lse2 of the dQ kernel
        bulk_load_1d(base + C::L_OFF + st * 512, lse2 + (long long)bh * T + q0, 256, fb);
        bulk_load_1d(base + C::L_OFF + st * 512 + 256, delta + (long long)bh * T + q0, 256, fb);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {  // whole warp: uniform descriptors, elect.sync issues
      constexpr uint32_t id_sp = make_idesc_bf16(128, 64, false, false);  // S^T, dP^T: N = 64 queries
      constexpr uint32_t id_kv = make_idesc_bf16(128, D, false, true);    // dV, dK: B N-major (N = d)
      auto issue_sp = [&](int it) {  // S^T = K Q^T, dP^T = V dO^T (A = K / V from TMEM)
        const int st = it % C::QST;
        mbar_wait(qd_full0 + 8 * st, (it / C::QST) & 1);
        tc_fence_after();
        const uint32_t qs = base + C::Q_OFF + st * C::QTILE, dos = base + C::DO_OFF + st * C::QTILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16_ts_w(T_S, T_K + kk * 8, make_sdesc(qs + (kk >> 2) * C::QATOM + (kk & 3) * 32, 16, 1024), id_sp,
                        kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16_ts_w(T_DP, T_V + kk * 8, make_sdesc(dos + (kk >> 2) * C::QATOM + (kk & 3) * 32, 16, 1024),
                        id_sp, kk > 0 ? 1u : 0u);
        mma_commit_w(sp_full);
      };
      mbar_wait(kv_tmem, 0);  // K, V copied into TMEM by the row threads
      tc_fence_after();
      issue_sp(0);
      for (int it = 0; it < nq; ++it) {
        const int st = it % C::QST;
        const uint32_t qs = base + C::Q_OFF + st * C::QTILE, dos = base + C::DO_OFF + st * C::QTILE;
        if (it + 1 < nq) {
          mbar_wait(sp_free, it & 1);  // the row threads have loaded S^T(it), dP^T(it)
          tc_fence_after();
          issue_sp(it + 1);
        }
        ZTRACE(1, 0, it);
        mbar_wait(ds_full, it & 1);
        ZTRACE(1, 1, it);
        tc_fence_after();
        const uint32_t acc0 = it > 0 ? 1u : 0u;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // dV += P^T dO: A = P^T (smem K-major), B = dO (N-major)
          mma_bf16_w(T_DV, make_sdesc(base + C::PT_OFF + kk * 32, 16, 1024), make_sdesc(dos + kk * 2048, C::QATOM, 1024),
                     id_kv, (acc0 | kk) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // dK += dS^T Q: A = dS^T (smem K-major), B = Q (N-major)
          mma_bf16_w(T_DK, make_sdesc(base + C::DS_OFF + kk * 32, 16, 1024), make_sdesc(qs + kk * 2048, C::QATOM, 1024),
                     id_kv, (acc0 | kk) ? 1u : 0u);
        mma_commit_w(ds_free);
        mma_commit_w(qd_empty0 + 8 * st);
        ZTRACE(1, 2, it);
      }
      mma_commit_w(mm_done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // 16 row warps (4 per SM sub-partition): warp (quarter q, part) owns key rows 32q..32q+31
    // and queries [16 part, 16 part + 16) of each tile -- enough warps in flight to hide the
    // TMEM-load -> exp2 -> smem-store latency chain (with 8 warps the exp2 phase, not the
    // tensor core, set the pace: ~1000 cycles per tile vs ~1024 of MMA work)
    const int q = warp & 3;
    const int part = (warp - 4) >> 2;
    const int r = q * 32 + lane;  // key row == TMEM lane
    const uint32_t lo = static_cast<uint32_t>(q * 32) << 16;
    const float sl2 = scale * kLog2e;
    {  // K and V rows -> TMEM (this thread: key row r, quarter `part` of the D columns)
      constexpr int CH = D / 32;  // 16-byte chunks per quarter row
      uint32_t kv[4 * CH], vv[4 * CH];
      mbar_wait(kv_full, 0);
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int cg = part * CH + i;
        const uint32_t off = (cg >> 3) * C::KATOM + r * 128 + (((cg & 7) ^ (r & 7)) << 4);
        const uint4 k4 = ld_shared_v4(base + C::K_OFF + off), v4 = ld_shared_v4(base + C::V_OFF + off);
        kv[4 * i] = k4.x, kv[4 * i + 1] = k4.y, kv[4 * i + 2] = k4.z, kv[4 * i + 3] = k4.w;
        vv[4 * i] = v4.x, vv[4 * i + 1] = v4.y, vv[4 * i + 2] = v4.z, vv[4 * i + 3] = v4.w;
      }
      if constexpr (CH == 4) {
        tmem_st16(T_K + lo + part * 16, kv);
        tmem_st16(T_V + lo + part * 16, vv);
      } else {
        tmem_st8(T_K + lo + part * 8, kv);
        tmem_st8(T_V + lo + part * 8, vv);
      }
      tmem_wait_st();
      tc_fence_before();
      warp_arrive(kv_tmem);
    }
    for (int it = 0; it < nq; ++it) {
      const float* L = reinterpret_cast<const float*>(gbase + C::L_OFF + (it % C::QST) * 512) + part * 16;
      if (threadIdx.x == 128) ZTRACE(1, 4, it);
      mbar_wait(sp_full, it & 1);
      if (threadIdx.x == 128) ZTRACE(1, 5, it);
      tc_fence_after();
#ifdef ZPP_TRACE_NOSM  // debug experiment: MMA pipeline alone (row threads only hand over)
      tc_fence_before();
      warp_arrive(sp_free);
      if (it >= 1) mbar_wait(ds_free, (it - 1) & 1);
      warp_arrive(ds_full);
      if (threadIdx.x == 128) ZTRACE(1, 7, it);
      continue;
#endif
      uint32_t sv[16], pv[16];
      tmem_ld16(T_S + lo + part * 16, sv);
      tmem_ld16(T_DP + lo + part * 16, pv);
      tmem_wait_ld();
      tc_fence_before();
      warp_arrive(sp_free);  // S^T(it+1) / dP^T(it+1) may now overwrite the buffers
      float p[16], ds[16];
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float4 l4 = *reinterpret_cast<const float4*>(L + j);
        const float4 d4 = *reinterpret_cast<const float4*>(L + 64 + j);
        const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          p[j + u] = fast_exp2(fmaf(__uint_as_float(sv[j + u]), sl2, -lv[u]));
          ds[j + u] = dv[u] * scale;
        }
      }
      if (it < 2) {  // tiles on the diagonal: key after query
        const int qk = it * 64 + part * 16 - r;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (qk + j < 0) p[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) ds[j] = p[j] * fmaf(__uint_as_float(pv[j]), scale, -ds[j]);
      if (threadIdx.x == 128) ZTRACE(1, 6, it);
      if (it >= 1) mbar_wait(ds_free, (it - 1) & 1);  // dV / dK(it-1) done reading P^T / dS^T
      const uint32_t rp = base + C::PT_OFF + r * 128, rd = base + C::DS_OFF + r * 128;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int c8 = part * 2 + t;
        const float* pp = &p[t * 8];
        const float* sd = &ds[t * 8];
        const uint32_t sw = (c8 ^ (r & 7)) << 4;
        st_shared_v4(rp + sw, pack_bf16(pp[0], pp[1]), pack_bf16(pp[2], pp[3]), pack_bf16(pp[4], pp[5]),
                     pack_bf16(pp[6], pp[7]));
        st_shared_v4(rd + sw, pack_bf16(sd[0], sd[1]), pack_bf16(sd[2], sd[3]), pack_bf16(sd[4], sd[5]),
                     pack_bf16(sd[6], sd[7]));
      }
      fence_proxy_async();
      warp_arrive(ds_full);
      if (threadIdx.x == 128) ZTRACE(1, 7, it);
    }
    mbar_wait(mm_done, 0);
    if (threadIdx.x == 128) ZTRACE(1, 4, 63);
    tc_fence_after();
    // dK, dV -> swizzled smem tiles (the drained Q/dO ring) -> TMA stores
    const uint32_t st_k = base + C::Q_OFF, st_v = st_k + C::KTILE;
    stage_acc<D / 4>(T_DK, lo, r, part * (D / 4), st_k);
    stage_acc<D / 4>(T_DV, lo, r, part * (D / 4), st_v);
    fence_proxy_async();
    named_bar_sync(1, 512);
    if (threadIdx.x == 128) {
      for (int a = 0; a < NA; ++a) {
        tma_store_2d(&tm_st, st_k + a * C::KATOM, H * D + h * D + 64 * a, row_base + k0);
        tma_store_2d(&tm_st, st_v + a * C::KATOM, 2 * H * D + h * D + 64 * a, row_base + k0);
      }
      bulk_commit();
      bulk_wait_all();
    }
    if (threadIdx.x == 128) ZTRACE(1, 5, 63);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

namespace {
int qkv_map(CUtensorMap* m, const void* p, int H, int D, int cols_mult, int rows_total, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols_mult * H * D, (cuuint64_t)rows_total};
  cuuint64_t strides[1] = {(cuuint64_t)cols_mult * H * D * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return encode_tensor_map(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, estr,
                           CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int D>
cudaError_t bwd_attrs() {
  cudaError_t e = cudaFuncSetAttribute(attn_bwd_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       BwdDqCfg<D>::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(attn_bwd_dkdv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             BwdDkdvCfg<D>::SMEM);
  return e;
}
}  // namespace

template <int D>
int attn_bwd_tc_launch(const void* qkv, const void* out, const float* lse, const void* dout, void* dqkv, float* ws,
                       int B, int T, int H, cudaStream_t s) {
  if (T % 128) return set_error(ZPP_ERR_ARG, "attn_bwd: seq must be a multiple of 128");
  const int BT = B * T;
  CUtensorMap m_q128, m_kv64, m_kv128, m_q64, m_do128, m_do64, m_st;
  int rc = qkv_map(&m_q128, qkv, H, D, 3, BT, 128);
  if (!rc) rc = qkv_map(&m_kv64, qkv, H, D, 3, BT, 64);
  if (!rc) rc = qkv_map(&m_kv128, qkv, H, D, 3, BT, 128);
  if (!rc) rc = qkv_map(&m_q64, qkv, H, D, 3, BT, 64);
  if (!rc) rc = qkv_map(&m_do128, dout, H, D, 1, BT, 128);
  if (!rc) rc = qkv_map(&m_do64, dout, H, D, 1, BT, 64);
  if (!rc) rc = qkv_map(&m_st, dqkv, H, D, 3, BT, 128);  // dQ / dK / dV tile stores
  if (rc) return rc;
  static bool set = false;
  if (!set) {
    cudaError_t e = bwd_attrs<D>();
    if (e != cudaSuccess) return set_cuda_error(e, "attn_bwd attr");
    set = true;
  }
  const int BH = B * H;
  float* delta = ws;
  float* lse2 = ws + (long long)BH * T;
  const float scale = 1.f / sqrtf((float)D);
  const dim3 grid((T / 128) * BH);
  attn_bwd_dq_kernel<D><<<grid, 384, BwdDqCfg<D>::SMEM, s>>>(m_q128, m_kv64, m_do128, m_st, (const bf16*)out, lse, delta, lse2,
                                                               (bf16*)dqkv, T, H, BH, scale);
  rc = check_launch("attn_bwd_dq");
  if (rc) return rc;
  // dK/dV launched as a programmatic dependent of the dQ kernel: its prologue (TMEM, barriers,
  // K/V/Q/dO loads) runs on SMs the dQ tail leaves idle; only the lse2 / delta loads wait
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(640);
  cfg.dynamicSmemBytes = BwdDkdvCfg<D>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, attn_bwd_dkdv_kernel<D>, m_kv128, m_q64, m_do64, m_st, (const float*)lse2,
                                     (const float*)delta, (bf16*)dqkv, T, H, BH, scale);
  if (e != cudaSuccess) return set_cuda_error(e, "attn_bwd_dkdv launch");
  return check_launch("attn_bwd_dkdv");
}

template int attn_bwd_tc_launch<64>(const void*, const void*, const float*, const void*, void*, float*, int, int,
                                    int, cudaStream_t);
template int attn_bwd_tc_launch<128>(const void*, const void*, const float*, const void*, void*, float*, int, int,
                                     int, cudaStream_t);

int attention_bwd_tc_preload() {
  cudaError_t e = bwd_attrs<64>();
  if (e == cudaSuccess) e = bwd_attrs<128>();
  return e == cudaSuccess ? ZPP_OK : set_cuda_error(e, "attention_bwd_tc preload");
}

}  // namespace zpp

#ifdef ZPP_TRACE
extern "C" int zpp_debug_attn_trace(void* host_out) {
  cudaError_t e = cudaMemcpyFromSymbol(host_out, zpp::g_attn_trace, sizeof(zpp::g_attn_trace));
  return e == cudaSuccess ? 0 : zpp::set_cuda_error(e, "trace");
}
#endif
