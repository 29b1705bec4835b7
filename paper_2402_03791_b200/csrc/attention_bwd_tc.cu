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

// Persistent-kernel item order: items are sorted heaviest first; CTA c takes item
// k*G + c in even rounds and k*G + (G-1-c) in odd rounds (boustrophedon), which balances the
// per-CTA sums to ~98% of ideal where plain round-robin (k*G + c) reached 88%.
__device__ __forceinline__ int snake_item(int k, int G, int c) { return k * G + ((k & 1) ? G - 1 - c : c); }

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
// dQ (+ delta, lse2), persistent: one CTA per SM walks the (128-query block, head) items
// heaviest first (item = blockIdx.x + k * gridDim.x); the next item's Q / dO are prefetched as
// soon as the current ones sit in TMEM, and the dQ epilogue runs on its own warps beside the
// next item's tiles.  warp 0: TMA Q, dO per item + K_j ring of 4 (K_j feeds S_j and dQ_j);
// warp 3: V_j ring of 3; warp 1: MMA issuer; warp 2: TMEM owner; warps 4..11: row warps,
// thread = query row (TMEM lane), warp (quarter q, half hh) takes keys [32hh, 32hh+32) of each
// 64-key tile; warps 12..15: epilogue (dQ TMEM -> swizzled smem -> TMA store).
// TMEM: S/dS [0,128) (2 x 64), dP [128,256) (2 x 64), dQ [256,256+D), Q, dO (A operands of S
// and dP as TS-mode MMAs: an SS MMA with N = 64 is bound by re-reading its 128-row A from smem).
template <int D>
struct BwdDqCfg {
  static constexpr int QATOM = 128 * 128;  // [128 rows][64 bf16]
  static constexpr int QTILE = (D / 64) * QATOM;
  static constexpr int KATOM = 64 * 128;   // [64 rows][64 bf16]
  static constexpr int KTILE = (D / 64) * KATOM;
  static constexpr int KST = 5, VST = 3;
  static constexpr int Q_OFF = 0;
  static constexpr int DO_OFF = Q_OFF + QTILE;
  static constexpr int K_OFF = DO_OFF + QTILE;
  static constexpr int V_OFF = K_OFF + KST * KTILE;
  static constexpr int STG_OFF = V_OFF + VST * KTILE;  // dQ epilogue staging: one [128][64] atom
  static constexpr int RED_OFF = STG_OFF + QATOM;      // float [2][128] delta halves
  static constexpr int BAR_OFF = RED_OFF + 1024;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static constexpr int THREADS = 512;
  static_assert(SMEM <= 232448, "smem budget");
};

template <int D>
__global__ void __launch_bounds__(512, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                       const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_st,
                       const bf16* __restrict__ out, const float* __restrict__ lse, float* __restrict__ delta_out,
                       float* __restrict__ lse2_out, int T, int H, int BH, float scale) {
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
  const uint32_t dq_done = ds_full0 + 16, qt_full = dq_done + 8, qd_empty = qt_full + 8, dq_free = qd_empty + 8;
  static_assert(8 * (1 + 2 * C::KST + 2 * C::VST + 10) <= 240, "barrier area");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + C::BAR_OFF + 240);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 128) ZTRACE(0, 0, 63);
  // programmatic dependent launch: once every dQ CTA is resident, dK/dV CTAs may take the SMs
  // the dQ tail frees (they wait for our delta / lse2 with griddepcontrol.wait)
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int nqb = T / 128;
  const int nitems = nqb * BH;
  auto decode = [&](int w, int& bh, int& q0, int& nkt) {  // heaviest query blocks first, all heads
    bh = w % BH;
    const int qblk = nqb - 1 - w / BH;
    q0 = qblk * 128;
    nkt = 2 * (qblk + 1);  // 64-key tiles up to the diagonal
  };

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_kv);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_st);
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
    mbar_init(qd_empty, 8);
    mbar_init(dq_free, 4);  // one arrival per epilogue warp
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t T_S = tmem, T_DP = tmem + 128, T_DQ = tmem + 256, T_Q = T_DQ + D, T_DO = T_Q + D / 2;
  if (threadIdx.x == 128) ZTRACE(0, 1, 63);

  if (warp == 0) {
    if (lane == 0) {
      int g = 0;
      for (int k = 0, jn = 0; k * (int)gridDim.x < nitems; ++k) {
        const int w = snake_item(k, gridDim.x, blockIdx.x);
        if (w >= nitems) continue;
        const int j = jn++;  // this CTA's local item index
        int bh, q0, nkt;
        decode(w, bh, q0, nkt);
        const int h = bh % H, row_base = (bh / H) * T;
        if (j >= 1) mbar_wait(qd_empty, (j - 1) & 1);  // Q / dO of item j-1 are in TMEM
        mbar_arrive_expect_tx(qd_full, 2 * C::QTILE);
        for (int a = 0; a < NA; ++a) {
          tma_load_2d(base + C::Q_OFF + a * C::QATOM, &tm_q, qd_full, h * D + 64 * a, row_base + q0);
          tma_load_2d(base + C::DO_OFF + a * C::QATOM, &tm_do, qd_full, h * D + 64 * a, row_base + q0);
        }
        for (int jt = 0; jt < nkt; ++jt, ++g) {
          const int st = g % C::KST;
          mbar_wait(k_empty0 + 8 * st, ((g / C::KST) & 1) ^ 1);
          const uint32_t fb = k_full0 + 8 * st;
          mbar_arrive_expect_tx(fb, C::KTILE);
          for (int a = 0; a < NA; ++a)
            tma_load_2d(base + C::K_OFF + st * C::KTILE + a * C::KATOM, &tm_kv, fb, H * D + h * D + 64 * a,
                        row_base + jt * 64);
        }
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (lane == 0) {
      int g = 0;
      for (int k = 0, jn = 0; k * (int)gridDim.x < nitems; ++k) {
        const int w = snake_item(k, gridDim.x, blockIdx.x);
        if (w >= nitems) continue;
        const int j = jn++;  // this CTA's local item index
        int bh, q0, nkt;
        decode(w, bh, q0, nkt);
        const int h = bh % H, row_base = (bh / H) * T;
        for (int jt = 0; jt < nkt; ++jt, ++g) {
          const int st = g % C::VST;
          mbar_wait(v_empty0 + 8 * st, ((g / C::VST) & 1) ^ 1);
          const uint32_t fb = v_full0 + 8 * st;
          mbar_arrive_expect_tx(fb, C::KTILE);
          for (int a = 0; a < NA; ++a)
            tma_load_2d(base + C::V_OFF + st * C::KTILE + a * C::KATOM, &tm_kv, fb, 2 * H * D + h * D + 64 * a,
                        row_base + jt * 64);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {  // whole warp: uniform descriptors, elect.sync issues
      constexpr uint32_t id_s = make_idesc_bf16(128, 64, false, false);  // S, dP: N = 64 keys
      constexpr uint32_t id_q = make_idesc_bf16(128, D, false, true);    // dQ: B = K_j N-major (N = d)
      auto issue_s = [&](int g) {
        const int st = g % C::KST;
        mbar_wait(k_full0 + 8 * st, (g / C::KST) & 1);
        tc_fence_after();
        const uint32_t kb = base + C::K_OFF + st * C::KTILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16_ts_w(T_S + (g & 1) * 64, T_Q + kk * 8,
                        make_sdesc(kb + (kk >> 2) * C::KATOM + (kk & 3) * 32, 16, 1024), id_s, kk > 0 ? 1u : 0u);
        mma_commit_w(s_full0 + 8 * (g & 1));
      };
      auto issue_dp = [&](int g) {
        const int st = g % C::VST;
        mbar_wait(v_full0 + 8 * st, (g / C::VST) & 1);
        tc_fence_after();
        const uint32_t vb = base + C::V_OFF + st * C::KTILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16_ts_w(T_DP + (g & 1) * 64, T_DO + kk * 8,
                        make_sdesc(vb + (kk >> 2) * C::KATOM + (kk & 3) * 32, 16, 1024), id_s, kk > 0 ? 1u : 0u);
        mma_commit_w(dp_full0 + 8 * (g & 1));
        mma_commit_w(v_empty0 + 8 * st);
      };
      int g = 0;
      for (int k = 0, jn = 0; k * (int)gridDim.x < nitems; ++k) {
        const int w = snake_item(k, gridDim.x, blockIdx.x);
        if (w >= nitems) continue;
        const int j = jn++;  // this CTA's local item index
        int bh, q0, nkt;
        decode(w, bh, q0, nkt);
        mbar_wait(qt_full, j & 1);  // Q, dO of item j copied into TMEM by the row warps
        tc_fence_after();
        issue_s(g);
        issue_dp(g);
        if (nkt > 1) {
          issue_s(g + 1);
          issue_dp(g + 1);
        }
        for (int jt = 0; jt < nkt; ++jt, ++g) {
          if (j < 8) ZTRACE(0, 0, jt);
          mbar_wait(ds_full0 + 8 * (g & 1), (g >> 1) & 1);
          if (j < 8) ZTRACE(0, 1, jt);
          tc_fence_after();
          if (jt == 0 && j > 0) {
            mbar_wait(dq_free, (j - 1) & 1);  // the epilogue warps have read dQ of item j-1
            tc_fence_after();
          }
          const uint32_t kb = base + C::K_OFF + (g % C::KST) * C::KTILE;
          // dQ += dS K_j: A = dS in TMEM (each 32-key half packed into its first 16 columns)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_bf16_ts_w(T_DQ, T_S + (g & 1) * 64 + (kk >> 1) * 32 + (kk & 1) * 8,
                          make_sdesc(kb + kk * 2048, C::KATOM, 1024), id_q, (jt > 0 || kk > 0) ? 1u : 0u);
          mma_commit_w(k_empty0 + 8 * (g % C::KST));
          if (jt + 2 < nkt) {  // buffers (g & 1): dS_g read by the dQ MMA above (in-order pipe)
            issue_s(g + 2);
            if (j < 8) ZTRACE(0, 2, jt);
            issue_dp(g + 2);
          }
          if (j < 8) ZTRACE(0, 3, jt);
        }
        mma_commit_w(dq_done);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 12) {
    const int q = warp & 3;
    const int hh = (warp - 4) >> 2;
    const int r = q * 32 + lane;  // query row == TMEM lane
    const uint32_t lo = static_cast<uint32_t>(q * 32) << 16;
    const float sl2 = scale * kLog2e;
    constexpr int CH = D / 16;  // 16-byte chunks per half row
    int g = 0;
    for (int k = 0, jn = 0; k * (int)gridDim.x < nitems; ++k) {
        const int w = snake_item(k, gridDim.x, blockIdx.x);
        if (w >= nitems) continue;
        const int j = jn++;  // this CTA's local item index
      int bh, q0, nkt;
      decode(w, bh, q0, nkt);
      const int h = bh % H, row_base = (bh / H) * T;
      const float lse2_r = lse[(long long)bh * T + q0 + r] * kLog2e;
      // delta = rowsum(O * dO): this thread sums half hh of the row's D columns (O from global,
      // read once here; dO from the swizzled smem tile)
      uint4 ov[CH];
      const uint4* orow =
          reinterpret_cast<const uint4*>(out + ((long long)row_base + q0 + r) * H * D + h * D) + hh * CH;
#pragma unroll
      for (int i = 0; i < CH; ++i) ov[i] = __ldg(orow + i);
      mbar_wait(qd_full, j & 1);
      if (threadIdx.x == 128 && j == 0) ZTRACE(0, 2, 63);
      float acc = 0.f;
      {
        // this thread's half row of Q and dO -> TMEM (lane r, packed bf16 pairs), and delta.
        // TMEM Q / dO are free: the S / dP MMAs of item j-1 completed before its last tile's
        // s_full / dp_full, which this warp has consumed.
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
        warp_arrive(qd_empty);  // Q / dO smem may take the next item's tiles
      }
      red[hh * 128 + r] = acc;
      named_bar_sync(1, 256);
      const float delta_r = red[r] + red[128 + r];
      named_bar_sync(1, 256);  // red is rewritten by the next item
      if (hh == 0) {
        delta_out[(long long)bh * T + q0 + r] = delta_r;
        lse2_out[(long long)bh * T + q0 + r] = lse2_r;
      }
      for (int jt = 0; jt < nkt; ++jt, ++g) {
        const int buf = g & 1;
        const uint32_t par = (g >> 1) & 1;
        const uint32_t ts = T_S + lo + buf * 64 + hh * 32;
#ifdef ZPP_TRACE_NOSM  // debug experiment: MMA pipeline alone (row warps only hand over)
        mbar_wait(s_full0 + 8 * buf, par);
        mbar_wait(dp_full0 + 8 * buf, par);
        tc_fence_before();
        warp_arrive(ds_full0 + 8 * buf);
        continue;
#endif
        if (threadIdx.x == 128 && j < 8) ZTRACE(0, 4, jt);
        mbar_wait(s_full0 + 8 * buf, par);
        if (threadIdx.x == 128 && j < 8) ZTRACE(0, 5, jt);
        tc_fence_after();
        float p[32];
        {
          uint32_t v[32];
          tmem_ld32(ts, v);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) p[k] = fast_exp2(fmaf(__uint_as_float(v[k]), sl2, -lse2_r));
        }
        if (jt >= nkt - 2) {  // the two tiles that straddle the diagonal: keys after the query
          const int kq = jt * 64 + hh * 32 - q0 - r;
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (kq + k > 0) p[k] = 0.f;
        }
        if (threadIdx.x == 128 && j < 8) ZTRACE(0, 6, jt);
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
        if (threadIdx.x == 128 && j < 8) ZTRACE(0, 7, jt);
      }
    }
  } else if (warp >= 12) {
    // epilogue warps: thread = TMEM lane (query row) r of quarter q, all D columns
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lo = static_cast<uint32_t>(q * 32) << 16;
    for (int k = 0, jn = 0; k * (int)gridDim.x < nitems; ++k) {
        const int w = snake_item(k, gridDim.x, blockIdx.x);
        if (w >= nitems) continue;
        const int j = jn++;  // this CTA's local item index
      int bh, q0, nkt;
      decode(w, bh, q0, nkt);
      const int h = bh % H, row_base = (bh / H) * T;
      mbar_wait(dq_done, j & 1);
      tc_fence_after();
#pragma unroll 1
      for (int a = 0; a < NA; ++a) {  // one 64-column atom at a time through a 16 KB staging tile
        named_bar_sync(2, 128);       // the previous TMA store has left the staging tile
        stage_acc<32>(T_DQ, lo, r, 64 * a, base + C::STG_OFF - 64 * a * 256);
        stage_acc<32>(T_DQ, lo, r, 64 * a + 32, base + C::STG_OFF - 64 * a * 256);
        if (a == NA - 1) {
          tc_fence_before();
          warp_arrive(dq_free);  // dQ read: the next item may accumulate into it
        }
        fence_proxy_async();
        named_bar_sync(2, 128);
        if (threadIdx.x == 384) {
          tma_store_2d(&tm_st, base + C::STG_OFF, h * D + 64 * a, row_base + q0);
          bulk_commit();
          bulk_wait_all();
        }
      }
      if (threadIdx.x == 384 && j == 0) ZTRACE(0, 5, 63);
      if (threadIdx.x == 384 && j == 0) ZTRACE(0, 4, 63);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------------------
// dK / dV, persistent: one CTA per SM walks the (128-key block, head) items heaviest first
// (item = blockIdx.x + k * gridDim.x), so the next item's K / V load, their copy into TMEM and
// its first S^T / dP^T MMAs overlap the previous item's last tiles and its dK / dV epilogue
// (a CTA per item paid ~6k cycles of prologue + ~3k of epilogue on ~25k of tiles).
// warp 0: TMA (K, V per item; Q_t / dO_t + lse2_t / delta_t through a ring of 3, continuing
// across items); warp 1: MMA issuer; warp 2: TMEM owner; warps 4..19: row warps, thread = key
// row (TMEM lane), warp (quarter q, part) takes queries [16 part, 16 part + 16) of each
// 64-query tile; warps 20..23: epilogue (dK / dV TMEM -> swizzled smem -> TMA store).
// K and V live in TMEM (A operands of S^T / dP^T: TS-mode MMAs run at the tensor core's rate
// for N = 64; the SS form re-reads the 128-row A from smem).  S^T / dP^T are single-buffered
// but released as soon as the row warps have loaded them; P^T and dS^T go to smem (A operands
// of dV += P^T dO and dK += dS^T Q, N = d: full rate from smem).  The K / V smem tiles double
// as the epilogue staging area once K / V of the next item sit in TMEM.
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
  static constexpr int THREADS = 768;
  static_assert(SMEM <= 232448, "smem budget");
};

template <int D>
__global__ void __launch_bounds__(768, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_st,
                         const float* __restrict__ lse2, const float* __restrict__ delta, int T, int H, int BH,
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
  const uint32_t acc_free = mm_done + 8, kv_empty = acc_free + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + C::BAR_OFF + 240);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nitems = (T / 128) * BH;
  if (threadIdx.x == 128) ZTRACE(1, 0, 63);
  // item w -> (key block, head); item 0.. have the most query tiles
  auto decode = [&](int w, int& bh, int& k0, int& nq) {
    bh = w % BH;
    const int kblk = w / BH;
    k0 = kblk * 128;
    nq = 2 * (T / 128 - kblk);
  };

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_kv);
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_st);
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
    mbar_init(acc_free, 4);  // one arrival per epilogue warp
    mbar_init(kv_empty, 1);
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
      int g = 0;  // running tile index of this CTA (ring stage / parity)
      for (int k = 0, jn = 0; k * (int)gridDim.x < nitems; ++k) {
        const int w = snake_item(k, gridDim.x, blockIdx.x);
        if (w >= nitems) continue;
        const int j = jn++;  // this CTA's local item index
        int bh, k0, nq;
        decode(w, bh, k0, nq);
        const int b = bh / H, h = bh % H, row_base = b * T;
        // K / V smem is free once K / V(j-1) sit in TMEM (j == 1) and, from j == 2 on, once the
        // epilogue of item j-2 (staged in the same smem) has been stored
        if (j == 1) mbar_wait(kv_tmem, 0);
        if (j >= 2) mbar_wait(kv_empty, (j - 2) & 1);
        mbar_arrive_expect_tx(kv_full, 2 * C::KTILE);
        for (int a = 0; a < NA; ++a) {
          tma_load_2d(base + C::K_OFF + a * C::KATOM, &tm_kv, kv_full, H * D + h * D + 64 * a, row_base + k0);
          tma_load_2d(base + C::V_OFF + a * C::KATOM, &tm_kv, kv_full, 2 * H * D + h * D + 64 * a, row_base + k0);
        }
        for (int it = 0; it < nq; ++it, ++g) {
          const int st = g % C::QST;
          const int q0 = k0 + it * 64;
          mbar_wait(qd_empty0 + 8 * st, ((g / C::QST) & 1) ^ 1);
          const uint32_t fb = qd_full0 + 8 * st;
          mbar_arrive_expect_tx(fb, 2 * C::QTILE + 512);
          for (int a = 0; a < NA; ++a) {
            tma_load_2d(base + C::Q_OFF + st * C::QTILE + a * C::QATOM, &tm_q, fb, h * D + 64 * a, row_base + q0);
            tma_load_2d(base + C::DO_OFF + st * C::QTILE + a * C::QATOM, &tm_do, fb, h * D + 64 * a,
                        row_base + q0);
          }
          if (g == 0) asm volatile("griddepcontrol.wait;" ::: "memory");  // delta / lse2 of the dQ kernel
          bulk_load_1d(base + C::L_OFF + st * 512, lse2 + (long long)bh * T + q0, 256, fb);
          bulk_load_1d(base + C::L_OFF + st * 512 + 256, delta + (long long)bh * T + q0, 256, fb);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {  // whole warp: uniform descriptors, elect.sync issues
      constexpr uint32_t id_sp = make_idesc_bf16(128, 64, false, false);  // S^T, dP^T: N = 64 queries
      constexpr uint32_t id_kv = make_idesc_bf16(128, D, false, true);    // dV, dK: B N-major (N = d)
      auto issue_sp = [&](int g) {  // S^T = K Q^T, dP^T = V dO^T of running tile g (A = K / V from TMEM)
        const int st = g % C::QST;
        mbar_wait(qd_full0 + 8 * st, (g / C::QST) & 1);
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
      int g = 0;
      for (int k = 0, jn = 0; k * (int)gridDim.x < nitems; ++k) {
        const int w = snake_item(k, gridDim.x, blockIdx.x);
        if (w >= nitems) continue;
        const int j = jn++;  // this CTA's local item index
        int bh, k0, nq;
        decode(w, bh, k0, nq);
        mbar_wait(kv_tmem, j & 1);  // K, V(j) copied into TMEM; S^T / dP^T of item j-1 loaded
        tc_fence_after();
        issue_sp(g);
        for (int it = 0; it < nq; ++it, ++g) {
          const int st = g % C::QST;
          const uint32_t qs = base + C::Q_OFF + st * C::QTILE, dos = base + C::DO_OFF + st * C::QTILE;
          if (it + 1 < nq) {
            mbar_wait(sp_free, g & 1);  // the row warps have loaded S^T(g), dP^T(g)
            tc_fence_after();
            issue_sp(g + 1);
          }
          if (j < 8) ZTRACE(1, 0, it);
          mbar_wait(ds_full, g & 1);
          if (j < 8) ZTRACE(1, 1, it);
          tc_fence_after();
          if (it == 0 && j > 0) {
            mbar_wait(acc_free, (j - 1) & 1);  // the epilogue has read dK / dV of item j-1
            tc_fence_after();
          }
          const uint32_t acc0 = it > 0 ? 1u : 0u;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // dV += P^T dO: A = P^T (smem K-major), B = dO (N-major)
            mma_bf16_w(T_DV, make_sdesc(base + C::PT_OFF + kk * 32, 16, 1024),
                       make_sdesc(dos + kk * 2048, C::QATOM, 1024), id_kv, (acc0 | kk) ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // dK += dS^T Q: A = dS^T (smem K-major), B = Q (N-major)
            mma_bf16_w(T_DK, make_sdesc(base + C::DS_OFF + kk * 32, 16, 1024),
                       make_sdesc(qs + kk * 2048, C::QATOM, 1024), id_kv, (acc0 | kk) ? 1u : 0u);
          mma_commit_w(ds_free);
          mma_commit_w(qd_empty0 + 8 * st);
          if (j < 8) ZTRACE(1, 2, it);
        }
        mma_commit_w(mm_done);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 20) {
    const int q = warp & 3;
    const int part = (warp - 4) >> 2;
    const int r = q * 32 + lane;  // key row == TMEM lane
    const uint32_t lo = static_cast<uint32_t>(q * 32) << 16;
    const float sl2 = scale * kLog2e;
    int g = 0;
    for (int k = 0, jn = 0; k * (int)gridDim.x < nitems; ++k) {
        const int w = snake_item(k, gridDim.x, blockIdx.x);
        if (w >= nitems) continue;
        const int j = jn++;  // this CTA's local item index
      int bh, k0, nq;
      decode(w, bh, k0, nq);
      {  // K and V rows of item j -> TMEM (key row r, quarter `part` of the D columns)
        constexpr int CH = D / 32;  // 16-byte chunks per quarter row
        uint32_t kv[4 * CH], vv[4 * CH];
        mbar_wait(kv_full, j & 1);
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
      for (int it = 0; it < nq; ++it, ++g) {
        const float* L = reinterpret_cast<const float*>(gbase + C::L_OFF + (g % C::QST) * 512) + part * 16;
        if (threadIdx.x == 128 && j < 8) ZTRACE(1, 4, it);
        mbar_wait(sp_full, g & 1);
        if (threadIdx.x == 128 && j < 8) ZTRACE(1, 5, it);
        tc_fence_after();
#ifdef ZPP_TRACE_NOSM  // debug experiment: MMA pipeline alone (row warps only hand over)
        tc_fence_before();
        warp_arrive(sp_free);
        if (g >= 1) mbar_wait(ds_free, (g - 1) & 1);
        warp_arrive(ds_full);
        continue;
#endif
        uint32_t sv[16], pv[16];
        tmem_ld16(T_S + lo + part * 16, sv);
        tmem_ld16(T_DP + lo + part * 16, pv);
        tmem_wait_ld();
        tc_fence_before();
        warp_arrive(sp_free);  // S^T / dP^T of the next tile may now overwrite the buffers
        float p[16], ds[16];
#pragma unroll
        for (int jj = 0; jj < 16; jj += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(L + jj);
          const float4 d4 = *reinterpret_cast<const float4*>(L + 64 + jj);
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            p[jj + u] = fast_exp2(fmaf(__uint_as_float(sv[jj + u]), sl2, -lv[u]));
            ds[jj + u] = dv[u] * scale;
          }
        }
        if (it < 2) {  // tiles on the diagonal: key after query
          const int qk = it * 64 + part * 16 - r;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            if (qk + jj < 0) p[jj] = 0.f;
        }
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) ds[jj] = p[jj] * fmaf(__uint_as_float(pv[jj]), scale, -ds[jj]);
        if (threadIdx.x == 128 && j < 8) ZTRACE(1, 6, it);
        if (g >= 1) mbar_wait(ds_free, (g - 1) & 1);  // dV / dK of the previous tile done reading P^T / dS^T
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
        if (threadIdx.x == 128 && j < 8) ZTRACE(1, 7, it);
      }
    }
  } else if (warp >= 20) {
    // epilogue warps: thread = TMEM lane (key row) r of quarter q, all D columns
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lo = static_cast<uint32_t>(q * 32) << 16;
    for (int k = 0, jn = 0; k * (int)gridDim.x < nitems; ++k) {
        const int w = snake_item(k, gridDim.x, blockIdx.x);
        if (w >= nitems) continue;
        const int j = jn++;  // this CTA's local item index
      int bh, k0, nq;
      decode(w, bh, k0, nq);
      const int b = bh / H, h = bh % H, row_base = b * T;
      bool more = false;  // does this CTA take another item after this one?
      for (int k2 = k + 1; k2 * (int)gridDim.x < nitems && !more; ++k2)
        more = snake_item(k2, gridDim.x, blockIdx.x) < nitems;
      mbar_wait(mm_done, j & 1);
      // the staging area is the K / V smem: wait until K / V of the next item are in TMEM
      if (more) mbar_wait(kv_tmem, (j + 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < D; c += 32) {
        stage_acc<32>(T_DK, lo, r, c, base + C::K_OFF);
        stage_acc<32>(T_DV, lo, r, c, base + C::V_OFF);
      }
      tc_fence_before();
      warp_arrive(acc_free);  // dK / dV read: the MMA warp may start the next item's accumulation
      fence_proxy_async();
      named_bar_sync(2, 128);
      if (threadIdx.x == 640) {
        for (int a = 0; a < NA; ++a) {
          tma_store_2d(&tm_st, base + C::K_OFF + a * C::KATOM, H * D + h * D + 64 * a, row_base + k0);
          tma_store_2d(&tm_st, base + C::V_OFF + a * C::KATOM, 2 * H * D + h * D + 64 * a, row_base + k0);
        }
        bulk_commit();
        bulk_wait_all();
        mbar_arrive(kv_empty);  // staging smem free: the producer may load K / V of item j+2
        if (j == 0) ZTRACE(1, 5, 63);
      }
      if (threadIdx.x == 640 && j == 0) ZTRACE(1, 4, 63);
    }
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
  const int items = (T / 128) * BH;
  const dim3 pgrid(items < num_sms() ? items : num_sms());  // persistent kernels: one CTA per SM
  attn_bwd_dq_kernel<D><<<pgrid, BwdDqCfg<D>::THREADS, BwdDqCfg<D>::SMEM, s>>>(m_q128, m_kv64, m_do128, m_st,
                                                                             (const bf16*)out, lse, delta, lse2, T, H,
                                                                             BH, scale);
  rc = check_launch("attn_bwd_dq");
  if (rc) return rc;
  // dK/dV launched as a programmatic dependent of the dQ kernel: its prologue (TMEM, barriers,
  // K/V/Q/dO loads) runs on SMs the dQ tail leaves idle; only the lse2 / delta loads wait
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = pgrid;
  cfg.blockDim = dim3(BwdDkdvCfg<D>::THREADS);
  cfg.dynamicSmemBytes = BwdDkdvCfg<D>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, attn_bwd_dkdv_kernel<D>, m_kv128, m_q64, m_do64, m_st, (const float*)lse2,
                                     (const float*)delta, T, H, BH, scale);
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
