// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M,N] (op)= sum_k A(m,k) * B(n,k)        bf16 operands, fp32 accumulation in TMEM
//
// A is K-major (A[m*lda+k]) or M-major (A[k*lda+m]); B is K-major (B[n*ldb+k]) or
// N-major (B[k*ldb+n]).  This covers the three GEMMs of a transformer linear
// (SURVEY.md section 2 kernel table) without any transpose pass:
//   fwd    Y  = X  W^T   A=X  (K-major)  B=W (K-major)
//   dgrad  dX = dY W     A=dY (K-major)  B=W (N-major)
//   wgrad  dW += dY^T X  A=dY (M-major)  B=X (N-major), fp32 TMA reduce-add epilogue
//
// CG = 1: one CTA computes a 128 x BN tile with tcgen05.mma.cta_group::1.
// CG = 2: a CTA pair (cluster of 2 on one TPC) computes a 256 x BN tile with
//         tcgen05.mma.cta_group::2: each CTA TMA-loads its 128 rows of A and half of
//         B; the leader issues the MMA and multicast-commits to both CTAs; each CTA
//         owns the TMEM accumulator of its 128 rows.  Per-SM operand traffic drops
//         from (128+BN)*64*2 to (128+BN/2)*64*2 bytes per k-block.
//
// Warp roles (256 threads, 1 CTA/SM, persistent over output tiles):
//   warp 0     TMA producer (one lane): A/B tiles -> smem ring (128B swizzle)
//   warp 1     MMA issuer (one lane, leader CTA only)
//   warp 2     TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4-7  epilogue: tcgen05.ld -> bias/GeLU/dGeLU/residual/cast -> swizzled
//              per-warp smem staging -> TMA store (bf16/fp32) or TMA reduce-add
//              (fp32 +=, so the gradient accumulation never round-trips the SM).
//
// Hybrid data-parallel + stream-K work list (wave quantisation): with U persistent units
// and T tiles, the floor(T/U)*U "full-wave" tiles are whole work items; the T mod U
// remainder tiles are split into p k-ranges ("pieces") so the last wave is p times
// finer.  A piece that finds the other p-1 already arrived (per-(tile, warp) counter)
// finalises the tile; otherwise it parks its fp32 partial in a per-stream workspace and
// bumps the counter -- and if that bump was the last, it finalises after all.  Nobody
// waits, and the finaliser sums the pieces in piece order (deterministic).  E.g. M=2048 x N=4096 at 74 SM pairs: 128 tiles = 1.73 waves
// -> 74 whole tiles + 54 tiles x 4 pieces = 1.75 tile-times instead of 2.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "ptx.cuh"
#include "zpp_internal.h"

namespace zpp {

constexpr int GEMM_BM = 128;  // rows per CTA
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 256;
constexpr int EPI_BUF = 4096;  // per-warp staging buffer: 32 rows x 128 B

struct EpiParams {
  const __nv_bfloat16* bias;
  const __nv_bfloat16* resid;
  long long ldr;
  __nv_bfloat16* aux;
  long long ldaux;
  int mode;
  int M, N;
};

// Stream-K split of the work list (see header).  No split: dp_tiles = tiles, pieces = 1.
struct SkParams {
  int dp_tiles;
  int pieces;
  float* ws;        // [(sk_tile * pieces + piece)][BN/32][TILE_M/32][8][32 lanes] float4 partials
  unsigned* flags;  // [sk_tile][CG][4 epilogue warps] arrival counters, re-armed by the finisher
  unsigned long long* trace;  // debug build (ZPP_TRACE): [cta][GEMM_TRACE_ITEMS][6] globaltimer stamps, or null
};
constexpr int GEMM_TRACE_ITEMS = 32;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int BN, int CG>
struct GemmCfg {
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr int B_BYTES = (BN / CG) * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_BYTES = 4 * 2 * EPI_BUF;  // 4 epilogue warps x 2 buffers
  static constexpr int STAGES = (224 * 1024 - EPI_BYTES) / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 512 /*barriers, tile ring*/;
  static_assert(SMEM <= 232448, "shared memory budget");
};

// Epilogue math for 32 consecutive columns of one row (values in x, in place).
__device__ __forceinline__ void epi_math(const EpiParams& p, int row, int col, float (&x)[32]) {
  const int mode = p.mode & 0xF;
  const bool full = (col + 32 <= p.N);
  if (p.bias) {
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 b = *reinterpret_cast<const uint4*>(p.bias + col + j);
        x[j] += bf16lo(b.x); x[j + 1] += bf16hi(b.x); x[j + 2] += bf16lo(b.y); x[j + 3] += bf16hi(b.y);
        x[j + 4] += bf16lo(b.z); x[j + 5] += bf16hi(b.z); x[j + 6] += bf16lo(b.w); x[j + 7] += bf16hi(b.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col + j < p.N) x[j] += __bfloat162float(p.bias[col + j]);
    }
  }
  if (mode == ZPP_EPI_BF16_GELU) {
    if (p.aux && row < p.M) {
      __nv_bfloat16* a = p.aux + (long long)row * p.ldaux + col;
      if (full) {
#pragma unroll
        for (int j = 0; j < 32; j += 8)
          *reinterpret_cast<uint4*>(a + j) = make_uint4(pack_bf16(x[j], x[j + 1]), pack_bf16(x[j + 2], x[j + 3]),
                                                        pack_bf16(x[j + 4], x[j + 5]), pack_bf16(x[j + 6], x[j + 7]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col + j < p.N) a[j] = __float2bfloat16(x[j]);
      }
    }
    // GeLU of the bf16-rounded pre-activation, matching what backward will see
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = gelu_f(__bfloat162float(__float2bfloat16(x[j])));
  } else if (mode == ZPP_EPI_BF16_DGELU && row < p.M) {
    const __nv_bfloat16* a = p.aux + (long long)row * p.ldaux + col;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 u = *reinterpret_cast<const uint4*>(a + j);
        x[j] *= gelu_grad_f(bf16lo(u.x)); x[j + 1] *= gelu_grad_f(bf16hi(u.x));
        x[j + 2] *= gelu_grad_f(bf16lo(u.y)); x[j + 3] *= gelu_grad_f(bf16hi(u.y));
        x[j + 4] *= gelu_grad_f(bf16lo(u.z)); x[j + 5] *= gelu_grad_f(bf16hi(u.z));
        x[j + 6] *= gelu_grad_f(bf16lo(u.w)); x[j + 7] *= gelu_grad_f(bf16hi(u.w));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col + j < p.N) x[j] *= gelu_grad_f(__bfloat162float(a[j]));
    }
  }
  if (p.resid && row < p.M) {
    const __nv_bfloat16* r = p.resid + (long long)row * p.ldr + col;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 b = *reinterpret_cast<const uint4*>(r + j);
        x[j] += bf16lo(b.x); x[j + 1] += bf16hi(b.x); x[j + 2] += bf16lo(b.y); x[j + 3] += bf16hi(b.y);
        x[j + 4] += bf16lo(b.z); x[j + 5] += bf16hi(b.z); x[j + 6] += bf16lo(b.w); x[j + 7] += bf16hi(b.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col + j < p.N) x[j] += __bfloat162float(r[j]);
    }
  }
}

// Tile raster: consecutive tiles (processed concurrently by neighbouring SMs) share the
// operand panel of the LARGER operand, so it streams through L2 once while the smaller
// operand stays resident.  n_fast: M > N (e.g. wgrad 16384 x 4096) -> walk N first.
// group > 0: neither operand fits in L2 (K-heavy dgrad, e.g. 4096 x 4096 x 16384): walk the
// fast dimension in bands of `group` panels so one wave of ~74 tile pairs touches ~8 + 9
// panels instead of all 16 of one operand (ncu: 2.3-3.8x DRAM re-reads without it).
// Measured and rejected (profiles/r02/gemm_raster_ab.txt): snaking 8 x 8 tile blocks so that
// consecutive blocks share 8 panels -- one block streams ~128 MB, more than L2 keeps, and
// traffic went UP 2-9%.
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, bool n_fast, int group, int& mt,
                                            int& nt) {
  int nf = n_fast ? num_n : num_m, ns = n_fast ? num_m : num_n, f, sl;
  if (group > 0 && group < nf) {
    const int band = tile / (group * ns);
    const int first = band * group;
    const int g = min(group, nf - first);
    const int w = tile - band * group * ns;
    f = first + w % g;
    sl = w / g;
  } else {
    f = tile % nf;
    sl = tile / nf;
  }
  if (n_fast) { nt = f; mt = sl; } else { mt = f; nt = sl; }
}

template <int BN, bool A_MN, bool B_MN, int CG>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC, int M, int N, int K, EpiParams ep,
                        SkParams sk, unsigned* __restrict__ sched) {
  using Cfg = GemmCfg<BN, CG>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int TILE_M = GEMM_BM * CG;
  constexpr int BNL = BN / CG;  // B rows (N) loaded by this CTA
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sA = base;
  const uint32_t sB = base + STAGES * Cfg::A_BYTES;
  const uint32_t sE = base + STAGES * Cfg::STAGE_BYTES;  // epilogue staging (1024-aligned)
  const uint32_t bars = sE + Cfg::EPI_BYTES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (bars - base) + 200);
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * STAGES + 2 + a); };
  // dynamic tile scheduler: ring of RING tile indices fed by the leader's producer
  constexpr int RING = 4;
  const uint32_t ring_base = bars + 256;  // RING x u32 tile ids, then full/empty barriers
  auto ring_slot = [&](int s) { return ring_base + 4u * s; };
  auto ring_full = [&](int s) { return ring_base + 32 + 8u * s; };
  auto ring_empty = [&](int s) { return ring_base + 32 + 8u * (RING + s); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = (CG == 2) ? cluster_rank() : 0u;
  const bool leader = crank == 0;

  if (threadIdx.x == 0) {
    // every CTA of this persistent grid is resident: let the next kernel's CTAs launch as ours exit
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      // One arrival (the leader's expect_tx); the peer's TMA bytes complete the
      // transaction on the leader's barrier.  (A .release.cluster remote arrive per
      // stage here halved pair throughput: it compiles to MEMBAR+ERRBAR.)
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 128 * CG);  // every epilogue thread of the pair
    }
    for (int r = 0; r < RING; ++r) {
      mbar_init(ring_full(r), 1);
      // readers: leader MMA + 4 epilogue warps (+ peer producer + 4 peer epilogue warps)
      mbar_init(ring_empty(r), CG == 2 ? 10 : 5);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    if (CG == 2) tmem_alloc2(smem_u32(tmem_slot), Cfg::TMEM_COLS);
    else tmem_alloc(smem_u32(tmem_slot), Cfg::TMEM_COLS);
  }
  tc_fence_before();
  if (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch (the launch sets ProgrammaticStreamSerialization): this CTA's
  // launch and prologue above overlapped the previous kernel's tail; everything below (the
  // tile counter the previous GEMM re-arms, operands, residuals) waits for it to complete.
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const int num_m = (M + TILE_M - 1) / TILE_M;
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_k = (K + GEMM_BK - 1) / GEMM_BK;
  const bool n_fast = M > N;
  constexpr long long kL2Resident = 48ll << 20;  // an operand this small stays in L2
  const int group = (2ll * M * K > kL2Resident && 2ll * N * K > kL2Resident) ? 8 : 0;
  const int num_items = sk.dp_tiles + (num_tiles - sk.dp_tiles) * sk.pieces;
  // work item -> (tile, k-block range, stream-K tile index or -1, piece)
  auto decode = [&](int item, int& tile, int& kb0, int& kb1, int& skt, int& piece) {
    if (item < sk.dp_tiles) {
      tile = item; kb0 = 0; kb1 = num_k; skt = -1; piece = 0;
    } else {
      const int j = item - sk.dp_tiles;
      skt = j / sk.pieces;
      piece = j - skt * sk.pieces;
      tile = sk.dp_tiles + skt;
      kb0 = piece * num_k / sk.pieces;
      kb1 = (piece + 1) * num_k / sk.pieces;
    }
  };
  // K-heavy banded GEMMs (group > 0): a wave of ~`units` concurrent tiles streams more operand
  // bytes than L2 holds, so the next wave would re-read its panels from HBM from k = 0.  Odd
  // waves walk K backwards instead and start on the k-blocks the previous wave touched last,
  // which are still in L2: -7 to -9% DRAM bytes on the K = 12288 / 16384 dgrads
  // (profiles/r02/gemm_raster_ab.txt).  Per tile the order is fixed: results stay deterministic.
  const int units = gridDim.x / CG;
  auto k_reverse = [&](int tile, int skt) { return group > 0 && skt < 0 && ((tile / units) & 1); };
  // Readers take the next tile id from the ring (leader's ring_empty counts the readers).
  const uint32_t ring_empty_leader = (CG == 2) ? map_cta(ring_empty(0), 0) : ring_empty(0);
  auto next_tile = [&](int it, bool arrive) -> int {
    const int slot = it % RING;
    if (CG == 2) mbar_wait_cluster(ring_full(slot), (it / RING) & 1);
    else mbar_wait(ring_full(slot), (it / RING) & 1);
    const int t = static_cast<int>(ld_shared_u32(ring_slot(slot)));
    if (arrive) {
      if (CG == 2) mbar_arrive_remote(ring_empty_leader + 8u * slot);
      else mbar_arrive(ring_empty(slot));
    }
    return t;
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        int tile;
        if (leader) {  // the scheduler: grab a tile and publish it to every role of the pair
          const int slot = it % RING;
          mbar_wait(ring_empty(slot), ((it / RING) & 1) ^ 1);
          tile = static_cast<int>(atomicAdd(sched, 1u));
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(ring_slot(slot)), "r"(tile) : "memory");
          mbar_arrive(ring_full(slot));
          if (CG == 2) {
            st_cluster_u32(map_cta(ring_slot(slot), 1), static_cast<uint32_t>(tile));
            mbar_arrive_cluster(map_cta(ring_full(slot), 1));
          }
        } else {
          tile = next_tile(it, true);
        }
        if (tile >= num_items) break;
        int kb0, kb1, skt, piece;
        decode(tile, tile, kb0, kb1, skt, piece);
        int mt, nt;
        tile_coords(tile, num_m, num_n, n_fast, group, mt, nt);
        const int m0 = mt * TILE_M + crank * GEMM_BM;
        const int n0 = nt * BN + crank * BNL;
        const bool rev = k_reverse(tile, skt);
        for (int j = 0; j < kb1 - kb0; ++j) {
          const int kb = rev ? kb1 - 1 - j : kb0 + j;
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t fb = full_bar(stage);
          if (leader) mbar_arrive_expect_tx(fb, Cfg::STAGE_BYTES * CG);
          const int k0 = kb * GEMM_BK;
          const uint32_t a_dst = sA + stage * Cfg::A_BYTES;
          const uint32_t b_dst = sB + stage * Cfg::B_BYTES;
          auto load = [&](uint32_t dst, const CUtensorMap* m, int c0, int c1) {
            if (CG == 2) tma_load_2d_2sm(dst, m, fb, c0, c1);
            else tma_load_2d(dst, m, fb, c0, c1);
          };
          if (!A_MN) {
            load(a_dst, &tmA, k0, m0);  // box {64 k, 128 m}
          } else {
#pragma unroll
            for (int i = 0; i < GEMM_BM / 64; ++i) load(a_dst + i * 64 * GEMM_BK * 2, &tmA, m0 + 64 * i, k0);
          }
          if (!B_MN) {
            load(b_dst, &tmB, k0, n0);  // box {64 k, BNL n}
          } else {
#pragma unroll
            for (int i = 0; i < BNL / 64; ++i) load(b_dst + i * 64 * GEMM_BK * 2, &tmB, n0 + 64 * i, k0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = make_idesc_bf16(TILE_M, BN, A_MN, B_MN);
      constexpr uint32_t A_LBO = A_MN ? 64 * GEMM_BK * 2 : 16;
      constexpr uint32_t B_LBO = B_MN ? 64 * GEMM_BK * 2 : 16;
      constexpr uint32_t A_KSTEP = A_MN ? 16 * 128 : 32;
      constexpr uint32_t B_KSTEP = B_MN ? 16 * 128 : 32;
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        const int item = next_tile(it, true);
        if (item >= num_items) break;
        int tile, kb0, kb1, skt, piece;
        decode(item, tile, kb0, kb1, skt, piece);
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        unsigned long long* tr = (sk.trace && it < GEMM_TRACE_ITEMS)
                                     ? sk.trace + ((size_t)blockIdx.x * GEMM_TRACE_ITEMS + it) * 6 : nullptr;
        if (tr) { tr[0] = item; tr[1] = gtimer(); }
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int j = 0; j < kb1 - kb0; ++j) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t a_s = sA + stage * Cfg::A_BYTES;
          const uint32_t b_s = sB + stage * Cfg::B_BYTES;
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = make_sdesc(a_s + k * A_KSTEP, A_LBO, 1024);
            const uint64_t bd = make_sdesc(b_s + k * B_KSTEP, B_LBO, 1024);
            const uint32_t accum = (j > 0 || k > 0) ? 1u : 0u;
            if (CG == 2) mma_bf16_2sm(d_tmem, ad, bd, idesc, accum);
            else mma_bf16(d_tmem, ad, bd, idesc, accum);
          }
          if (CG == 2) mma_commit_2sm(empty_bar(stage), 0x3);
          else mma_commit(empty_bar(stage));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (CG == 2) mma_commit_2sm(tfull_bar(acc), 0x3);
        else mma_commit(tfull_bar(acc));
        if (tr) tr[2] = gtimer();
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int mode = ep.mode & 0xF;
    const bool f32out = (mode == ZPP_EPI_F32 || mode == ZPP_EPI_F32_ACC);
    const uint32_t ebuf0 = sE + q * 2 * EPI_BUF;
    const uint32_t tempty_leader = (CG == 2) ? map_cta(tempty_bar(0), 0) : tempty_bar(0);
    int nb = 0;  // nb: staging buffers used so far (ring of 2)
    for (int it = 0;; ++it) {
      const int item = next_tile(it, false);
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_remote(ring_empty_leader + 8u * (it % RING));
        else mbar_arrive(ring_empty(it % RING));
      }
      if (item >= num_items) break;
      int tile, kb0, kb1, skt, piece;
      decode(item, tile, kb0, kb1, skt, piece);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int rl = crank * GEMM_BM + q * 32 + lane;  // row within the TILE_M tile
      unsigned long long* etr = (sk.trace && it < GEMM_TRACE_ITEMS && q == 0 && lane == 0)
                                    ? sk.trace + ((size_t)blockIdx.x * GEMM_TRACE_ITEMS + it) * 6 : nullptr;
      if (etr) { if (!leader || CG == 1) etr[0] = item; etr[3] = gtimer(); }
      // stream-K item: the LAST piece of a tile to arrive finalises it; the others park
      // their fp32 partial in the workspace.  Nobody waits.
      bool own_in_ws = false;  // finisher whose own partial already went to the workspace
      if (skt >= 0) {
        unsigned* f = sk.flags + (skt * CG + crank) * 4 + q;
        uint32_t seen = 0;
        if (lane == 0) seen = ld_acquire_gpu_u32(f);
        seen = __shfl_sync(0xffffffffu, seen, 0);
        if (seen != static_cast<uint32_t>(sk.pieces - 1)) {
          mbar_wait(tfull_bar(acc), acc_phase);
          tc_fence_after();
          if (etr) etr[4] = gtimer();
          const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
          float* dst = sk.ws + (static_cast<long long>(skt) * sk.pieces + piece) * (TILE_M * BN);
#pragma unroll 1
          for (int c = 0; c < BN; c += 32) {
            uint32_t v[32];
            tmem_ld32(t_row + c, v);
            tmem_wait_ld();
            if (c + 32 >= BN) {
              tc_fence_before();
              if (CG == 2) mbar_arrive_remote(tempty_leader + 8u * acc);
              else mbar_arrive(tempty_bar(acc));
            }
            // lane-contiguous: float4 j of every lane is one 512-byte run (coalesced)
            float4* d4 = reinterpret_cast<float4*>(dst) + ((c / 32) * (TILE_M / 32) + (rl >> 5)) * 256 + lane;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              __stcg(d4 + 32 * j, make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                         __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])));
          }
          __threadfence();
          __syncwarp();
          uint32_t prev = 0;
          if (lane == 0) prev = atomicAdd(f, 1u);
          prev = __shfl_sync(0xffffffffu, prev, 0);
          if (etr) etr[5] = gtimer() | (1ull << 63);  // partial parked
          if (prev != static_cast<uint32_t>(sk.pieces - 1)) continue;  // a later piece finalises
          own_in_ws = true;
        }
        __threadfence();  // acquire: every other piece's partial is visible
        if (lane == 0) *f = 0;  // re-arm (the next launch on this stream is ordered after this one)
      }
      const bool finisher = skt >= 0;
      int mt, nt;
      tile_coords(tile, num_m, num_n, n_fast, group, mt, nt);
      const int row0 = mt * TILE_M + crank * GEMM_BM + q * 32;
      const int n0 = nt * BN;
      if (mode == ZPP_EPI_BF16_DGELU && row0 + lane < M) {
        // the dGeLU pre-activation this thread's row will read, into L2 while the MMAs run: read
        // at the point of use it costs an HBM latency per 64-column chunk (FC2 dgrad 121.6 ->
        // 119.0 ms/step in-step, profiles/r02/gemm_streamk_ab.txt; a residual prefetch gained nothing)
        const char* a = reinterpret_cast<const char*>(ep.aux + (long long)(row0 + lane) * ep.ldaux + n0);
        for (int o = 0; o < min(BN, N - n0) * 2; o += 128) prefetch_l2(a + o);
      }
      if (!own_in_ws) {
        mbar_wait(tfull_bar(acc), acc_phase);
        tc_fence_after();
      }
      if (etr) etr[4] = gtimer();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      const int row = row0 + lane;
      constexpr int CHUNK = 32;
      const int cols_per_store = f32out ? 32 : 64;
#pragma unroll 1
      for (int c = 0; c < BN; c += cols_per_store) {
        float x[2][32];
        const int nsub = cols_per_store / CHUNK;
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
          if (sub < nsub && !own_in_ws) {
            uint32_t v[32];
            tmem_ld32(t_row + c + sub * CHUNK, v);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) x[sub][j] = __uint_as_float(v[j]);
          }
        }
        if (finisher) {  // sum all pieces in piece order (deterministic whoever finalises)
          float y[2][32];
#pragma unroll
          for (int sub = 0; sub < 2; ++sub)
#pragma unroll
            for (int j = 0; j < 32; ++j) y[sub][j] = 0.f;
#pragma unroll 1
          for (int pc = 0; pc < sk.pieces; ++pc) {
            if (pc == piece && !own_in_ws) {
#pragma unroll
              for (int sub = 0; sub < 2; ++sub)
#pragma unroll
                for (int j = 0; j < 32; ++j) y[sub][j] += x[sub][j];
              continue;
            }
            const float* src = sk.ws + (static_cast<long long>(skt) * sk.pieces + pc) * (TILE_M * BN);
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
              if (sub < nsub) {
                const float4* s4 = reinterpret_cast<const float4*>(src) +
                                   (((c + sub * CHUNK) / 32) * (TILE_M / 32) + (rl >> 5)) * 256 + lane;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const float4 t = __ldcg(s4 + 32 * j);
                  y[sub][4 * j] += t.x; y[sub][4 * j + 1] += t.y; y[sub][4 * j + 2] += t.z; y[sub][4 * j + 3] += t.w;
                }
              }
            }
          }
#pragma unroll
          for (int sub = 0; sub < 2; ++sub)
#pragma unroll
            for (int j = 0; j < 32; ++j) x[sub][j] = y[sub][j];
        }
        if (c + cols_per_store >= BN && !own_in_ws) {  // accumulator in registers: release TMEM early
          tc_fence_before();
          if (CG == 2) mbar_arrive_remote(tempty_leader + 8u * acc);
          else mbar_arrive(tempty_bar(acc));
        }
        const int col = n0 + c;
        if (col >= N) continue;  // whole chunk beyond the matrix (ragged last tile)
        if (!f32out) {
#pragma unroll
          for (int sub = 0; sub < 2; ++sub)
            if (col + sub * CHUNK < N) epi_math(ep, row, col + sub * CHUNK, x[sub]);
        }
        // stage this warp's 32 rows x 128 B into a 128B-swizzled buffer, then TMA it out
        const uint32_t buf = ebuf0 + (nb & 1) * EPI_BUF;
        if (lane == 0) bulk_wait_read<1>();  // the store that used this buffer has read it
        __syncwarp();
        const uint32_t rbase = buf + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t w0, w1, w2, w3;
          if (f32out) {
            w0 = __float_as_uint(x[0][4 * j]); w1 = __float_as_uint(x[0][4 * j + 1]);
            w2 = __float_as_uint(x[0][4 * j + 2]); w3 = __float_as_uint(x[0][4 * j + 3]);
          } else {
            const float* s = &x[j >> 2][(j & 3) * 8];
            w0 = pack_bf16(s[0], s[1]); w1 = pack_bf16(s[2], s[3]);
            w2 = pack_bf16(s[4], s[5]); w3 = pack_bf16(s[6], s[7]);
          }
          st_shared_v4(rbase + ((j ^ (lane & 7)) << 4), w0, w1, w2, w3);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          if (mode == ZPP_EPI_F32_ACC) tma_reduce_add_2d(&tmC, buf, col, row0);
          else tma_store_2d(&tmC, buf, col, row0);
          bulk_commit();
        }
        ++nb;
      }
      if (etr) etr[5] = gtimer();
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }
  tc_fence_before();
  if (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if (CG == 2) tmem_dealloc2(tmem_base, Cfg::TMEM_COLS);
    else tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
  if (threadIdx.x == 0) {  // the last CTA out re-arms the scheduler slot (stream-ordered reuse)
    __threadfence();
    if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// host side

static int make_map(CUtensorMap* map, CUtensorMapDataType dt, int esize, const void* ptr, uint64_t inner,
                    uint64_t outer, uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * esize};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return encode_tensor_map(map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_SWIZZLE_128B);
}

// Scheduler counters: [tile counter, CTAs done] per stream, zeroed at preload and re-armed by
// the last CTA of each launch.  Launches on one stream are ordered, so a stream owns one
// slot; concurrent GEMMs on different streams never share a counter.  Allocated in
// gemm_preload() -- the launch path never allocates or synchronises.
constexpr int SCHED_STREAMS = 32;
struct SchedSlot {
  cudaStream_t stream;
  bool used;
};
static SchedSlot g_sched_tab[SCHED_STREAMS];
static unsigned* g_sched = nullptr;

static unsigned* sched_slot(cudaStream_t s) {
  if (!g_sched) return nullptr;
  for (int i = 0; i < SCHED_STREAMS; ++i)
    if (g_sched_tab[i].used && g_sched_tab[i].stream == s) return g_sched + 2 * i;
  for (int i = 0; i < SCHED_STREAMS; ++i)
    if (!g_sched_tab[i].used) {
      g_sched_tab[i].used = true;
      g_sched_tab[i].stream = s;
      return g_sched + 2 * i;
    }
  return nullptr;
}

// Stream-K workspaces: one per stream that launches split GEMMs (launches on one stream
// are ordered, so they can share it).  Allocated at preload time -- never inside a step,
// where an allocation could wait on spinning NCCL kernels.  A launch on a stream beyond
// the table simply runs without the split.
constexpr int SK_MAX_PIECES = 4;
constexpr int SK_CTX = 2;
constexpr long long SK_WS_FLOATS = 148LL * SK_MAX_PIECES * 128 * 256;  // (units-1)*p*tile, both CGs
constexpr int SK_FLAGS = 148 * 4;
struct SkCtx {
  cudaStream_t stream;
  bool used;
  float* ws;
  unsigned* flags;
};
static SkCtx g_sk[SK_CTX];
static unsigned long long* g_gemm_trace = nullptr;  // debug build (ZPP_TRACE): last launch's timeline
static bool g_sk_ready = false;
static int g_sk_mode = 1;  // stream-K split of the last partial wave (zpp_gemm_set_streamk)

static int sk_alloc() {
  if (g_sk_ready) return ZPP_OK;
  if (cudaMalloc(&g_sched, SCHED_STREAMS * 2 * sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(g_sched, 0, SCHED_STREAMS * 2 * sizeof(unsigned)) != cudaSuccess)
    return set_error(ZPP_ERR_CUDA, "gemm: scheduler counter allocation failed");
  for (auto& c : g_sk) {
    if (cudaMalloc(&c.ws, SK_WS_FLOATS * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&c.flags, SK_FLAGS * sizeof(unsigned)) != cudaSuccess)
      return set_error(ZPP_ERR_CUDA, "gemm: stream-K workspace allocation failed");
    if (cudaMemset(c.flags, 0, SK_FLAGS * sizeof(unsigned)) != cudaSuccess)
      return set_error(ZPP_ERR_CUDA, "gemm: stream-K flag init failed");
    c.used = false;
  }
#ifdef ZPP_TRACE
  {
    const size_t bytes = 148ull * GEMM_TRACE_ITEMS * 6 * sizeof(unsigned long long);
    if (cudaMalloc(&g_gemm_trace, bytes) != cudaSuccess) return set_error(ZPP_ERR_CUDA, "gemm trace alloc");
    cudaMemset(g_gemm_trace, 0, bytes);
  }
#endif
  cudaDeviceSynchronize();
  g_sk_ready = true;
  return ZPP_OK;
}

static SkCtx* sk_ctx(cudaStream_t s) {
  if (!g_sk_ready) return nullptr;
  for (auto& c : g_sk)
    if (c.used && c.stream == s) return &c;
  for (auto& c : g_sk)
    if (!c.used) {
      c.used = true;
      c.stream = s;
      return &c;
    }
  return nullptr;
}

// Choose the split: whole tiles for the full waves, p pieces for the remainder, p
// minimising (k-blocks on the critical path + a per-piece overhead for the partial
// round trip and pipeline refill).
static SkParams sk_plan(int tiles, int units, int num_k, int tile_m, int bn, cudaStream_t s) {
  SkParams sk{tiles, 1, nullptr, nullptr, g_gemm_trace};
  if (!g_sk_mode || tiles <= units || tiles % units == 0) return sk;
  const int full = tiles / units, r = tiles % units;
  // Measured (tools/gemm_trace.py): parking a 128 KB partial ~6 us and summing it back
  // ~7 us per piece -- the read-back is latency-bound at ~32 KB in flight per SM -- so one
  // extra piece costs ~22 k-blocks (0.34 us each at 256x256 pair tiles) standalone.  In the
  // step (lower clocks, concurrent kernels) it costs more: with 22 the K = 4096 shapes chose a
  // 2-piece split and ran 1-4% slower than whole tiles, while K >= 12288 gains 5-7%
  // (tools/gemm_instep.py --no-streamk, profiles/r02/gemm_streamk_ab.txt); 40 keeps the latter only.
  constexpr int OVH_KB = 40;
  long long best = (long long)(full + 1) * num_k;
  int best_p = 1;
  for (int p = 2; p <= SK_MAX_PIECES; ++p) {
    if (num_k < 4 * p) break;
    const int waves = (r * p + units - 1) / units;
    const long long cost = (long long)full * num_k + (long long)waves * ((num_k + p - 1) / p) + OVH_KB * (p - 1);
    if (cost < best) { best = cost; best_p = p; }
  }
  if (best_p == 1) return sk;
  SkCtx* c = sk_ctx(s);
  if (!c || (long long)r * best_p * tile_m * bn > SK_WS_FLOATS) return sk;
  sk.dp_tiles = full * units;
  sk.pieces = best_p;
  sk.ws = c->ws;
  sk.flags = c->flags;
  return sk;
}

template <int BN, bool A_MN, bool B_MN, int CG>
static int launch_gemm(const void* A, long long lda, const void* B, long long ldb, void* C, long long ldc, int M,
                       int N, int K, const EpiParams& ep, cudaStream_t stream) {
  using Cfg = GemmCfg<BN, CG>;
  constexpr int BNL = BN / CG;
  const CUtensorMapDataType BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUtensorMap ma, mb, mc;
  int rc;
  if (!A_MN) rc = make_map(&ma, BF, 2, A, K, M, lda, GEMM_BK, GEMM_BM);
  else rc = make_map(&ma, BF, 2, A, M, K, lda, 64, GEMM_BK);
  if (rc) return rc;
  if (!B_MN) rc = make_map(&mb, BF, 2, B, K, N, ldb, GEMM_BK, BNL);
  else rc = make_map(&mb, BF, 2, B, N, K, ldb, 64, GEMM_BK);
  if (rc) return rc;
  const int mode = ep.mode & 0xF;
  if (mode == ZPP_EPI_F32 || mode == ZPP_EPI_F32_ACC)
    rc = make_map(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, C, N, M, ldc, 32, 32);
  else
    rc = make_map(&mc, BF, 2, C, N, M, ldc, 64, 32);
  if (rc) return rc;
  auto kern = gemm_tcgen05_kernel<BN, A_MN, B_MN, CG>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "gemm smem attribute");
    attr_set = true;
  }
  const int tiles = ((M + GEMM_BM * CG - 1) / (GEMM_BM * CG)) * ((N + BN - 1) / BN);
  const int units = num_sms() / CG;
  const int grid = (tiles < units ? tiles : units) * CG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  unsigned* sched = sched_slot(stream);
  if (!sched)
    return set_error(ZPP_ERR_ARG, g_sched ? "gemm: more than 32 launching streams"
                                          : "gemm: call zpp_preload_kernels() before the first GEMM");
  const SkParams sk = sk_plan(tiles, grid / CG, (K + GEMM_BK - 1) / GEMM_BK, GEMM_BM * CG, BN, stream);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, M, N, K, ep, sk, sched);
  if (e != cudaSuccess) return set_cuda_error(e, "gemm launch");
  return check_launch("gemm_tcgen05");
}

template <int BN, bool A_MN, bool B_MN, int CG>
static int preload_one() {
  cudaError_t e = cudaFuncSetAttribute(gemm_tcgen05_kernel<BN, A_MN, B_MN, CG>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<BN, CG>::SMEM);
  return e == cudaSuccess ? ZPP_OK : set_cuda_error(e, "gemm preload");
}

int gemm_preload() {
  int rc = sk_alloc();
  rc |= preload_one<256, false, false, 1>(); rc |= preload_one<256, false, true, 1>();
  rc |= preload_one<256, true, false, 1>();  rc |= preload_one<256, true, true, 1>();
  rc |= preload_one<128, false, false, 1>(); rc |= preload_one<128, false, true, 1>();
  rc |= preload_one<128, true, false, 1>();  rc |= preload_one<128, true, true, 1>();
  rc |= preload_one<256, false, false, 2>(); rc |= preload_one<256, false, true, 2>();
  rc |= preload_one<256, true, false, 2>();  rc |= preload_one<256, true, true, 2>();
  rc |= preload_one<128, false, false, 2>(); rc |= preload_one<128, false, true, 2>();
  rc |= preload_one<128, true, false, 2>();  rc |= preload_one<128, true, true, 2>();
  return rc;
}

template <bool A_MN, bool B_MN>
static int dispatch(const void* A, long long lda, const void* B, long long ldb, void* C, long long ldc, int M, int N,
                    int K, const EpiParams& ep, cudaStream_t s, int cg_pref) {
  // Pairs (CG=2, 256-row tiles) whenever there are at least two 256-row tiles; narrow
  // problems use 128-wide tiles so the last N tile wastes less.
  const bool pair = (cg_pref != 1) && M > 256;
  const bool wide = N > 128;
  if (pair) {
    return wide ? launch_gemm<256, A_MN, B_MN, 2>(A, lda, B, ldb, C, ldc, M, N, K, ep, s)
                : launch_gemm<128, A_MN, B_MN, 2>(A, lda, B, ldb, C, ldc, M, N, K, ep, s);
  }
  return wide ? launch_gemm<256, A_MN, B_MN, 1>(A, lda, B, ldb, C, ldc, M, N, K, ep, s)
              : launch_gemm<128, A_MN, B_MN, 1>(A, lda, B, ldb, C, ldc, M, N, K, ep, s);
}

}  // namespace zpp

static int g_cg_pref = 0;  // 0 = auto, 1 = force single-CTA tiles, 2 = prefer pairs

// Debug: copy the last traced launch's timeline ([cta][32 items][item, mma0, mma1, epi0,
// epi_acc, epi1] globaltimer ns) to host memory; returns the number of u64 copied.
#ifdef ZPP_TRACE  // debug build only (make trace)
extern "C" long long zpp_gemm_trace_dump(unsigned long long* host, long long max_u64) {
  if (!zpp::g_gemm_trace) return 0;
  long long n = 148LL * zpp::GEMM_TRACE_ITEMS * 6;
  if (n > max_u64) n = max_u64;
  cudaDeviceSynchronize();
  cudaMemcpy(host, zpp::g_gemm_trace, n * 8, cudaMemcpyDeviceToHost);
  cudaMemset(zpp::g_gemm_trace, 0, 148ull * zpp::GEMM_TRACE_ITEMS * 6 * 8);
  return n;
}
#endif

extern "C" int zpp_gemm_set_streamk(int on) {
  zpp::g_sk_mode = on ? 1 : 0;
  return ZPP_OK;
}

extern "C" int zpp_gemm_set_cta_group(int cg) {
  if (cg < 0 || cg > 2) return zpp::set_error(ZPP_ERR_ARG, "cta group must be 0, 1 or 2");
  g_cg_pref = cg;
  return ZPP_OK;
}

extern "C" int zpp_gemm(const void* A, int a_mn_major, long long lda, const void* B, int b_mn_major,
                        long long ldb, void* C, long long ldc, int M, int N, int K, int epilogue,
                        const void* bias, const void* resid, long long ldr, void* aux, long long ldaux,
                        uintptr_t stream) {
  using namespace zpp;
  if (M <= 0 || N <= 0 || K <= 0) return set_error(ZPP_ERR_ARG, "gemm: empty shape");
  if ((lda % 8) || (ldb % 8)) return set_error(ZPP_ERR_ARG, "gemm: lda/ldb must be multiples of 8 elements");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
    return set_error(ZPP_ERR_ARG, "gemm: A/B/C must be 16-byte aligned");
  const int mode = epilogue & 0xF;
  if (epilogue >> 4) return set_error(ZPP_ERR_ARG, "gemm: bad epilogue flags");
  if (mode > ZPP_EPI_F32_ACC) return set_error(ZPP_ERR_ARG, "gemm: bad epilogue");
  if (mode == ZPP_EPI_BF16_DGELU && !aux) return set_error(ZPP_ERR_ARG, "gemm: DGELU needs aux");
  if ((N % 8) || (ldc % 8) || (resid && ldr % 8) || (aux && ldaux % 8))
    return set_error(ZPP_ERR_ARG, "gemm: N/ldc/ldr/ldaux must be multiples of 8");
  const bool f32 = (mode == ZPP_EPI_F32 || mode == ZPP_EPI_F32_ACC);
  if (f32 && (bias || resid)) return set_error(ZPP_ERR_ARG, "gemm: fp32 epilogues take no bias/resid");
  EpiParams ep{reinterpret_cast<const __nv_bfloat16*>(bias), reinterpret_cast<const __nv_bfloat16*>(resid), ldr,
               reinterpret_cast<__nv_bfloat16*>(aux), ldaux, epilogue, M, N};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!a_mn_major && !b_mn_major) return dispatch<false, false>(A, lda, B, ldb, C, ldc, M, N, K, ep, s, g_cg_pref);
  if (!a_mn_major && b_mn_major) return dispatch<false, true>(A, lda, B, ldb, C, ldc, M, N, K, ep, s, g_cg_pref);
  if (a_mn_major && b_mn_major) return dispatch<true, true>(A, lda, B, ldb, C, ldc, M, N, K, ep, s, g_cg_pref);
  return dispatch<true, false>(A, lda, B, ldb, C, ldc, M, N, K, ep, s, g_cg_pref);
}
