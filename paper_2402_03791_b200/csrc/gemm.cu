// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M,N] (op)= sum_k A(m,k) * B(n,k)        bf16 operands, fp32 accumulation in TMEM
//
// A is K-major (A[m*lda+k]) or M-major (A[k*lda+m]); B is K-major (B[n*ldb+k]) or
// N-major (B[k*ldb+n]).  This covers the three GEMMs of a transformer linear
// (SURVEY.md section 2 kernel table):
//   fwd    Y  = X  W^T   A=X  (K-major)  B=W (K-major)
//   dgrad  dX = dY W     A=dY (K-major)  B=W (N-major)
//   wgrad  dW += dY^T X  A=dY (M-major)  B=X (N-major), fp32 accumulate epilogue
//
// CTA layout (256 threads, 1 CTA/SM, persistent over output tiles):
//   warp 0     TMA producer (one lane): A/B tiles -> smem ring (128B swizzle)
//   warp 1     MMA issuer (one lane): tcgen05.mma 128xBNx16 into TMEM
//   warp 2     TMEM allocator
//   warps 4-7  epilogue: tcgen05.ld -> bias/GeLU/residual/cast -> global
// TMEM holds two BN-column fp32 accumulators so the epilogue of tile i overlaps
// the MMAs of tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ptx.cuh"
#include "zpp_internal.h"

namespace zpp {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 256;

struct EpiParams {
  void* C;
  long long ldc;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* resid;
  long long ldr;
  __nv_bfloat16* aux;
  long long ldaux;
  int mode;
  int M, N;
};

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr int B_BYTES = BN * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr int TMEM_COLS = 2 * BN;  // double-buffered accumulator
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ void store_row_chunk(const EpiParams& p, int row, int col, const uint32_t (&v)[32]) {
  const int mode = p.mode & 0xF;
  const bool full = (col + 32 <= p.N);
  if (mode == ZPP_EPI_F32 || mode == ZPP_EPI_F32_ACC) {
    float* c = reinterpret_cast<float*>(p.C) + (long long)row * p.ldc + col;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 o = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                               __uint_as_float(v[j + 3]));
        if (mode == ZPP_EPI_F32_ACC) {
          float4 old = *reinterpret_cast<float4*>(c + j);
          o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
        }
        *reinterpret_cast<float4*>(c + j) = o;
      }
    } else {
      #pragma unroll
      for (int j = 0; j < 32; ++j) if (col + j < p.N) {
        float o = __uint_as_float(v[j]);
        if (mode == ZPP_EPI_F32_ACC) o += c[j];
        c[j] = o;
      }
    }
    return;
  }
  // bf16 outputs
  float x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = __uint_as_float(v[j]);
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
      for (int j = 0; j < 32; ++j) if (col + j < p.N) x[j] += __bfloat162float(p.bias[col + j]);
    }
  }
  if (mode == ZPP_EPI_BF16_GELU) {
    if (p.aux) {
      __nv_bfloat16* a = p.aux + (long long)row * p.ldaux + col;
      if (full) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 o = make_uint4(pack_bf16(x[j], x[j + 1]), pack_bf16(x[j + 2], x[j + 3]),
                               pack_bf16(x[j + 4], x[j + 5]), pack_bf16(x[j + 6], x[j + 7]));
          *reinterpret_cast<uint4*>(a + j) = o;
        }
      } else {
        #pragma unroll
      for (int j = 0; j < 32; ++j) if (col + j < p.N) a[j] = __float2bfloat16(x[j]);
      }
    }
    // GeLU of the bf16-rounded pre-activation, matching what backward will see
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = gelu_f(__bfloat162float(__float2bfloat16(x[j])));
  } else if (mode == ZPP_EPI_BF16_DGELU) {
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
      for (int j = 0; j < 32; ++j) if (col + j < p.N) x[j] *= gelu_grad_f(__bfloat162float(a[j]));
    }
  }
  if (p.resid) {
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
      for (int j = 0; j < 32; ++j) if (col + j < p.N) x[j] += __bfloat162float(r[j]);
    }
  }
  __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(p.C) + (long long)row * p.ldc + col;
  if (full) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4 o = make_uint4(pack_bf16(x[j], x[j + 1]), pack_bf16(x[j + 2], x[j + 3]), pack_bf16(x[j + 4], x[j + 5]),
                           pack_bf16(x[j + 6], x[j + 7]));
      *reinterpret_cast<uint4*>(c + j) = o;
    }
  } else {
    #pragma unroll
      for (int j = 0; j < 32; ++j) if (col + j < p.N) c[j] = __float2bfloat16(x[j]);
  }
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        int M, int N, int K, EpiParams ep) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sA = base;                                   // STAGES * A_BYTES
  const uint32_t sB = base + STAGES * Cfg::A_BYTES;           // STAGES * B_BYTES
  const uint32_t bars = base + STAGES * Cfg::STAGE_BYTES;     // barrier block
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + STAGES * Cfg::STAGE_BYTES + 200);
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * STAGES + 2 + a); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_m = (M + GEMM_BM - 1) / GEMM_BM;
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_k = (K + GEMM_BK - 1) / GEMM_BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile % num_m) * GEMM_BM;
        const int n0 = (tile / num_m) * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t fb = full_bar(stage);
          mbar_arrive_expect_tx(fb, Cfg::STAGE_BYTES);
          const int k0 = kb * GEMM_BK;
          const uint32_t a_dst = sA + stage * Cfg::A_BYTES;
          const uint32_t b_dst = sB + stage * Cfg::B_BYTES;
          if (!A_MN) {
            tma_load_2d(a_dst, &tmA, fb, k0, m0);  // box {64 k, 128 m}
          } else {
#pragma unroll
            for (int i = 0; i < GEMM_BM / 64; ++i)  // boxes {64 m, 64 k}
              tma_load_2d(a_dst + i * 64 * GEMM_BK * 2, &tmA, fb, m0 + 64 * i, k0);
          }
          if (!B_MN) {
            tma_load_2d(b_dst, &tmB, fb, k0, n0);  // box {64 k, BN n}
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_2d(b_dst + i * 64 * GEMM_BK * 2, &tmB, fb, n0 + 64 * i, k0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(GEMM_BM, BN, A_MN, B_MN);
      // K-major: SBO = 8 rows * 128 B; MN-major: LBO = stride between 64-wide MN atoms.
      constexpr uint32_t A_LBO = A_MN ? 64 * GEMM_BK * 2 : 16;
      constexpr uint32_t B_LBO = B_MN ? 64 * GEMM_BK * 2 : 16;
      // advance per UMMA_K=16 step: K-major +32 B inside the swizzled row; MN-major +16 rows.
      constexpr uint32_t A_KSTEP = A_MN ? 16 * 128 : 32;
      constexpr uint32_t B_KSTEP = B_MN ? 16 * 128 : 32;
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t a_s = sA + stage * Cfg::A_BYTES;
          const uint32_t b_s = sB + stage * Cfg::B_BYTES;
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = make_sdesc(a_s + k * A_KSTEP, A_LBO, 1024);
            const uint64_t bd = make_sdesc(b_s + k * B_KSTEP, B_LBO, 1024);
            mma_bf16(d_tmem, ad, bd, idesc, (kb | k) ? 1u : 0u);
          }
          mma_commit(empty_bar(stage));  // frees the smem slot once these MMAs retire
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(tfull_bar(acc));  // accumulator ready for the epilogue
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row_in_tile = q * 32 + lane;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m0 = (tile % num_m) * GEMM_BM;
      const int n0 = (tile / num_m) * BN;
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      const int row = m0 + row_in_tile;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(t_row + c * 32, v);
        tmem_wait_ld();
        const int col = n0 + c * 32;
        if (row < M && col < N) store_row_chunk(ep, row, col, v);
      }
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
}

// ---------------------------------------------------------------------------
// host side

static int make_map_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                         uint32_t box_inner, uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return encode_tensor_map(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                           estr, CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int BN, bool A_MN, bool B_MN>
static int launch_gemm(const void* A, long long lda, const void* B, long long ldb, int M, int N, int K,
                       const EpiParams& ep, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  CUtensorMap ma, mb;
  int rc;
  if (!A_MN) rc = make_map_bf16(&ma, A, K, M, lda, GEMM_BK, GEMM_BM);
  else rc = make_map_bf16(&ma, A, M, K, lda, 64, GEMM_BK);
  if (rc) return rc;
  if (!B_MN) rc = make_map_bf16(&mb, B, K, N, ldb, GEMM_BK, BN);
  else rc = make_map_bf16(&mb, B, N, K, ldb, 64, GEMM_BK);
  if (rc) return rc;
  auto kern = gemm_tcgen05_kernel<BN, A_MN, B_MN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "gemm smem attribute");
    attr_set = true;
  }
  const int tiles = ((M + GEMM_BM - 1) / GEMM_BM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  kern<<<grid, GEMM_THREADS, Cfg::SMEM, stream>>>(ma, mb, M, N, K, ep);
  return check_launch("gemm_tcgen05");
}

}  // namespace zpp

extern "C" int zpp_gemm(const void* A, int a_mn_major, long long lda, const void* B, int b_mn_major,
                        long long ldb, void* C, long long ldc, int M, int N, int K, int epilogue,
                        const void* bias, const void* resid, long long ldr, void* aux, long long ldaux,
                        uintptr_t stream) {
  using namespace zpp;
  if (M <= 0 || N <= 0 || K <= 0) return set_error(ZPP_ERR_ARG, "gemm: empty shape");
  if ((lda % 8) || (ldb % 8)) return set_error(ZPP_ERR_ARG, "gemm: lda/ldb must be multiples of 8 elements");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15)
    return set_error(ZPP_ERR_ARG, "gemm: A/B must be 16-byte aligned");
  const int mode = epilogue & 0xF;
  if (mode > ZPP_EPI_F32_ACC) return set_error(ZPP_ERR_ARG, "gemm: bad epilogue");
  if (mode == ZPP_EPI_BF16_DGELU && !aux) return set_error(ZPP_ERR_ARG, "gemm: DGELU needs aux");
  if ((N % 8) || (ldc % 8) || (resid && ldr % 8) || (aux && ldaux % 8))
    return set_error(ZPP_ERR_ARG, "gemm: N/ldc/ldr/ldaux must be multiples of 8");
  EpiParams ep{C, ldc, reinterpret_cast<const __nv_bfloat16*>(bias), reinterpret_cast<const __nv_bfloat16*>(resid),
               ldr, reinterpret_cast<__nv_bfloat16*>(aux), ldaux, epilogue, M, N};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // Narrow problems waste half a 256-wide tile; use BN=128 there.
  const bool wide = N > 128;
  if (!a_mn_major && !b_mn_major)
    return wide ? launch_gemm<256, false, false>(A, lda, B, ldb, M, N, K, ep, s)
                : launch_gemm<128, false, false>(A, lda, B, ldb, M, N, K, ep, s);
  if (!a_mn_major && b_mn_major)
    return wide ? launch_gemm<256, false, true>(A, lda, B, ldb, M, N, K, ep, s)
                : launch_gemm<128, false, true>(A, lda, B, ldb, M, N, K, ep, s);
  if (a_mn_major && b_mn_major)
    return wide ? launch_gemm<256, true, true>(A, lda, B, ldb, M, N, K, ep, s)
                : launch_gemm<128, true, true>(A, lda, B, ldb, M, N, K, ep, s);
  return wide ? launch_gemm<256, true, false>(A, lda, B, ldb, M, N, K, ep, s)
              : launch_gemm<128, true, false>(A, lda, B, ldb, M, N, K, ep, s);
}
