// Causal multi-head attention forward/backward over packed qkv [b, s, 3, heads, d].
//
// Round-1 implementation: FlashAttention-2 style tiling (online softmax, no s^2
// materialisation, recompute in backward) on the legacy mma.sync m16n8k16 bf16
// tensor path with XOR-swizzled cp.async tiles and ldmatrix fragments.  It is
// the stop-gap the design notes call out: attention is ~8% of GPT-6.2B FLOPs
// and moves to tcgen05/TMEM next ("next").
//
// fwd : grid (s/64, b*heads), 4 warps, each warp owns 16 query rows; K/V tiles of
//       64 keys double-buffered; writes O (bf16) and lse (fp32, natural log).
// bwd : delta = rowsum(dO*O); grid (s/64 key blocks, b*heads); per key block
//       loop over query blocks on/after the diagonal: recompute P, dV += P^T dO,
//       dS = P*(dP-delta)*scale, dK += dS^T Q, dQ += dS K (fp32 atomics into a
//       workspace, converted to bf16 at the end).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ptx.cuh"
#include "zpp_internal.h"

namespace zpp {

typedef __nv_bfloat16 bf16;

template <int D>
int attn_fwd_tc_launch(const void* qkv, void* out, float* lse, int B, int T, int H, cudaStream_t s);
template <int D>
int attn_fwd2_tc_launch(const void* qkv, void* out, float* lse, int B, int T, int H, cudaStream_t s);
template <int D>
int attn_bwd_split_tc_launch(const void* qkv, const void* dout, const float* lse, const float* delta, void* dqkv,
                             int B, int T, int H, cudaStream_t s);
template <int D>
int attn_bwd_tc_launch(const void* qkv, const void* dout, const float* lse, const float* delta, void* dqkv,
                       float* dq_acc, int B, int T, int H, cudaStream_t s);

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Swizzled [rows][D] bf16 tile: 16-byte chunk c of row r lives at chunk c ^ (r & 7).
template <int D>
__device__ __forceinline__ uint32_t tile_addr(uint32_t base, int r, int col) {
  const int chunk = (col >> 3) ^ (r & 7);
  return base + r * (D * 2) + chunk * 16 + (col & 7) * 2;
}

// Async-copy a [64][D] tile whose row t lives at src + t*stride (elements).
template <int D, int NT>
__device__ __forceinline__ void load_tile(uint32_t dst, const bf16* src, long long stride) {
  constexpr int CH = D / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < 64 * CH; i += NT) {
    const int r = i / CH, c = i % CH;
    cp_async16(dst + r * (D * 2) + ((c ^ (r & 7)) * 16), src + r * stride + c * 8);
  }
}

constexpr float LOG2E = 1.4426950408889634f;

// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(128) attn_fwd_kernel(const bf16* __restrict__ qkv, bf16* __restrict__ out,
                                                       float* __restrict__ lse, int T, int H, float scale) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK0 = sQ + 64 * D * 2;
  const uint32_t sV0 = sK0 + 2 * 64 * D * 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int qblk = gridDim.x - 1 - blockIdx.x;  // longest (latest) query blocks first
  const int q0 = qblk * 64;
  const long long rs = 3LL * H * D;
  const bf16* qb = qkv + (long long)b * T * rs + (long long)h * D;
  const bf16* kb_ = qb + (long long)H * D;
  const bf16* vb_ = qb + 2LL * H * D;
  const float sl2 = scale * LOG2E;

  load_tile<D, 128>(sQ, qb + q0 * rs, rs);
  load_tile<D, 128>(sK0, kb_, rs);
  load_tile<D, 128>(sV0, vb_, rs);
  cp_commit();

  uint32_t qf[D / 16][4];
  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  const int nkb = qblk + 1;
  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) {
      load_tile<D, 128>(sK0 + (buf ^ 1) * 64 * D * 2, kb_ + (kb + 1) * 64 * rs, rs);
      load_tile<D, 128>(sV0 + (buf ^ 1) * 64 * D * 2, vb_ + (kb + 1) * 64 * rs, rs);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = kk * 16 + (lane >> 4) * 8;
        ldsm_x4(tile_addr<D>(sQ, r, c), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    const uint32_t sK = sK0 + buf * 64 * D * 2, sV = sV0 + buf * 64 * D * 2;
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of 8-key n-tiles
        uint32_t b0, b1, b2, b3;
        const int r = np * 16 + (lane & 7) + (lane >> 4) * 8;
        const int c = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(tile_addr<D>(sK, r, c), b0, b1, b2, b3);
        mma16816(s[2 * np], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
        mma16816(s[2 * np + 1], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
      }
    }
    // scale into log2 domain, causal mask on the diagonal block
    const int qr0 = q0 + warp * 16 + g, qr1 = qr0 + 8;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v = s[nt][j] * sl2;
        if (kb == qblk) {
          const int key = kb * 64 + nt * 8 + 2 * t4 + (j & 1);
          const int q = (j < 2) ? qr0 : qr1;
          if (key > q) v = -INFINITY;
        }
        s[nt][j] = v;
      }
    }
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
    }
#pragma unroll
    for (int o_ = 1; o_ <= 2; o_ <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o_));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o_));
    }
    const float c0 = exp2f(m0 - mx0), c1 = exp2f(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = exp2f(s[nt][0] - m0);
      s[nt][1] = exp2f(s[nt][1] - m0);
      s[nt][2] = exp2f(s[nt][2] - m1);
      s[nt][3] = exp2f(s[nt][3] - m1);
      rs0 += s[nt][0] + s[nt][1];
      rs1 += s[nt][2] + s[nt][3];
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= c0; o[i][1] *= c0;
      o[i][2] *= c1; o[i][3] *= c1;
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t a0 = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      const uint32_t a1 = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      const uint32_t a2 = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      const uint32_t a3 = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t b0, b1, b2, b3;
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = dn * 16 + (lane >> 4) * 8;
        ldsm_x4_t(tile_addr<D>(sV, r, c), b0, b1, b2, b3);
        mma16816(o[2 * dn], a0, a1, a2, a3, b0, b1);
        mma16816(o[2 * dn + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();
  }
  // finalize
#pragma unroll
  for (int o_ = 1; o_ <= 2; o_ <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o_);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o_);
  }
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  const int r0 = q0 + warp * 16 + g;
  bf16* ob = out + ((long long)b * T) * H * D + (long long)h * D;
#pragma unroll
  for (int dn = 0; dn < D / 8; ++dn) {
    const int col = dn * 8 + 2 * t4;
    *reinterpret_cast<uint32_t*>(ob + (long long)r0 * H * D + col) = pack_bf16(o[dn][0] * i0, o[dn][1] * i0);
    *reinterpret_cast<uint32_t*>(ob + (long long)(r0 + 8) * H * D + col) = pack_bf16(o[dn][2] * i1, o[dn][3] * i1);
  }
  if (t4 == 0) {
    float* lb = lse + (long long)bh * T;
    lb[r0] = (m0 + log2f(l0)) / LOG2E;
    lb[r0 + 8] = (m1 + log2f(l1)) / LOG2E;
  }
}

// delta[bh][t] = sum_d dO[t,h,d] * O[t,h,d]; one warp per (t, h)
template <int D>
// delta[b,h,t] = sum_d out*dout; also zeroes the fp32 dQ accumulator row it owns (the
// backward kernels reduce-add into it), so no separate memset is launched.
__global__ void attn_delta_kernel(const bf16* __restrict__ out, const bf16* __restrict__ dout,
                                  float* __restrict__ delta, float* __restrict__ dq, int B, int T, int H) {
  // D/8 threads per (token, head): one 16-byte vector of O and of dO each, reduced over the
  // D/8 lanes with shuffles (full-sector coalesced loads, 32 B in flight per thread)
  constexpr int L = D / 8;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long w = tid / L;
  const int c = static_cast<int>(tid % L);
  const bool ok = w < (long long)B * T * H;
  float acc = 0.f;
  if (ok) {
    const uint4 ov = reinterpret_cast<const uint4*>(out + w * D)[c];
    const uint4 dv = reinterpret_cast<const uint4*>(dout + w * D)[c];
    acc = bf16lo(ov.x) * bf16lo(dv.x) + bf16hi(ov.x) * bf16hi(dv.x) + bf16lo(ov.y) * bf16lo(dv.y) +
          bf16hi(ov.y) * bf16hi(dv.y) + bf16lo(ov.z) * bf16lo(dv.z) + bf16hi(ov.z) * bf16hi(dv.z) +
          bf16lo(ov.w) * bf16lo(dv.w) + bf16hi(ov.w) * bf16hi(dv.w);
  }
#pragma unroll
  for (int x = L / 2; x > 0; x >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, x);
  if (!ok) return;
  const int h = w % H;
  const long long bt = w / H;
  const int t = bt % T, b = bt / T;
  if (c == 0) delta[((long long)b * H + h) * T + t] = acc;
  if (!dq) return;
  float4* z = reinterpret_cast<float4*>(dq + w * D);
  for (int i = c; i < D / 4; i += L) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(128) attn_bwd_kernel(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                       const float* __restrict__ lse, const float* __restrict__ delta,
                                                       bf16* __restrict__ dqkv, float* __restrict__ dq_acc, int T,
                                                       int H, float scale) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sK = smem_u32(smem);
  const uint32_t sV = sK + 64 * D * 2;
  const uint32_t sQ = sV + 64 * D * 2;
  const uint32_t sdO = sQ + 64 * D * 2;
  const uint32_t sP = sdO + 64 * D * 2;   // [64 q][64 k] bf16, swizzled as D=64 tile
  const uint32_t sdS = sP + 64 * 64 * 2;
  float* sL = reinterpret_cast<float*>(smem + 4 * 64 * D * 2 + 2 * 64 * 64 * 2);  // lse*log2e [64]
  float* sDl = sL + 64;                                                           // delta [64]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int kblk = blockIdx.x;
  const int k0 = kblk * 64;
  const long long rs = 3LL * H * D;
  const long long ors = (long long)H * D;
  const bf16* qb = qkv + (long long)b * T * rs + (long long)h * D;
  const bf16* kbase = qb + (long long)H * D;
  const bf16* vbase = qb + 2LL * H * D;
  const bf16* dob = dout + (long long)b * T * ors + (long long)h * D;
  const float sl2 = scale * LOG2E;

  load_tile<D, 128>(sK, kbase + k0 * rs, rs);
  load_tile<D, 128>(sV, vbase + k0 * rs, rs);
  cp_commit();

  float dv[D / 8][4], dk[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) {
    dv[i][0] = dv[i][1] = dv[i][2] = dv[i][3] = 0.f;
    dk[i][0] = dk[i][1] = dk[i][2] = dk[i][3] = 0.f;
  }
  const int nq = T / 64;
  for (int qblk = kblk; qblk < nq; ++qblk) {
    const int q0 = qblk * 64;
    load_tile<D, 128>(sQ, qb + q0 * rs, rs);
    load_tile<D, 128>(sdO, dob + q0 * ors, ors);
    cp_commit();
    if (threadIdx.x < 64) {
      sL[threadIdx.x] = lse[(long long)bh * T + q0 + threadIdx.x] * LOG2E;
      sDl[threadIdx.x] = delta[(long long)bh * T + q0 + threadIdx.x];
    }
    cp_wait<0>();
    __syncthreads();

    // S = Q K^T and dP = dO V^T for this warp's 16 query rows
    float s[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
      dp[i][0] = dp[i][1] = dp[i][2] = dp[i][3] = 0.f;
    }
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t a0, a1, a2, a3, e0, e1, e2, e3;
      const int ra = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      const int ca = kk * 16 + (lane >> 4) * 8;
      ldsm_x4(tile_addr<D>(sQ, ra, ca), a0, a1, a2, a3);
      ldsm_x4(tile_addr<D>(sdO, ra, ca), e0, e1, e2, e3);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b0, b1, b2, b3;
        const int r = np * 16 + (lane & 7) + (lane >> 4) * 8;
        const int c = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(tile_addr<D>(sK, r, c), b0, b1, b2, b3);
        mma16816(s[2 * np], a0, a1, a2, a3, b0, b1);
        mma16816(s[2 * np + 1], a0, a1, a2, a3, b2, b3);
        ldsm_x4(tile_addr<D>(sV, r, c), b0, b1, b2, b3);
        mma16816(dp[2 * np], e0, e1, e2, e3, b0, b1);
        mma16816(dp[2 * np + 1], e0, e1, e2, e3, b2, b3);
      }
    }
    const int lr0 = warp * 16 + g, lr1 = lr0 + 8;  // local query rows
    const float L0 = sL[lr0], L1 = sL[lr1], D0 = sDl[lr0], D1 = sDl[lr1];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int lq = (j < 2) ? lr0 : lr1;
        const int key = k0 + nt * 8 + 2 * t4 + (j & 1);
        float p = exp2f(s[nt][j] * sl2 - ((j < 2) ? L0 : L1));
        if (key > q0 + lq) p = 0.f;
        s[nt][j] = p;
        dp[nt][j] = p * (dp[nt][j] - ((j < 2) ? D0 : D1)) * scale;
      }
      // write P and dS rows (q-major) to smem as bf16
      const int col = nt * 8 + 2 * t4;
      *reinterpret_cast<uint32_t*>(smem + (tile_addr<64>(sP, lr0, col) - sK)) = pack_bf16(s[nt][0], s[nt][1]);
      *reinterpret_cast<uint32_t*>(smem + (tile_addr<64>(sP, lr1, col) - sK)) = pack_bf16(s[nt][2], s[nt][3]);
      *reinterpret_cast<uint32_t*>(smem + (tile_addr<64>(sdS, lr0, col) - sK)) = pack_bf16(dp[nt][0], dp[nt][1]);
      *reinterpret_cast<uint32_t*>(smem + (tile_addr<64>(sdS, lr1, col) - sK)) = pack_bf16(dp[nt][2], dp[nt][3]);
    }
    __syncthreads();

    // dV += P^T dO ; dK += dS^T Q   (this warp: keys 16*warp .. +15)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // over 16-query chunks
      uint32_t p0, p1, p2, p3, d0, d1, d2, d3;
      // A = P^T rows=keys, cols=queries: transposed read of sP [q][k]
      const int rq = kk * 16 + (lane & 7) + (lane >> 4) * 8;
      const int ck = warp * 16 + ((lane >> 3) & 1) * 8;
      ldsm_x4_t(tile_addr<64>(sP, rq, ck), p0, p1, p2, p3);
      ldsm_x4_t(tile_addr<64>(sdS, rq, ck), d0, d1, d2, d3);
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t b0, b1, b2, b3;
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = dn * 16 + (lane >> 4) * 8;
        ldsm_x4_t(tile_addr<D>(sdO, r, c), b0, b1, b2, b3);
        mma16816(dv[2 * dn], p0, p1, p2, p3, b0, b1);
        mma16816(dv[2 * dn + 1], p0, p1, p2, p3, b2, b3);
        ldsm_x4_t(tile_addr<D>(sQ, r, c), b0, b1, b2, b3);
        mma16816(dk[2 * dn], d0, d1, d2, d3, b0, b1);
        mma16816(dk[2 * dn + 1], d0, d1, d2, d3, b2, b3);
      }
    }
    // dQ (this warp's 16 query rows) += dS K, flushed with fp32 atomics in two halves of d
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float dq[D / 16][4];
#pragma unroll
      for (int i = 0; i < D / 16; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // over 16-key chunks
        uint32_t a0, a1, a2, a3;
        const int ra = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int ca = kk * 16 + (lane >> 4) * 8;
        ldsm_x4(tile_addr<64>(sdS, ra, ca), a0, a1, a2, a3);
#pragma unroll
        for (int dn = 0; dn < D / 32; ++dn) {
          uint32_t b0, b1, b2, b3;
          const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
          const int c = half * (D / 2) + dn * 16 + (lane >> 4) * 8;
          ldsm_x4_t(tile_addr<D>(sK, r, c), b0, b1, b2, b3);
          mma16816(dq[2 * dn], a0, a1, a2, a3, b0, b1);
          mma16816(dq[2 * dn + 1], a0, a1, a2, a3, b2, b3);
        }
      }
      float* dqb = dq_acc + ((long long)b * T) * H * D + (long long)h * D;
#pragma unroll
      for (int i = 0; i < D / 16; ++i) {
        const int col = half * (D / 2) + i * 8 + 2 * t4;
        float* p0 = dqb + (long long)(q0 + lr0) * H * D + col;
        float* p1 = dqb + (long long)(q0 + lr1) * H * D + col;
        atomicAdd(p0, dq[i][0]);
        atomicAdd(p0 + 1, dq[i][1]);
        atomicAdd(p1, dq[i][2]);
        atomicAdd(p1 + 1, dq[i][3]);
      }
    }
    __syncthreads();
  }
  // write dK, dV for this warp's 16 keys
  bf16* dkb = dqkv + (long long)b * T * rs + (long long)H * D + (long long)h * D;
  bf16* dvb = dkb + (long long)H * D;
  const int kr0 = k0 + warp * 16 + g;
#pragma unroll
  for (int dn = 0; dn < D / 8; ++dn) {
    const int col = dn * 8 + 2 * t4;
    *reinterpret_cast<uint32_t*>(dkb + kr0 * rs + col) = pack_bf16(dk[dn][0], dk[dn][1]);
    *reinterpret_cast<uint32_t*>(dkb + (kr0 + 8) * rs + col) = pack_bf16(dk[dn][2], dk[dn][3]);
    *reinterpret_cast<uint32_t*>(dvb + kr0 * rs + col) = pack_bf16(dv[dn][0], dv[dn][1]);
    *reinterpret_cast<uint32_t*>(dvb + (kr0 + 8) * rs + col) = pack_bf16(dv[dn][2], dv[dn][3]);
  }
}

// dq (fp32 [b,T,H,D]) -> dqkv q slot (bf16)
template <int D>
__global__ void dq_convert_kernel(const float* __restrict__ dq, bf16* __restrict__ dqkv, long long rows, int H) {
  const long long n = rows * H * D / 4;  // rows = b*T
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long e = i * 4;
    const long long row = e / ((long long)H * D);
    const long long within = e % ((long long)H * D);
    const float4 v = reinterpret_cast<const float4*>(dq)[i];
    bf16* dst = dqkv + row * 3LL * H * D + within;
    *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
  }
}

template <int D>
static int attn_fwd_launch(const void* qkv, void* out, float* lse, int B, int T, int H, cudaStream_t s) {
  const int smem = 5 * 64 * D * 2;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_fwd attr");
    set = true;
  }
  dim3 grid(T / 64, B * H);
  attn_fwd_kernel<D><<<grid, 128, smem, s>>>((const bf16*)qkv, (bf16*)out, lse, T, H, 1.f / sqrtf((float)D));
  return check_launch("attn_fwd");
}

// Two-kernel tcgen05 backward (attention_bwd_tc.cu) unless ZPP_ATTN_BWD_FUSED=1 selects the
// fused key-outer kernel with fp32 dQ reduction (kept for comparison).
static bool bwd_split() {
  static int v = -1;
  if (v < 0) v = getenv("ZPP_ATTN_BWD_FUSED") ? 0 : 1;
  return v == 1;
}

template <int D>
static int attn_bwd_launch(const void* qkv, const void* out, const float* lse, const void* dout, void* dqkv,
                           float* ws, int B, int T, int H, cudaStream_t s, bool use_tc) {
  const int smem = 4 * 64 * D * 2 + 2 * 64 * 64 * 2 + 2 * 64 * 4;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_bwd attr");
    set = true;
  }
  float* delta = ws;
  float* dq = ws + (long long)B * H * T;
  const long long nrows = (long long)B * T;
  const long long warps = nrows * H;
  const bool split = use_tc && bwd_split();
  attn_delta_kernel<D><<<(int)((warps * (D / 8) + 255) / 256), 256, 0, s>>>((const bf16*)out, (const bf16*)dout,
                                                                           delta, split ? nullptr : dq, B, T, H);
  int rc = check_launch("attn_delta");
  if (rc) return rc;
  if (split) return attn_bwd_split_tc_launch<D>(qkv, dout, lse, delta, dqkv, B, T, H, s);
  if (use_tc) {
    rc = attn_bwd_tc_launch<D>(qkv, dout, lse, delta, dqkv, dq, B, T, H, s);
  } else {
    dim3 grid(T / 64, B * H);
    attn_bwd_kernel<D><<<grid, 128, smem, s>>>((const bf16*)qkv, (const bf16*)dout, lse, delta, (bf16*)dqkv, dq, T,
                                                H, 1.f / sqrtf((float)D));
    rc = check_launch("attn_bwd");
  }
  if (rc) return rc;
  const long long n4 = nrows * H * D / 4;
  int blocks = (int)((n4 + 255) / 256);
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  dq_convert_kernel<D><<<blocks, 256, 0, s>>>(dq, (bf16*)dqkv, nrows, H);
  return check_launch("attn_dq_convert");
}


}  // namespace zpp

using namespace zpp;

namespace zpp {
int attention_tc_preload();
int attention_fwd2_preload();
int attention_bwd_tc_preload();
int gemm_preload();
int kernels_preload();
}  // namespace zpp

// Force-load every kernel of the library (CUDA lazy loading would otherwise load a
// kernel at its first launch, which needs a context-wide synchronisation: that
// deadlocks against NCCL kernels spinning on a peer rank).
extern "C" int zpp_preload_kernels(void) {
  int rc = gemm_preload();
  if (rc) return rc;
  rc = attention_tc_preload();
  if (rc) return rc;
  rc = attention_bwd_tc_preload();
  if (rc) return rc;
  rc = attention_fwd2_preload();
  if (rc) return rc;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, attn_fwd_kernel<64>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, attn_fwd_kernel<128>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, attn_bwd_kernel<64>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, attn_bwd_kernel<128>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, attn_delta_kernel<64>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, attn_delta_kernel<128>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, dq_convert_kernel<64>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, dq_convert_kernel<128>);
  if (e != cudaSuccess) return set_cuda_error(e, "attention preload");
  return kernels_preload();
}

// 0 = auto (tcgen05; two query tiles per CTA when seq % 256 == 0), 1 = mma.sync FA2 tiles,
// 2 = tcgen05 with one query tile per CTA (forward only; comparison / tests)
static int g_attn_impl = 0;

extern "C" int zpp_attn_set_impl(int impl) {
  if (impl < 0 || impl > 2) return set_error(ZPP_ERR_ARG, "attn impl must be 0, 1 or 2");
  g_attn_impl = impl;
  return ZPP_OK;
}

extern "C" int zpp_attn_fwd(const void* qkv, void* out, float* lse, int batch, int seq, int heads, int head_dim,
                            uintptr_t stream) {
  if (seq % 64) return set_error(ZPP_ERR_ARG, "attn: seq must be a multiple of 64");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (g_attn_impl == 0 && seq % 256 == 0) {
    if (head_dim == 128) return attn_fwd2_tc_launch<128>(qkv, out, lse, batch, seq, heads, s);
    if (head_dim == 64) return attn_fwd2_tc_launch<64>(qkv, out, lse, batch, seq, heads, s);
  }
  if (g_attn_impl != 1 && seq % 128 == 0) {
    if (head_dim == 128) return attn_fwd_tc_launch<128>(qkv, out, lse, batch, seq, heads, s);
    if (head_dim == 64) return attn_fwd_tc_launch<64>(qkv, out, lse, batch, seq, heads, s);
  }
  if (head_dim == 128) return attn_fwd_launch<128>(qkv, out, lse, batch, seq, heads, s);
  if (head_dim == 64) return attn_fwd_launch<64>(qkv, out, lse, batch, seq, heads, s);
  return set_error(ZPP_ERR_ARG, "attn: head_dim must be 64 or 128");
}

extern "C" long long zpp_attn_bwd_workspace_floats(int batch, int seq, int heads, int head_dim) {
  return (long long)batch * heads * seq + (long long)batch * seq * heads * head_dim;
}

extern "C" int zpp_attn_bwd(const void* qkv, const void* out, const float* lse, const void* dout, void* dqkv,
                            float* workspace, int batch, int seq, int heads, int head_dim, uintptr_t stream) {
  if (seq % 64) return set_error(ZPP_ERR_ARG, "attn_bwd: seq must be a multiple of 64");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool tc = g_attn_impl != 1 && seq % 128 == 0;
  if (head_dim == 128) return attn_bwd_launch<128>(qkv, out, lse, dout, dqkv, workspace, batch, seq, heads, s, tc);
  if (head_dim == 64) return attn_bwd_launch<64>(qkv, out, lse, dout, dqkv, workspace, batch, seq, heads, s, tc);
  return set_error(ZPP_ERR_ARG, "attn_bwd: head_dim must be 64 or 128");
}
