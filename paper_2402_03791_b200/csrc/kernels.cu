// HBM-bound kernels of the ZeroPP step: LayerNorm / RMSNorm fwd/bwd, bias-grad column
// sums, GeLU, SwiGLU fwd/bwd, rotary embedding, embedding fwd/bwd, fused softmax cross-entropy, ZeRO grad cast/accumulate,
// sharded AdamW and the deterministic parameter initialiser.
//
// Every kernel moves 16-byte vectors, keeps fp32 statistics, and uses fixed-order
// (deterministic) reductions except the embedding scatter (fp32 atomics).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ptx.cuh"
#include "zpp_internal.h"

namespace zpp {

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum for blockDim.x == NT (NT / 32 warps); result broadcast to all threads.
template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = (l < NT / 32) ? red[l] : 0.f;
  t = warp_sum(t);
  return t;
}

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  f[0] = bf16lo(u.x); f[1] = bf16hi(u.x); f[2] = bf16lo(u.y); f[3] = bf16hi(u.y);
  f[4] = bf16lo(u.z); f[5] = bf16hi(u.z); f[6] = bf16lo(u.w); f[7] = bf16hi(u.w);
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  return make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
}

// ----------------------------------------------------------------------------
// LayerNorm: one NT-thread block per row, row cached in registers (cols <= 8 * LN_VPT * NT).
// NT = 128 for rows of <= 4096 columns: 4 vectors in flight per thread and 16 rows per SM.
constexpr int LN_VPT = 4;  // uint4 (8 bf16) vectors per thread

// RMS = true: RMSNorm (LLaMA): mean fixed at 0, no beta; mean_out may be null.
template <bool RMS, int NT>
__global__ void __launch_bounds__(NT) layernorm_fwd_kernel(const bf16* __restrict__ x, const bf16* __restrict__ g,
                                                            const bf16* __restrict__ b, bf16* __restrict__ y,
                                                            float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                            int cols, float eps) {
  __shared__ float red[NT / 32];
  const int row = blockIdx.x;
  const bf16* xr = x + (long long)row * cols;
  const int nvec = cols / 8;
  float v[LN_VPT][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < LN_VPT; ++i) {
    const int vi = threadIdx.x + i * NT;
    if (vi < nvec) {
      unpack8(*reinterpret_cast<const uint4*>(xr + vi * 8), v[i]);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[i][j];
    }
  }
  const float mean = RMS ? 0.f : block_sum<NT>(s, red) / cols;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < LN_VPT; ++i) {
    const int vi = threadIdx.x + i * NT;
    if (vi < nvec) {
#pragma unroll
      for (int j = 0; j < 8; ++j) { const float d = v[i][j] - mean; q += d * d; }
    }
  }
  const float rstd = rsqrtf(block_sum<NT>(q, red) / cols + eps);
  bf16* yr = y + (long long)row * cols;
#pragma unroll
  for (int i = 0; i < LN_VPT; ++i) {
    const int vi = threadIdx.x + i * NT;
    if (vi < nvec) {
      float gg[8], bb[8] = {0, 0, 0, 0, 0, 0, 0, 0}, o[8];
      unpack8(*reinterpret_cast<const uint4*>(g + vi * 8), gg);
      if (!RMS) unpack8(*reinterpret_cast<const uint4*>(b + vi * 8), bb);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = (v[i][j] - mean) * rstd * gg[j] + bb[j];
      *reinterpret_cast<uint4*>(yr + vi * 8) = pack8(o);
    }
  }
  if (threadIdx.x == 0) {
    if (!RMS) mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

// Row data streamed past L1 (gamma/beta, read by every row, stay L1-resident).
__device__ __forceinline__ uint4 ld_na(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Backward dx for rows of <= 4096 columns (the default there): x, dy and the residual grad
// are held as packed bf16 (48 registers instead of 64 floats + 16) and xhat, dy*g are
// recomputed at each use, so 8 rows fit per SM instead of 5: 42.3 -> 34.6 us at 4096 x 4096
// (profiles/r01d_ln_pk_ab.txt).  The same packing in the forward was slower (24.2 -> 26.1 us)
// and is not used.
template <bool RMS>
__global__ void __launch_bounds__(128) layernorm_bwd_dx_pk_kernel(const bf16* __restrict__ dy,
                                                                  const bf16* __restrict__ x,
                                                                  const float* __restrict__ mean,
                                                                  const float* __restrict__ rstd,
                                                                  const bf16* __restrict__ g,
                                                                  const bf16* __restrict__ dres,
                                                                  bf16* __restrict__ dx, int cols) {
  constexpr int NT = 128;
  __shared__ float2 red[NT / 32];
  const int row = blockIdx.x;
  const int nvec = cols / 8;
  const float mu = RMS ? 0.f : mean[row], rs = rstd[row];
  const bf16* xr = x + (long long)row * cols;
  const bf16* dyr = dy + (long long)row * cols;
  uint4 xw[LN_VPT], dw[LN_VPT], rv[LN_VPT];
#pragma unroll
  for (int i = 0; i < LN_VPT; ++i) {
    const int vi = threadIdx.x + i * NT;
    if (vi < nvec) {
      xw[i] = ld_na(xr + vi * 8);
      dw[i] = ld_na(dyr + vi * 8);
      if (dres) rv[i] = ld_na(dres + (long long)row * cols + vi * 8);
    }
  }
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < LN_VPT; ++i) {
    const int vi = threadIdx.x + i * NT;
    if (vi < nvec) {
      float xv[8], dv[8], gv[8];
      unpack8(xw[i], xv);
      unpack8(dw[i], dv);
      unpack8(*reinterpret_cast<const uint4*>(g + vi * 8), gv);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float xh = (xv[j] - mu) * rs, dg = dv[j] * gv[j];
        s1 += dg;
        s2 += dg * xh;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = make_float2(s1, s2);
  __syncthreads();
  float2 t = red[0];
#pragma unroll
  for (int i = 1; i < NT / 32; ++i) { t.x += red[i].x; t.y += red[i].y; }
  const float m1 = RMS ? 0.f : t.x / cols, m2 = t.y / cols;
  bf16* dxr = dx + (long long)row * cols;
#pragma unroll
  for (int i = 0; i < LN_VPT; ++i) {
    const int vi = threadIdx.x + i * NT;
    if (vi < nvec) {
      float xv[8], dv[8], gv[8], o[8];
      unpack8(xw[i], xv);
      unpack8(dw[i], dv);
      unpack8(*reinterpret_cast<const uint4*>(g + vi * 8), gv);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float xh = (xv[j] - mu) * rs, dg = dv[j] * gv[j];
        o[j] = rs * (dg - m1 - xh * m2);
      }
      if (dres) {
        float r[8];
        unpack8(rv[i], r);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] += r[j];
      }
      *reinterpret_cast<uint4*>(dxr + vi * 8) = pack8(o);
    }
  }
}

// dx = rstd * (dy*g - mean(dy*g) - xhat * mean(dy*g*xhat)) (+ dresid); one row per block,
// the two row sums fused into a single float2 block reduction.  RMS: mean = 0 and the
// mean(dy*g) term drops (xhat = x * rstd).
template <bool RMS, int NT>
__global__ void __launch_bounds__(NT) layernorm_bwd_dx_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                                              const float* __restrict__ mean,
                                                              const float* __restrict__ rstd,
                                                              const bf16* __restrict__ g, const bf16* __restrict__ dres,
                                                              bf16* __restrict__ dx, int cols) {
  __shared__ float2 red[NT / 32];
  const int row = blockIdx.x;
  const int nvec = cols / 8;
  const float mu = RMS ? 0.f : mean[row], rs = rstd[row];
  const bf16* xr = x + (long long)row * cols;
  const bf16* dyr = dy + (long long)row * cols;
  float xh[LN_VPT][8], dg[LN_VPT][8];
  uint4 rv[LN_VPT];  // residual-gradient vectors, loaded with x / dy (more bytes in flight)
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < LN_VPT; ++i) {
    const int vi = threadIdx.x + i * NT;
    if (vi < nvec) {
      float xv[8], dv[8], gv[8];
      unpack8(*reinterpret_cast<const uint4*>(xr + vi * 8), xv);
      unpack8(*reinterpret_cast<const uint4*>(dyr + vi * 8), dv);
      unpack8(*reinterpret_cast<const uint4*>(g + vi * 8), gv);
      if (dres) rv[i] = *reinterpret_cast<const uint4*>(dres + (long long)row * cols + vi * 8);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        xh[i][j] = (xv[j] - mu) * rs;
        dg[i][j] = dv[j] * gv[j];
        s1 += dg[i][j];
        s2 += dg[i][j] * xh[i][j];
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = make_float2(s1, s2);
  __syncthreads();
  float2 t = red[0];
#pragma unroll
  for (int i = 1; i < NT / 32; ++i) { t.x += red[i].x; t.y += red[i].y; }
  const float m1 = RMS ? 0.f : t.x / cols, m2 = t.y / cols;
  bf16* dxr = dx + (long long)row * cols;
#pragma unroll
  for (int i = 0; i < LN_VPT; ++i) {
    const int vi = threadIdx.x + i * NT;
    if (vi < nvec) {
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = rs * (dg[i][j] - m1 - xh[i][j] * m2);
      if (dres) {
        float r[8];
        unpack8(rv[i], r);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] += r[j];
      }
      *reinterpret_cast<uint4*>(dxr + vi * 8) = pack8(o);
    }
  }
}

// Column reductions (deterministic, one launch):
//   LN mode : out0[c] += sum_r dy[r,c] * (x[r,c]-mean[r])*rstd[r],  out1[c] += sum_r dy[r,c]
//   SUM mode: out0[c] += sum_r dy[r,c]                               (bias gradients)
// grid = (256-column strips, row splits), sized to one wave.  Each block streams its row slab
// through a 4-stage shared-memory ring of cp.async copies: bytes in flight no longer cost
// registers -- the register-staged version kept too few loads in flight and reached 0.32 / 0.54
// of HBM (profiles/r02/ncu_colred_summary.csv).  256 threads = 32 column vectors (8 bf16) x 8
// row lanes; a thread copies exactly the 16-byte chunks it later reads (rows rl + 8i, vector
// cv), so the ring needs no block barrier -- only the thread's own cp.async group waits.  Each
// block reduces its rows in a fixed order into a workspace slot; the last block of a strip
// (atomic ticket) adds the split partials in split order to out.
constexpr int CR_MAX_SPLIT = 32;
constexpr int CR_COLS = 256;
constexpr int CR_NS = 4;  // stages
template <bool LN>
constexpr int colred_rps() {  // rows per stage: a 64 KB ring either way (LN streams two tensors)
  return LN ? 16 : 32;
}
template <bool LN>
constexpr int colred_smem() {
  return CR_NS * colred_rps<LN>() * CR_COLS * 2 * (LN ? 2 : 1);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
template <bool LN>
__global__ void __launch_bounds__(256) colred_kernel(const bf16* __restrict__ dy, long long ld,
                                                     const bf16* __restrict__ x, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, float* __restrict__ out0,
                                                     float* __restrict__ out1, float* __restrict__ ws,
                                                     unsigned* __restrict__ tickets, int rows, int cols,
                                                     int ws_ld, int accumulate) {
  constexpr int NO = LN ? 2 : 1;
  constexpr int CR_RPS = colred_rps<LN>();
  constexpr int RPT = CR_RPS / 8;             // rows per thread and stage
  constexpr int SLAB = CR_RPS * CR_COLS * 2;  // bytes of one tensor in one stage
  extern __shared__ __align__(128) uint8_t cr_smem[];
  __shared__ float sh[NO][8][CR_COLS + 4];
  __shared__ unsigned last;
  const uint32_t ring = smem_u32(cr_smem);
  const int cv = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int strip = blockIdx.x, split = blockIdx.y, nsplit = gridDim.y;
  const int c0 = strip * CR_COLS + cv * 8;
  const bool active = c0 < cols;
  const int rows_per = (rows + nsplit - 1) / nsplit;
  const int r_lo = split * rows_per, r_hi = min(rows, r_lo + rows_per);
  const int nst = r_hi > r_lo ? (r_hi - r_lo + CR_RPS - 1) / CR_RPS : 0;
  auto issue = [&](int it) {  // this thread's chunks of stage `it` into slot it % CR_NS (one group)
    if (active && it < nst) {
      const int s = it % CR_NS, r0 = r_lo + it * CR_RPS, nr = min(CR_RPS, r_hi - r0);
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int ri = rl + 8 * i;
        if (ri < nr) {
          const uint32_t off = s * SLAB + ri * CR_COLS * 2 + cv * 16;
          cp_async16(ring + off, dy + (long long)(r0 + ri) * ld + c0);
          if (LN) cp_async16(ring + CR_NS * SLAB + off, x + (long long)(r0 + ri) * cols + c0);
        }
      }
    }
    cp_async_commit();  // possibly empty: keeps the group count per stage uniform
  };
#pragma unroll
  for (int it = 0; it < CR_NS; ++it) issue(it);
  float a0[8] = {0, 0, 0, 0, 0, 0, 0, 0}, a1[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // LN: the row statistics of a stage are loaded one stage ahead (their L2 latency would
  // otherwise sit on every stage's critical path)
  float mu_n[RPT], rs_n[RPT];
  auto stats = [&](int it) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = min(r_lo + it * CR_RPS + rl + 8 * i, rows - 1);
      mu_n[i] = (LN && mean) ? __ldg(mean + r) : 0.f;
      rs_n[i] = LN ? __ldg(rstd + r) : 0.f;
    }
  };
  if (LN) stats(0);
  for (int it = 0; it < nst; ++it) {
    const int s = it % CR_NS, r0 = r_lo + it * CR_RPS, nr = min(CR_RPS, r_hi - r0);
    float mu_c[RPT], rs_c[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) mu_c[i] = mu_n[i], rs_c[i] = rs_n[i];
    if (LN && it + 1 < nst) stats(it + 1);
    cp_async_wait<CR_NS - 1>();  // stage it's group (groups complete in order)
    if (active) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int ri = rl + 8 * i;
        if (ri < nr) {
          const uint32_t off = s * SLAB + ri * CR_COLS * 2 + cv * 16;
          float d[8];
          unpack8(ld_shared_v4(ring + off), d);
          if (LN) {
            float xv[8];
            unpack8(ld_shared_v4(ring + CR_NS * SLAB + off), xv);
            const float mu = mu_c[i], rs = rs_c[i];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              a0[j] += d[j] * (xv[j] - mu) * rs;
              a1[j] += d[j];
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) a0[j] += d[j];
          }
        }
      }
    }
    issue(it + CR_NS);  // the slot this thread just read (its own chunks only)
  }
  cp_async_wait<0>();
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sh[0][rl][cv * 8 + j] = a0[j];
    if (LN) sh[NO - 1][rl][cv * 8 + j] = a1[j];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < NO * CR_COLS; idx += 256) {
    const int k = idx / CR_COLS, c = idx % CR_COLS;
    float part = 0.f;
#pragma unroll
    for (int r = 0; r < 8; ++r) part += sh[k][r][c];
    ws[((long long)split * NO + k) * ws_ld + strip * CR_COLS + c] = part;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&tickets[strip], 1u) == (unsigned)(nsplit - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int idx = threadIdx.x; idx < NO * CR_COLS; idx += 256) {
    const int k = idx / CR_COLS, c = idx % CR_COLS;
    const int col = strip * CR_COLS + c;
    if (col >= cols) continue;
    // all split partials in flight at once (L2 latency once, not nsplit times), then summed
    // in split order: same bits as a sequential loop
    float v[CR_MAX_SPLIT];
#pragma unroll
    for (int sp = 0; sp < CR_MAX_SPLIT; ++sp)
      v[sp] = sp < nsplit ? __ldcg(&ws[((long long)sp * NO + k) * ws_ld + col]) : 0.f;
    float sum = 0.f;
#pragma unroll
    for (int sp = 0; sp < CR_MAX_SPLIT; ++sp)
      if (sp < nsplit) sum += v[sp];
    float* o = k == 0 ? out0 : out1;
    if (o) o[col] = accumulate ? o[col] + sum : sum;
  }
  if (threadIdx.x == 0) tickets[strip] = 0;  // re-arm for the next launch (stream-ordered)
}

// Splits so that the grid is about one wave at the kernel's smem occupancy (2 / 3 blocks per SM),
// each split at least 32 rows.
static int colred_splits(bool ln, int rows, int strips) {
  const int per_sm = ln ? 2 : 3;  // 64 KB ring + the cross-lane buffer (16.6 / 8.3 KB) per block
  const int target = per_sm * num_sms();
  int s = target / strips;  // never more blocks than one wave: a second, short wave doubles the time
  if (s > CR_MAX_SPLIT) s = CR_MAX_SPLIT;
  while (s > 1 && rows / s < 32) --s;
  return s < 1 ? 1 : s;
}

// ----------------------------------------------------------------------------
__global__ void gelu_kernel(const bf16* __restrict__ u, bf16* __restrict__ g, long long nvec) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(u)[i], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = gelu_f(f[j]);
    reinterpret_cast<uint4*>(g)[i] = pack8(f);
  }
}

// ----------------------------------------------------------------------------
// SwiGLU (LLaMA MLP): gu [T, 2f] = [gate | up] -> a [T, f] = silu(gate) * up.
// Backward: dgate = da * up * s * (1 + gate * (1 - s)), dup = da * silu(gate), s = sigmoid(gate).
__device__ __forceinline__ float sigmoid_f(float x) { return 1.f / (1.f + __expf(-x)); }

__global__ void swiglu_fwd_kernel(const bf16* __restrict__ gu, bf16* __restrict__ a, int f, long long nvec) {
  const int fv = f / 8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / fv, c = i % fv;
    const bf16* row = gu + t * 2 * f;
    float g[8], u[8];
    unpack8(reinterpret_cast<const uint4*>(row)[c], g);
    unpack8(reinterpret_cast<const uint4*>(row + f)[c], u);
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] = g[j] * sigmoid_f(g[j]) * u[j];
    reinterpret_cast<uint4*>(a)[i] = pack8(g);
  }
}

__global__ void swiglu_bwd_kernel(const bf16* __restrict__ da, const bf16* __restrict__ gu, bf16* __restrict__ dgu,
                                  int f, long long nvec) {
  const int fv = f / 8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / fv, c = i % fv;
    const bf16* row = gu + t * 2 * f;
    float g[8], u[8], d[8], dg[8], du[8];
    unpack8(reinterpret_cast<const uint4*>(row)[c], g);
    unpack8(reinterpret_cast<const uint4*>(row + f)[c], u);
    unpack8(reinterpret_cast<const uint4*>(da)[i], d);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float sg = sigmoid_f(g[j]);
      du[j] = d[j] * g[j] * sg;
      dg[j] = d[j] * u[j] * sg * (1.f + g[j] * (1.f - sg));
    }
    bf16* orow = dgu + t * 2 * f;
    reinterpret_cast<uint4*>(orow)[c] = pack8(dg);
    reinterpret_cast<uint4*>(orow + f)[c] = pack8(du);
  }
}

// Rotary position embedding (rotate-half convention) in place on the q and k parts of
// qkv [T, 3, H, D]: for i < D/2, (x_i, x_{i+D/2}) rotates by angle pos * base^(-2i/D),
// pos = t % seq.  inverse = 1 rotates by -angle (the backward of the forward rotation).
// One thread per (token, q|k, head, 8-pair group): 16-byte loads of both halves.
__global__ void rope_kernel(bf16* __restrict__ qkv, int seq, int H, int D, float log2_base, int inverse,
                            long long nwork) {
  const int hv = D / 16;  // 8-pair groups per head
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < nwork; w += (long long)gridDim.x * blockDim.x) {
    const int grp = w % hv;
    const long long th = w / hv;           // (token, part, head)
    const int head = th % H;
    const int part = (th / H) % 2;
    const long long t = th / (2 * H);
    bf16* base = qkv + t * 3 * H * D + (long long)part * H * D + (long long)head * D;
    float lo[8], hi[8];
    unpack8(reinterpret_cast<const uint4*>(base)[grp], lo);
    unpack8(reinterpret_cast<const uint4*>(base + D / 2)[grp], hi);
    const float pos = (float)(t % seq);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = grp * 8 + j;
      const float inv_freq = exp2f(-(2.f * i / D) * log2_base);
      float sn, cs;
      sincosf(pos * inv_freq, &sn, &cs);
      if (inverse) sn = -sn;
      const float a = lo[j], b = hi[j];
      lo[j] = a * cs - b * sn;
      hi[j] = b * cs + a * sn;
    }
    reinterpret_cast<uint4*>(base)[grp] = pack8(lo);
    reinterpret_cast<uint4*>(base + D / 2)[grp] = pack8(hi);
  }
}

// ----------------------------------------------------------------------------
// Embedding: out[t] = wte[ids[t]] + wpe[t % seq]  (wpe may be null: no learned positions)
__global__ void embed_fwd_kernel(const int64_t* __restrict__ ids, const bf16* __restrict__ wte,
                                 const bf16* __restrict__ wpe, bf16* __restrict__ out, int seq, int hidden) {
  const int t = blockIdx.x;
  const long long id = ids[t];
  const bf16* e = wte + id * hidden;
  const bf16* p = wpe ? wpe + (long long)(t % seq) * hidden : nullptr;
  bf16* o = out + (long long)t * hidden;
  for (int v = threadIdx.x; v < hidden / 8; v += blockDim.x) {
    if (!p) {
      reinterpret_cast<uint4*>(o)[v] = reinterpret_cast<const uint4*>(e)[v];
      continue;
    }
    float a[8], b[8];
    unpack8(reinterpret_cast<const uint4*>(e)[v], a);
    unpack8(reinterpret_cast<const uint4*>(p)[v], b);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] += b[j];
    reinterpret_cast<uint4*>(o)[v] = pack8(a);
  }
}

// Embedding backward, deterministic (no fp32 atomics): dwte rows are owned by CTAs (a range
// of EMB_ROWS vocabulary rows each); every CTA compacts, in token order, the tokens whose id
// falls in its range and adds their gradient rows one after another (thread = column slice),
// so each row's sum order is the token order whatever the scheduling.  dwpe: one CTA per
// position sums the micro-batch's samples in order.
constexpr int EMB_ROWS = 128;
__global__ void __launch_bounds__(256) embed_bwd_wte_kernel(const int64_t* __restrict__ ids,
                                                            const bf16* __restrict__ dout, float* __restrict__ dwte,
                                                            int tokens, int hidden, int vocab) {
  extern __shared__ int match[];  // [tokens]
  __shared__ int warp_cnt[8];
  __shared__ int total;
  const int v0 = blockIdx.x * EMB_ROWS, v1 = min(vocab, v0 + EMB_ROWS);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) total = 0;
  __syncthreads();
  for (int c = 0; c < tokens; c += 256) {
    const int t = c + threadIdx.x;
    const long long id = t < tokens ? ids[t] : -1;
    const bool hit = id >= v0 && id < v1;
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (l == 0) warp_cnt[w] = __popc(bal);
    __syncthreads();
    int off = total;
    for (int i = 0; i < w; ++i) off += warp_cnt[i];
    if (hit) match[off + __popc(bal & ((1u << l) - 1u))] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      int sum = 0;
      for (int i = 0; i < 8; ++i) sum += warp_cnt[i];
      total += sum;
    }
    __syncthreads();
  }
  const int n = total;
  for (int k = 0; k < n; ++k) {
    const int t = match[k];
    float* e = dwte + ids[t] * (long long)hidden;
    const bf16* d = dout + (long long)t * hidden;
    for (int v = threadIdx.x; v < hidden / 8; v += 256) {
      float a[8];
      unpack8(reinterpret_cast<const uint4*>(d)[v], a);
      float4* ep = reinterpret_cast<float4*>(e + v * 8);
      float4 x0 = ep[0], x1 = ep[1];
      x0.x += a[0]; x0.y += a[1]; x0.z += a[2]; x0.w += a[3];
      x1.x += a[4]; x1.y += a[5]; x1.z += a[6]; x1.w += a[7];
      ep[0] = x0;
      ep[1] = x1;
    }
  }
}

__global__ void __launch_bounds__(256) embed_bwd_wpe_kernel(const bf16* __restrict__ dout, float* __restrict__ dwpe,
                                                            int tokens, int seq, int hidden) {
  const int pos = blockIdx.x;
  for (int v = threadIdx.x; v < hidden / 8; v += 256) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int t = pos; t < tokens; t += seq) {
      float a[8];
      unpack8(reinterpret_cast<const uint4*>(dout + (long long)t * hidden)[v], a);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += a[j];
    }
    float4* ep = reinterpret_cast<float4*>(dwpe + (long long)pos * hidden + v * 8);
    float4 x0 = ep[0], x1 = ep[1];
    x0.x += acc[0]; x0.y += acc[1]; x0.z += acc[2]; x0.w += acc[3];
    x1.x += acc[4]; x1.y += acc[5]; x1.z += acc[6]; x1.w += acc[7];
    ep[0] = x0;
    ep[1] = x1;
  }
}

// ----------------------------------------------------------------------------
// Fused softmax cross-entropy, one 256-thread block per row.  Pass 1: online
// max / sum-exp in fp32; pass 2: dlogits = (softmax - onehot) * scale in place.
__global__ void __launch_bounds__(256) xent_kernel(bf16* __restrict__ logits, long long ld,
                                                   const int64_t* __restrict__ labels, float* __restrict__ loss_sum,
                                                   int vocab, float scale) {
  __shared__ float sm[8], ss[8];
  const int row = blockIdx.x;
  bf16* lr = logits + (long long)row * ld;
  const int nvec = vocab / 8;
  float m = -INFINITY, s = 0.f;
  for (int v = threadIdx.x; v < nvec; v += 256) {
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(lr)[v], f);
    float bm = f[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) bm = fmaxf(bm, f[j]);
    const float nm = fmaxf(m, bm);
    float acc = s * __expf(m - nm);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += __expf(f[j] - nm);
    m = nm;
    s = acc;
  }
  // warp reduce (m, s)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
    const float nm = fmaxf(m, om);
    s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
    m = nm;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sm[w] = m; ss[w] = s; }
  __syncthreads();
  float M = sm[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) M = fmaxf(M, sm[i]);
  float S = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) S += ss[i] * __expf(sm[i] - M);
  const float lse = M + logf(S);
  const int lab = static_cast<int>(labels[row]);
  const float xl = __bfloat162float(lr[lab]);
  __syncthreads();  // everyone read lr[lab] before it is overwritten
  if (threadIdx.x == 0) atomicAdd(loss_sum, lse - xl);
  for (int v = threadIdx.x; v < nvec; v += 256) {
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(lr)[v], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float p = __expf(f[j] - lse);
      if (v * 8 + j == lab) p -= 1.f;
      f[j] = p * scale;
    }
    reinterpret_cast<uint4*>(lr)[v] = pack8(f);
  }
}

// ----------------------------------------------------------------------------
__global__ void cast_scale_kernel(const float* __restrict__ in, bf16* __restrict__ out, long long nvec, float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(in)[2 * i];
    const float4 b = reinterpret_cast<const float4*>(in)[2 * i + 1];
    const float f[8] = {a.x * scale, a.y * scale, a.z * scale, a.w * scale,
                        b.x * scale, b.y * scale, b.z * scale, b.w * scale};
    reinterpret_cast<uint4*>(out)[i] = pack8(f);
  }
}

// acc += in (fp32 wire of the gradient reduce-scatter, Runtime(rs_wire="fp32"))
__global__ void accum_f32_kernel(const float4* __restrict__ in, float4* __restrict__ acc, long long nvec) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
    const float4 x = in[i];
    float4 a = acc[i];
    a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
    acc[i] = a;
  }
}

__global__ void accum_kernel(const bf16* __restrict__ in, float* __restrict__ acc, long long nvec) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(in)[i], f);
    float4* a = reinterpret_cast<float4*>(acc) + 2 * i;
    float4 x = a[0], y = a[1];
    x.x += f[0]; x.y += f[1]; x.z += f[2]; x.w += f[3];
    y.x += f[4]; y.y += f[5]; y.z += f[6]; y.w += f[7];
    a[0] = x;
    a[1] = y;
  }
}

// torch.optim.AdamW semantics: p *= 1 - lr*wd; p -= (lr/bc1) * m / (sqrt(v)/sqrt(bc2) + eps)
__global__ void adamw_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                             const float* __restrict__ g, bf16* __restrict__ pb, long long nvec, float lr, float b1,
                             float b2, float eps, float decay, float step_size, float inv_sqrt_bc2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
    float4 P = reinterpret_cast<float4*>(p)[i], Mv = reinterpret_cast<float4*>(m)[i];
    float4 Vv = reinterpret_cast<float4*>(v)[i];
    const float4 G = reinterpret_cast<const float4*>(g)[i];
    float* pp = &P.x; float* mm = &Mv.x; float* vv = &Vv.x; const float* gg = &G.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mm[j] = b1 * mm[j] + (1.f - b1) * gg[j];
      vv[j] = b2 * vv[j] + (1.f - b2) * gg[j] * gg[j];
      pp[j] = pp[j] * decay;
      pp[j] -= step_size * mm[j] / (sqrtf(vv[j]) * inv_sqrt_bc2 + eps);
    }
    reinterpret_cast<float4*>(p)[i] = P;
    reinterpret_cast<float4*>(m)[i] = Mv;
    reinterpret_cast<float4*>(v)[i] = Vv;
    reinterpret_cast<uint2*>(pb)[i] = make_uint2(pack_bf16(P.x, P.y), pack_bf16(P.z, P.w));
  }
}

// ----------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void init_param_kernel(float* __restrict__ master, bf16* __restrict__ pb, long long n, uint64_t seed,
                                  long long offset, float mean, float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint64_t base = seed + 4ull * static_cast<uint64_t>(offset + i);
    float u[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) u[j] = static_cast<float>(splitmix64(base + j) >> 40) * 5.9604644775390625e-08f;
    float s = __fadd_rn(__fadd_rn(__fadd_rn(u[0], u[1]), u[2]), u[3]);
    s = __fsub_rn(s, 2.0f);
    const float val = __fadd_rn(mean, __fmul_rn(s, scale));
    master[i] = val;
    pb[i] = __float2bfloat16_rn(val);
  }
}

static int grid_for(long long n, int per_block) {
  long long g = (n + per_block - 1) / per_block;
  const long long cap = (long long)num_sms() * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

int kernels_preload() {
  cudaFuncAttributes fa;
  const void* fns[] = {(const void*)layernorm_fwd_kernel<false, 128>, (const void*)layernorm_bwd_dx_kernel<false, 128>,
                       (const void*)layernorm_fwd_kernel<true, 128>, (const void*)layernorm_bwd_dx_kernel<true, 128>,
                       (const void*)layernorm_fwd_kernel<false, 256>, (const void*)layernorm_bwd_dx_kernel<false, 256>,
                       (const void*)layernorm_fwd_kernel<true, 256>, (const void*)layernorm_bwd_dx_kernel<true, 256>,
                       (const void*)layernorm_bwd_dx_pk_kernel<false>, (const void*)layernorm_bwd_dx_pk_kernel<true>,
                       (const void*)swiglu_fwd_kernel, (const void*)swiglu_bwd_kernel, (const void*)rope_kernel,
                       (const void*)colred_kernel<true>, (const void*)colred_kernel<false>,
                       (const void*)gelu_kernel, (const void*)embed_fwd_kernel, (const void*)embed_bwd_wte_kernel, (const void*)embed_bwd_wpe_kernel,
                       (const void*)xent_kernel, (const void*)cast_scale_kernel, (const void*)accum_kernel, (const void*)accum_f32_kernel,
                       (const void*)adamw_kernel, (const void*)init_param_kernel};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return set_cuda_error(e, "kernels preload");
  }
  // column reductions: shared-memory ring beyond the 48 KB default
  cudaError_t e = cudaFuncSetAttribute(colred_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       colred_smem<true>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(colred_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, colred_smem<false>());
  if (e != cudaSuccess) return set_cuda_error(e, "colred smem attribute");
  return ZPP_OK;
}

}  // namespace zpp

using namespace zpp;

#define STREAM(s) reinterpret_cast<cudaStream_t>(s)

// 128 threads per row when the row fits in 4 vectors per thread, else 256
#define LN_DISPATCH(cols, KERNEL, RMSV, ...)                                                 \
  ((cols) <= 128 * 8 * LN_VPT ? (KERNEL<RMSV, 128><<<rows, 128, 0, STREAM(stream)>>>(__VA_ARGS__), 0) \
                              : (KERNEL<RMSV, 256><<<rows, 256, 0, STREAM(stream)>>>(__VA_ARGS__), 0))
#define LN_BWD_DISPATCH(cols, RMSV, ...)                                                                       \
  ((cols) <= 128 * 8 * LN_VPT                                                                                  \
       ? (layernorm_bwd_dx_pk_kernel<RMSV><<<rows, 128, 0, STREAM(stream)>>>(__VA_ARGS__), 0)                  \
       : (layernorm_bwd_dx_kernel<RMSV, 256><<<rows, 256, 0, STREAM(stream)>>>(__VA_ARGS__), 0))

extern "C" int zpp_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd,
                                 int rows, int cols, float eps, uintptr_t stream) {
  if (cols % 8 || cols > 256 * 8 * LN_VPT) return set_error(ZPP_ERR_ARG, "layernorm: cols % 8 != 0 or cols > 8192");
  if (rows <= 0) return ZPP_OK;
  LN_DISPATCH(cols, layernorm_fwd_kernel, false, (const bf16*)x, (const bf16*)gamma, (const bf16*)beta, (bf16*)y, mean,
              rstd, cols, eps);
  return check_launch("layernorm_fwd");
}

// workspace layout for the column reductions: [splits][2][cols_pad] floats + tickets
extern "C" long long zpp_layernorm_bwd_workspace_floats(int rows, int cols) {
  const int cols_pad = (cols + CR_COLS - 1) / CR_COLS * CR_COLS;
  return (long long)CR_MAX_SPLIT * 2 * cols_pad + cols_pad / CR_COLS;
}

static int colred_launch(bool ln, const void* dy, long long ld, const void* x, const float* mean, const float* rstd,
                         float* out0, float* out1, float* ws, int rows, int cols, int accumulate, cudaStream_t st) {
  const int strips = (cols + CR_COLS - 1) / CR_COLS;
  const int cols_pad = strips * CR_COLS;
  const int splits = colred_splits(ln, rows, strips);
  float* part = ws;
  unsigned* tickets = reinterpret_cast<unsigned*>(ws + (long long)CR_MAX_SPLIT * 2 * cols_pad);
  dim3 grid(strips, splits);
  if (ln)
    colred_kernel<true><<<grid, 256, colred_smem<true>(), st>>>((const bf16*)dy, ld, (const bf16*)x, mean, rstd, out0,
                                                                out1, part, tickets, rows, cols, cols_pad, accumulate);
  else
    colred_kernel<false><<<grid, 256, colred_smem<false>(), st>>>((const bf16*)dy, ld, nullptr, nullptr, nullptr,
                                                                  out0, nullptr, part, tickets, rows, cols, cols_pad,
                                                                  accumulate);
  return check_launch("colred");
}

extern "C" int zpp_layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd,
                                 const void* gamma, const void* dresid, void* dx, float* dgamma, float* dbeta,
                                 float* workspace, int rows, int cols, int accumulate, uintptr_t stream) {
  if (cols % 8 || cols > 256 * 8 * LN_VPT) return set_error(ZPP_ERR_ARG, "layernorm_bwd: cols % 8 != 0 or > 8192");
  if (!workspace && dgamma) return set_error(ZPP_ERR_ARG, "layernorm_bwd: workspace required");
  if (rows <= 0) return ZPP_OK;
  LN_BWD_DISPATCH(cols, false, (const bf16*)dy, (const bf16*)x, mean, rstd, (const bf16*)gamma,
              (const bf16*)dresid, (bf16*)dx, cols);
  int rc = check_launch("layernorm_bwd_dx");
  if (rc || !dgamma) return rc;  // dgamma == null: parameter grads via zpp_norm_param_grads
  return colred_launch(true, dy, cols, x, mean, rstd, dgamma, dbeta, workspace, rows, cols, accumulate,
                       STREAM(stream));
}

extern "C" int zpp_rmsnorm_fwd(const void* x, const void* gamma, void* y, float* rstd, int rows, int cols, float eps,
                               uintptr_t stream) {
  if (cols % 8 || cols > 256 * 8 * LN_VPT) return set_error(ZPP_ERR_ARG, "rmsnorm: cols % 8 != 0 or cols > 8192");
  if (rows <= 0) return ZPP_OK;
  LN_DISPATCH(cols, layernorm_fwd_kernel, true, (const bf16*)x, (const bf16*)gamma, nullptr, (bf16*)y, nullptr, rstd,
              cols, eps);
  return check_launch("rmsnorm_fwd");
}

extern "C" int zpp_rmsnorm_bwd(const void* dy, const void* x, const float* rstd, const void* gamma,
                               const void* dresid, void* dx, float* dgamma, float* workspace, int rows, int cols,
                               int accumulate, uintptr_t stream) {
  if (cols % 8 || cols > 256 * 8 * LN_VPT) return set_error(ZPP_ERR_ARG, "rmsnorm_bwd: cols % 8 != 0 or > 8192");
  if (!workspace && dgamma) return set_error(ZPP_ERR_ARG, "rmsnorm_bwd: workspace required");
  if (rows <= 0) return ZPP_OK;
  LN_BWD_DISPATCH(cols, true, (const bf16*)dy, (const bf16*)x, nullptr, rstd, (const bf16*)gamma,
              (const bf16*)dresid, (bf16*)dx, cols);
  int rc = check_launch("rmsnorm_bwd_dx");
  if (rc || !dgamma) return rc;
  return colred_launch(true, dy, cols, x, nullptr, rstd, dgamma, nullptr, workspace, rows, cols, accumulate,
                       STREAM(stream));
}

extern "C" int zpp_norm_param_grads(const void* dy, const void* x, const float* mean, const float* rstd,
                                    float* dgamma, float* dbeta, float* workspace, int rows, int cols, int accumulate,
                                    uintptr_t stream) {
  if (cols % 8) return set_error(ZPP_ERR_ARG, "norm_param_grads: cols % 8 != 0");
  if (!workspace || !dgamma) return set_error(ZPP_ERR_ARG, "norm_param_grads: workspace and dgamma required");
  if (rows <= 0) return ZPP_OK;
  return colred_launch(true, dy, cols, x, mean, rstd, dgamma, dbeta, workspace, rows, cols, accumulate,
                       STREAM(stream));
}

extern "C" int zpp_swiglu_fwd(const void* gu, void* a, int rows, int ffn, uintptr_t stream) {
  if (ffn % 8) return set_error(ZPP_ERR_ARG, "swiglu: ffn % 8 != 0");
  const long long nvec = (long long)rows * ffn / 8;
  if (nvec == 0) return ZPP_OK;
  swiglu_fwd_kernel<<<grid_for(nvec, 256), 256, 0, STREAM(stream)>>>((const bf16*)gu, (bf16*)a, ffn, nvec);
  return check_launch("swiglu_fwd");
}

extern "C" int zpp_swiglu_bwd(const void* da, const void* gu, void* dgu, int rows, int ffn, uintptr_t stream) {
  if (ffn % 8) return set_error(ZPP_ERR_ARG, "swiglu_bwd: ffn % 8 != 0");
  const long long nvec = (long long)rows * ffn / 8;
  if (nvec == 0) return ZPP_OK;
  swiglu_bwd_kernel<<<grid_for(nvec, 256), 256, 0, STREAM(stream)>>>((const bf16*)da, (const bf16*)gu, (bf16*)dgu,
                                                                     ffn, nvec);
  return check_launch("swiglu_bwd");
}

extern "C" int zpp_rope(void* qkv, int tokens, int seq, int heads, int head_dim, float base, int inverse,
                        uintptr_t stream) {
  if (head_dim % 16) return set_error(ZPP_ERR_ARG, "rope: head_dim % 16 != 0");
  const long long nwork = (long long)tokens * 2 * heads * (head_dim / 16);
  if (nwork == 0) return ZPP_OK;
  rope_kernel<<<grid_for(nwork, 256), 256, 0, STREAM(stream)>>>((bf16*)qkv, seq, heads, head_dim, log2f(base),
                                                                inverse, nwork);
  return check_launch("rope");
}

extern "C" int zpp_colsum_acc(const void* dy, long long ld, float* dbias, float* workspace, int rows, int cols,
                              int accumulate, uintptr_t stream) {
  if (cols % 8 || ld % 8) return set_error(ZPP_ERR_ARG, "colsum: cols / ld % 8 != 0");
  if (!workspace) return set_error(ZPP_ERR_ARG, "colsum: workspace required");
  if (rows <= 0) return ZPP_OK;
  return colred_launch(false, dy, ld, nullptr, nullptr, nullptr, dbias, nullptr, workspace, rows, cols, accumulate,
                       STREAM(stream));
}

extern "C" int zpp_gelu_fwd(const void* u, void* g, long long n, uintptr_t stream) {
  if (n % 8) return set_error(ZPP_ERR_ARG, "gelu: n % 8 != 0");
  gelu_kernel<<<grid_for(n / 8, 256), 256, 0, STREAM(stream)>>>((const bf16*)u, (bf16*)g, n / 8);
  return check_launch("gelu");
}

extern "C" int zpp_embed_fwd(const int64_t* ids, const void* wte, const void* wpe, void* out, int tokens, int seq,
                             int hidden, uintptr_t stream) {
  if (hidden % 8) return set_error(ZPP_ERR_ARG, "embed: hidden % 8 != 0");
  embed_fwd_kernel<<<tokens, 256, 0, STREAM(stream)>>>(ids, (const bf16*)wte, (const bf16*)wpe, (bf16*)out, seq, hidden);
  return check_launch("embed_fwd");
}

extern "C" int zpp_embed_bwd(const int64_t* ids, const void* dout, float* dwte, float* dwpe, int tokens, int seq,
                             int hidden, int vocab, uintptr_t stream) {
  if (hidden % 8) return set_error(ZPP_ERR_ARG, "embed_bwd: hidden % 8 != 0");
  const size_t smem = (size_t)tokens * sizeof(int);  // the CTA's ordered match list
  if (smem > 200 * 1024) return set_error(ZPP_ERR_ARG, "embed_bwd: more than 51200 tokens per call");
  static size_t smem_set = 48 * 1024;
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(embed_bwd_wte_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return set_cuda_error(e, "embed_bwd attr");
    smem_set = 200 * 1024;
  }
  embed_bwd_wte_kernel<<<(vocab + EMB_ROWS - 1) / EMB_ROWS, 256, smem, STREAM(stream)>>>(ids, (const bf16*)dout, dwte,
                                                                                       tokens, hidden, vocab);
  int rc = check_launch("embed_bwd_wte");
  if (rc || !dwpe) return rc;
  embed_bwd_wpe_kernel<<<seq, 256, 0, STREAM(stream)>>>((const bf16*)dout, dwpe, tokens, seq, hidden);
  return check_launch("embed_bwd_wpe");
}

extern "C" int zpp_xent_fwd_bwd(void* logits, long long ld, const int64_t* labels, float* loss_sum, int rows,
                                int vocab, float grad_scale, uintptr_t stream) {
  if (vocab % 8 || ld % 8) return set_error(ZPP_ERR_ARG, "xent: vocab/ld % 8 != 0");
  xent_kernel<<<rows, 256, 0, STREAM(stream)>>>((bf16*)logits, ld, labels, loss_sum, vocab, grad_scale);
  return check_launch("xent");
}

extern "C" int zpp_cast_scale_f32_bf16(const float* in, void* out, long long n, float scale, uintptr_t stream) {
  if (n % 8) return set_error(ZPP_ERR_ARG, "cast: n % 8 != 0");
  cast_scale_kernel<<<grid_for(n / 8, 256), 256, 0, STREAM(stream)>>>(in, (bf16*)out, n / 8, scale);
  return check_launch("cast_scale");
}

extern "C" int zpp_accum_bf16_f32(const void* in, float* acc, long long n, uintptr_t stream) {
  if (n % 8) return set_error(ZPP_ERR_ARG, "accum: n % 8 != 0");
  accum_kernel<<<grid_for(n / 8, 256), 256, 0, STREAM(stream)>>>((const bf16*)in, acc, n / 8);
  return check_launch("accum");
}

extern "C" int zpp_accum_f32_f32(const float* in, float* acc, long long n, uintptr_t stream) {
  if (n % 4) return set_error(ZPP_ERR_ARG, "accum_f32: n % 4 != 0");
  if (n == 0) return ZPP_OK;
  const long long nvec = n / 4;
  accum_f32_kernel<<<grid_for(nvec, 256), 256, 0, STREAM(stream)>>>(reinterpret_cast<const float4*>(in),
                                                                     reinterpret_cast<float4*>(acc), nvec);
  return check_launch("accum_f32");
}

extern "C" int zpp_adamw(float* master, float* exp_avg, float* exp_avg_sq, const float* grad, void* param_bf16,
                         long long n, float lr, float beta1, float beta2, float eps, float weight_decay, int step,
                         uintptr_t stream) {
  if (n % 4) return set_error(ZPP_ERR_ARG, "adamw: n % 4 != 0");
  if (step < 1) return set_error(ZPP_ERR_ARG, "adamw: step must be >= 1");
  const double bc1 = 1.0 - pow((double)beta1, step), bc2 = 1.0 - pow((double)beta2, step);
  adamw_kernel<<<grid_for(n / 4, 256), 256, 0, STREAM(stream)>>>(
      master, exp_avg, exp_avg_sq, grad, (bf16*)param_bf16, n / 4, lr, beta1, beta2, eps, 1.f - lr * weight_decay,
      (float)(lr / bc1), (float)(1.0 / sqrt(bc2)));
  return check_launch("adamw");
}

extern "C" int zpp_init_param(float* master, void* param_bf16, long long n, unsigned long long seed, long long offset,
                              float mean, float std, uintptr_t stream) {
  const float scale = std * 1.7320508075688772f;
  init_param_kernel<<<grid_for(n, 256), 256, 0, STREAM(stream)>>>(master, (bf16*)param_bf16, n, seed, offset, mean,
                                                                  scale);
  return check_launch("init_param");
}
