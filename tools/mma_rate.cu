// Microbenchmark: raw tcgen05.mma throughput (smem operands, no TMA / epilogue).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2402_03791_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace zpp;

template <int CG, int N, int COMMIT, bool AMN = false, bool BMN = false, bool TS = false>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); mbar_init(smem_u32(&bar2), 1 << 20); fence_mbar_init(); }
  if (warp == 0) { if (CG == 2) tmem_alloc2(smem_u32(&tslot), 512); else tmem_alloc(smem_u32(&tslot), 512); }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const bool leader = (CG == 1) || cluster_rank() == 0;
  if (threadIdx.x == 0 && leader) {
    constexpr uint32_t idesc = make_idesc_bf16(128 * CG, N, AMN, BMN);
    const uint64_t ad = make_sdesc(base, AMN ? 8192 : 16, 1024), bd = make_sdesc(base + 16384, BMN ? 8192 : 16, 1024);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ka = AMN ? (uint64_t)(128 * k) : (uint64_t)(2 * k), kb = BMN ? (uint64_t)(128 * k) : (uint64_t)(2 * k);
        if (CG == 2) mma_bf16_2sm(tmem, ad + ka, bd + kb, idesc, 1u);
        else if (TS) mma_bf16_ts(tmem, tmem + 256 + 8 * k, bd + kb, idesc, 1u);
        else mma_bf16(tmem, ad + ka, bd + kb, idesc, 1u);
      }
      if (COMMIT == 1) { if (CG == 2) mma_commit_2sm(smem_u32(&bar2), 0x3); else mma_commit(smem_u32(&bar2)); }
      if (COMMIT == 2) { if (CG == 2) mma_commit_2sm(smem_u32(&bar2), 0x1); else mma_commit(smem_u32(&bar2)); }
    }
    if (CG == 2) mma_commit_2sm(smem_u32(&bar), 0x3); else mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  if (CG == 2 && !leader && threadIdx.x == 0) mbar_wait(smem_u32(&bar), 0);
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) { if (CG == 2) tmem_dealloc2(tmem, 512); else tmem_dealloc(tmem, 512); }
}

// whole-warp issue with elect.sync (uniform descriptors), 8 K-steps per iteration
template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_loop_w(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, false, false);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t bd = make_sdesc(base + 16384 + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024);
        if (TS) mma_bf16_ts_w(tmem, tmem + 256 + 8 * (k & 3), bd, idesc, 1u);
        else mma_bf16_w(tmem, make_sdesc(base + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024), bd, idesc, 1u);
      }
    }
    mma_commit_w(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int N, bool TS>
void run_w(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  auto k = mma_loop_w<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 1024;
  k<<<148, 128, 64 * 1024>>>(16, d);
  k<<<148, 128, 64 * 1024>>>(iters, d);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("%-22s %s  %.1f cycles/MMA-instr (floor %d)\n", name, cudaGetErrorString(err), double(cyc) / (iters * 8),
         128 * N / 256);
}

template <int CG, int N, int COMMIT, bool AMN = false, bool BMN = false, bool TS = false>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  auto k = mma_loop<CG, N, COMMIT, AMN, BMN, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 64 * 1024;
  cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = CG; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a; cfg.numAttrs = 1;
  const int iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k, 16, d);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  double macs_per_sm = double(iters) * 4 * 128 * N * 16;  // per SM (each SM owns 128 rows)
  printf("%-22s %s  %.1f cycles/MMA-instr, %.0f MACs/cycle/SM, %.1f TFLOP/s chip\n", name, cudaGetErrorString(err),
         double(cyc) / (iters * 4), macs_per_sm / cyc, 2.0 * macs_per_sm * 148 / (ms * 1e-3) / 1e12);
}


// the dK/dV kernel's per-tile MMA mix: S^T, dP^T (TS, N=64, K=128) + dV, dK (SS, N=128, K=64)
template <int SYNC>
__global__ void __launch_bounds__(128, 1) mma_mix(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, cb[4], done;
  __shared__ uint32_t tslot;
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&cb[i]), 1 << 20);  // never completes: commits only
    mbar_init(smem_u32(&done), 1);
    mbar_arrive(smem_u32(&done));  // phase 0 complete: waits on it return at once
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  auto sync_point = [&](int k) {
    if (SYNC >= 1) mma_commit_w(smem_u32(&cb[k]));
    if (SYNC >= 2) { mbar_wait(smem_u32(&done), 0); tc_fence_after(); }
  };
  if (warp == 0) {
    constexpr uint32_t id_sp = make_idesc_bf16(128, 64, false, false);
    constexpr uint32_t id_kv = make_idesc_bf16(128, 128, false, true);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_bf16_ts_w(tmem + 384, tmem + 256 + kk * 8, make_sdesc(base + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024),
                      id_sp, kk > 0);
      sync_point(0);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_bf16_ts_w(tmem + 448, tmem + 320 + kk * 8, make_sdesc(base + 16384 + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024),
                      id_sp, kk > 0);
      sync_point(1);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16_w(tmem, make_sdesc(base + 32768 + kk * 32, 16, 1024), make_sdesc(base + kk * 2048, 8192, 1024), id_kv, 1);
      sync_point(2);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16_w(tmem + 128, make_sdesc(base + 49152 + kk * 32, 16, 1024), make_sdesc(base + 16384 + kk * 2048, 8192, 1024),
                   id_kv, 1);
      sync_point(3);
    }
    mma_commit_w(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int SYNC>
void run_mix() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mma_mix<SYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int iters = 512;
  mma_mix<SYNC><<<148, 128, 96 * 1024>>>(16, d);
  mma_mix<SYNC><<<148, 128, 96 * 1024>>>(iters, d);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("dkdv tile mix (16 TS N64 + 8 SS N128), sync %d  %s  %.1f cycles/tile (floor 1024)\n", SYNC,
         cudaGetErrorString(err), double(cyc) / iters);
}


// dQ-kernel round: dQ += dS K (TS, A = TMEM buffer X, N=128, 4 x K16), then S = Q K^T and
// dP = dO V^T (TS, N=64, 8 x K16 each) written into buffer Y.  WAR = Y is the buffer dQ read.
template <bool WAR>
__global__ void __launch_bounds__(128, 1) mma_dq_round(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    constexpr uint32_t id_s = make_idesc_bf16(128, 64, false, false);
    constexpr uint32_t id_q = make_idesc_bf16(128, 128, false, true);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t x = (i & 1) * 64;                       // dS buffer read by dQ
      const uint32_t y = WAR ? x : ((i + 1) & 1) * 64;       // buffer S / dP are written into
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16_ts_w(tmem + 256, tmem + x + (kk >> 1) * 32 + (kk & 1) * 8, make_sdesc(base + kk * 2048, 8192, 1024),
                      id_q, 1);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_bf16_ts_w(tmem + y, tmem + 384 + kk * 8, make_sdesc(base + 16384 + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024),
                      id_s, kk > 0);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_bf16_ts_w(tmem + 128 + y, tmem + 448 + kk * 8,
                      make_sdesc(base + 32768 + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
    }
    mma_commit_w(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <bool WAR>
void run_dq_round() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mma_dq_round<WAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int iters = 512;
  mma_dq_round<WAR><<<148, 128, 96 * 1024>>>(16, d);
  mma_dq_round<WAR><<<148, 128, 96 * 1024>>>(iters, d);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("dq round (4 TS N128 + 16 TS N64), S/dP over the dS buffer dQ just read: %d  %s  %.1f cycles (floor 768)\n",
         (int)WAR, cudaGetErrorString(err), double(cyc) / iters);
}

int main() {
  run<2, 256, 1, false, false>("cta2 K/K");
  run<2, 256, 1, false, true>("cta2 K/MN");
  run<2, 256, 1, true, true>("cta2 MN/MN");
  run<1, 256, 1, true, true>("cta1 MN/MN");
  run<1, 256, 0>("cta1 N256 SS K/K");
  run<1, 128, 0>("cta1 N128 SS K/K");
  run<1, 64, 0>("cta1 N64 SS K/K");
  run<1, 32, 0>("cta1 N32 SS K/K");
  run<1, 128, 0, false, true>("cta1 N128 SS K/MN");
  run<1, 128, 0, false, true, true>("cta1 N128 TS K/MN");
  run<1, 64, 0, false, false, true>("cta1 N64 TS K/K");
  run<1, 32, 0, false, false, true>("cta1 N32 TS K/K");
  run<1, 256, 0, false, true, true>("cta1 N256 TS K/MN");
  run_w<64, false>("warp N64 SS");
  run_w<64, true>("warp N64 TS");
  run_w<32, true>("warp N32 TS");
  run_w<32, false>("warp N32 SS");
  run_w<128, false>("warp N128 SS");
  run_mix<0>();
  run_dq_round<false>();
  run_dq_round<true>();
  return 0;
}
