// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput vs. number of warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2402_03791_b200/csrc tmem_rate.cu -o tmem_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace zpp;

__device__ __forceinline__ void ld64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]),
        "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]),
        "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
        "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),
        "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}

template <int X>
__global__ void tmem_ld_loop(int iters, unsigned long long* cycles, float* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  float acc = 0.f;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t col = ((i * 64 + (warp >> 2) * 128) & 511);
    if (X == 32) {
      uint32_t v[32];
      tmem_ld32(tm + (col & 480), v);
      tmem_wait_ld();
      acc += __uint_as_float(v[0]) + __uint_as_float(v[31]);
    } else {
      uint32_t v[64];
      ld64(tm + (col & 448), v);
      tmem_wait_ld();
      acc += __uint_as_float(v[0]) + __uint_as_float(v[63]);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tslot, 512);
}

template <int X>
void run(int warps) {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4);
  const int iters = 4096;
  tmem_ld_loop<X><<<148, warps * 32>>>(16, d, sink);
  tmem_ld_loop<X><<<148, warps * 32>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = double(iters) * warps * 32 * X * 4;
  printf("x%-3d warps %2d: %s  %.1f cycles per load per warp, %.1f B/cycle/SM\n", X, warps, cudaGetErrorString(e),
         double(cyc) / iters, bytes / cyc);
}

int main() {
  for (int w : {4, 8, 16}) run<32>(w);
  for (int w : {4, 8, 16}) run<64>(w);
  return 0;
}
