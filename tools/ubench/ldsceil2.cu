// Microbenchmark: shared-memory lookup throughput with NO per-lookup ALU
// work (ldsceil.cu computes each address with ~5 ALU ops, which can make it
// ALU- or latency-bound at low warp counts).  Each lane holds NF
// precomputed conflict-free addresses; every iteration issues NF LDS with
// immediate offsets into NF distinct result registers that are never read
// (asm volatile keeps them), so the only limits are the LSU/crossbar and the
// write-after-write wait on a result register NF lookups later.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench/ldsceil2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int VEC, int NF>
__global__ void k(int iters, uint32_t* out) {
  extern __shared__ uint4 tab[];
  for (int i = threadIdx.x; i < 1024 * 8; i += blockDim.x) tab[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab);
  const uint32_t rep = (lane & (VEC == 4 ? 7 : VEC == 2 ? 15 : 31)) * (VEC * 4);
  uint32_t a[NF];
  uint32_t code = (threadIdx.x + 1) * 2654435761u;
#pragma unroll
  for (int j = 0; j < NF; ++j) {
    code = code * 1664525u + 1013904223u;
    a[j] = base + rep + ((code >> 20) & 511) * 128;  // 64 KB window; +imm stays inside 128 KB
  }
  // two register sets: the loads of step u are issued before the results of
  // step u-1 are consumed (one IADD3 per lookup keeps ptxas from deleting them)
  uint32_t r[2][NF][VEC];
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < NF; ++j)
#pragma unroll
    for (int v = 0; v < VEC; ++v) r[1][j][v] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b = u & 1;
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const uint32_t ad = a[j] + u * 16384;
        if (VEC == 1)
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r[b][j][0]) : "r"(ad));
        else if (VEC == 2)
          asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                       : "=r"(r[b][j][0]), "=r"(r[b][j][VEC > 1 ? 1 : 0])
                       : "r"(ad));
        else
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(r[b][j][0]), "=r"(r[b][j][VEC > 1 ? 1 : 0]),
                         "=r"(r[b][j][VEC > 2 ? 2 : 0]), "=r"(r[b][j][VEC > 3 ? 3 : 0])
                       : "r"(ad));
      }
#pragma unroll
      for (int j = 0; j < NF; ++j)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc += r[b ^ 1][j][v];
    }
  }
#pragma unroll
  for (int j = 0; j < NF; ++j) acc += r[1][j][0];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int VEC, int NF>
void run(int warps) {
  uint32_t* out;
  cudaMalloc(&out, 148 * 1024 * 4);
  const int smem = 1024 * 8 * 16;
  cudaFuncSetAttribute(k<VEC, NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  k<VEC, NF><<<148, warps * 32, smem>>>(10, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<VEC, NF><<<148, warps * 32, smem>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double lds = (double)warps * iters * 4 * NF;  // warp-wide LDS per SM
  const double wf = lds * VEC;                       // 128-B wavefronts (conflict-free)
  const double clk = ms * 1e-3 * 1.965e9;
  printf("LDS.%-3d warps %2d in-flight %2d: %.3f ms  %.3f wavefronts/clk  %.2f cyc/LDS  (%s)\n",
         32 * VEC, warps, NF, ms, wf / clk, clk / lds, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 12, 16, 32}) {
    run<1, 16>(w);
    run<2, 8>(w);
    run<2, 16>(w);
    run<2, 32>(w);
    run<4, 16>(w);
  }
  return 0;
}
