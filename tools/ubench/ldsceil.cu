// Microbenchmark: practical ceiling of conflict-free random shared-memory
// lookups (the K3 dequant table pattern) on one SM: L1 wavefronts per clock
// for LDS.32 / LDS.64 / LDS.128 at 8 / 16 / 32 warps per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int VEC>
__global__ void k(int iters, uint32_t* out) {
  extern __shared__ uint4 tab[];
  for (int i = threadIdx.x; i < 1024 * 8; i += blockDim.x) tab[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // replica layout: entry e, replica r at byte e * 32 * VEC*4... keep 16 replicas of VEC*4 bytes
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab);
  const uint32_t rep = (lane & (VEC == 4 ? 7 : VEC == 2 ? 15 : 31)) * (VEC * 4);
  const uint32_t stride = VEC == 4 ? 128 : VEC == 2 ? 128 : 128;
  const uint32_t nent = (1024 * 8 * 16) / stride;
  uint32_t acc = 0, code = lane * 2654435761u;
  for (int it = 0; it < iters; ++it) {
    uint32_t c[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = (code >> (j & 15)) ^ (j * 0x9e3779b9u);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t a = base + rep + ((c[j] & (nent - 1)) * stride);
      if (VEC == 1) {
        uint32_t r;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
        acc += r;
      } else if (VEC == 2) {
        uint2 r;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(a));
        acc += r.x ^ r.y;
      } else {
        uint4 r;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
        acc += r.x ^ r.y ^ r.z ^ r.w;
      }
    }
    code = code * 1664525u + 1013904223u + acc;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int VEC>
void run(int warps) {
  uint32_t* out;
  cudaMalloc(&out, 148 * 1024 * 4);
  const int smem = 1024 * 8 * 16;
  cudaFuncSetAttribute(k<VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  k<VEC><<<148, warps * 32, smem>>>(10, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<VEC><<<148, warps * 32, smem>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double wf = (double)warps * iters * 16 * VEC;  // wavefronts per SM (VEC*4*32/128)
  const double clk = ms * 1e-3 * 1.965e9;
  printf("LDS.%-3d warps %2d: %.3f ms  %.3f wavefronts/clk  (%s)\n", 32 * VEC, warps, ms, wf / clk,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16, 32}) { run<1>(w); run<2>(w); run<4>(w); }
  return 0;
}
