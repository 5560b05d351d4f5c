// Microbenchmark: can table lookups through the texture path (tex1Dfetch of
// an 8 KB table, L1TEX cache) add lookup throughput next to conflict-free
// shared-memory LDS.64 lookups?  Per warp and step: NL LDS.64 + NT TEX
// lookups of random 8-byte entries (addresses precomputed, results consumed
// one step later); reported as warp-wide lookups per SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench/texceil.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NL, int NT>
__global__ void __launch_bounds__(256, 1) k(cudaTextureObject_t tx, int iters, uint32_t* out) {
  extern __shared__ uint2 tab[];
  for (int i = threadIdx.x; i < 1024 * 16; i += blockDim.x) tab[i] = make_uint2(i, i * 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab) + ((lane & 15) << 3);
  uint32_t a[NL > 0 ? NL : 1];
  int ti[NT > 0 ? NT : 1];
  uint32_t code = (threadIdx.x + 1) * 2654435761u;
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    code = code * 1664525u + 1013904223u;
    a[j] = base + ((code >> 20) & 255) * 128;  // 32 KB window (+ perturbation < 64 KB)
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    code = code * 1664525u + 1013904223u;
    ti[j] = (int)((code >> 20) & 1023);  // 1024-entry table, 8 KB
  }
  uint32_t acc = 0;
  uint2 rl[2][NL > 0 ? NL : 1], rt[2][NT > 0 ? NT : 1];
#pragma unroll
  for (int j = 0; j < (NL > 0 ? NL : 1); ++j) rl[1][j] = make_uint2(0, 0);
#pragma unroll
  for (int j = 0; j < (NT > 0 ? NT : 1); ++j) rt[1][j] = make_uint2(0, 0);
  for (int it = 0; it < iters; ++it) {
    // per-iteration address perturbation (one LOP3 per lookup in both paths)
    // so that nothing is loop-invariant
    const uint32_t pl = ((uint32_t)it & 63u) << 7;  // whole entries: same replica offset
    const int pt = (it & 63) << 4;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b = u & 1;
#pragma unroll
      for (int j = 0; j < NL; ++j)
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                     : "=r"(rl[b][j].x), "=r"(rl[b][j].y)
                     : "r"((a[j] ^ pl) + u * 16384));
#pragma unroll
      for (int j = 0; j < NT; ++j) rt[b][j] = tex1Dfetch<uint2>(tx, ti[j] ^ pt ^ (u * 64));
#pragma unroll
      for (int j = 0; j < NL; ++j) acc += rl[b ^ 1][j].x + rl[b ^ 1][j].y;
#pragma unroll
      for (int j = 0; j < NT; ++j) acc += rt[b ^ 1][j].x + rt[b ^ 1][j].y;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int NL, int NT>
void run(cudaTextureObject_t tx, int warps, uint32_t* out) {
  const int smem = 1024 * 16 * 8;
  cudaFuncSetAttribute(k<NL, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  k<NL, NT><<<148, warps * 32, smem>>>(tx, 10, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<NL, NT><<<148, warps * 32, smem>>>(tx, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double clk = ms * 1e-3 * 1.965e9;
  const double lk = (double)warps * iters * 4 * (NL + NT);  // warp-wide lookups per SM
  printf("LDS %2d + TEX %2d, warps %2d: %.3f ms  %.3f lookups/clk (LDS.64 alone peaks at 0.5)  (%s)\n",
         NL, NT, warps, ms, lk / clk, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint2* buf;
  cudaMalloc(&buf, 1024 * 8);
  uint2 h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = make_uint2(i, 3 * i);
  cudaMemcpy(buf, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = buf;
  rd.res.linear.desc = cudaCreateChannelDesc<uint2>();
  rd.res.linear.sizeInBytes = 1024 * 8;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tx;
  cudaCreateTextureObject(&tx, &rd, &td, nullptr);
  uint32_t* out;
  cudaMalloc(&out, 148 * 1024 * 4);
  for (int w : {8}) {
    run<16, 0>(tx, w, out);
    run<0, 16>(tx, w, out);
    run<12, 4>(tx, w, out);
    run<8, 8>(tx, w, out);
    run<14, 2>(tx, w, out);
  }
  return 0;
}
