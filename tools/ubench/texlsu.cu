// Microbenchmark: does streaming global data through the TEX path (tex1Dfetch)
// relieve the L1 LSU data pipe that shared-memory table lookups saturate?
// Each warp: NL LDS.64 table lookups (16x replicated, conflict-free) per
// "tile" + streaming 3.7 KB of global codes per tile via LDG or TEX.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 1) k(const uint32_t* __restrict__ g, cudaTextureObject_t tx,
                                            size_t words_per_warp, int mode, int iters,
                                            uint32_t* out) {
  extern __shared__ uint2 tab[];
  for (int i = threadIdx.x; i < 1024 * 16; i += blockDim.x) tab[i] = make_uint2(i, i * 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t* base = g + warp * words_per_warp;
  uint32_t acc = lane, code = lane * 7919u;
  const uint32_t toff = (uint32_t)__cvta_generic_to_shared(tab) + ((lane & 15) << 3);
  for (int it = 0; it < iters; ++it) {
    // global stream: 29 words per lane per tile (like K+V codes)
    uint32_t w[29];
    const size_t t0 = (size_t)(it % 64) * 29 * 32;
    if (mode == 1) {
#pragma unroll
      for (int i = 0; i < 29; ++i) w[i] = __ldg(base + t0 + 32 * i + lane);
    } else if (mode == 2) {
#pragma unroll
      for (int i = 0; i < 29; ++i) w[i] = tex1Dfetch<uint32_t>(tx, (int)(warp * words_per_warp + t0 + 32 * i + lane));
    } else if (mode == 3) {
#pragma unroll
      for (int i = 0; i < 28; i += 4) {
        const uint4 v = tex1Dfetch<uint4>(tx, (int)((warp * words_per_warp + t0) / 4 + (i / 4) * 32 + lane));
        w[i] = v.x; w[i + 1] = v.y; w[i + 2] = v.z; w[i + 3] = v.w;
      }
      w[28] = 0;
    } else {
#pragma unroll
      for (int i = 0; i < 29; ++i) w[i] = i;
    }
    // 92 random lookups
#pragma unroll
    for (int j = 0; j < 92; ++j) {
      code = code * 1664525u + 1013904223u + w[j % 29];
      uint2 r;
      asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(toff + ((code >> 22) << 7)));
      acc += r.x ^ r.y;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const int sms = 148, threads = 256, iters = 2000;
  const size_t warps = sms * threads / 32;
  const size_t wpw = 64 * 29 * 32;  // words per warp
  const size_t nwords = warps * wpw;
  uint32_t *g, *out;
  cudaMalloc(&g, nwords * 4);
  cudaMemset(g, 1, nwords * 4);
  cudaMalloc(&out, sms * threads * 4);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = g;
  rd.res.linear.desc = cudaCreateChannelDesc<uint32_t>();
  rd.res.linear.sizeInBytes = nwords * 4;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tx, tx4;
  cudaCreateTextureObject(&tx, &rd, &td, nullptr);
  rd.res.linear.desc = cudaCreateChannelDesc<uint4>();
  cudaCreateTextureObject(&tx4, &rd, &td, nullptr);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 * 16 * 8);
  const char* names[] = {"lds only", "lds + LDG.32", "lds + TEX.32", "lds + TEX.128"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaTextureObject_t t = mode == 3 ? tx4 : tx;
    k<<<sms, threads, 1024 * 16 * 8>>>(g, t, wpw, mode, 10, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<sms, threads, 1024 * 16 * 8>>>(g, t, wpw, mode, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-14s %.3f ms  (%.1f cycles/tile/SM at 1.965 GHz, err=%s)\n", names[mode], ms,
           ms * 1e-3 * 1.965e9 / (iters * 8.0), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
