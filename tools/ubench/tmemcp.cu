// Micro-test: smem -> TMEM with tcgen05.cp.128x256b (no swizzle) and back to
// registers with tcgen05.ld.32x32b.x8; prints which smem word each TMEM
// (lane, column) received, to pin the descriptor's LBO/SBO semantics.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(uint32_t* out, uint32_t lbo, uint32_t sbo) {
  __shared__ __align__(1024) uint32_t buf[128 * 8 + 256];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 8 + 256; i += blockDim.x) buf[i] = i;  // word index
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(sa(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = taddr_s;
  if (tid == 0) {
    const uint64_t start = (sa(buf) >> 4) & 0x3FFF;
    uint64_t desc = start | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
                    ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
    if (lbo == 0) {  // 32x128b.warpx4: 32 rows x 16 B, replicated to all four lane quarters
      asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr + 8), "l"(desc));
    } else {
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(desc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
  }
  asm volatile("{\n .reg .pred p;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(sa(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[8];
  const uint32_t a = taddr + ((uint32_t)(warp * 32) << 16) + (lbo == 0 ? 8 : 0);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(a));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int j = 0; j < 8; ++j) out[(warp * 32 + lane) * 8 + j] = r[j];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(taddr));
}

int main() {
  uint32_t* d; cudaMalloc(&d, 128 * 8 * 4);
  uint32_t h[128 * 8];
  const uint32_t cfg[][2] = {{2048, 128}, {0, 128}};
  for (auto& c : cfg) {
    cudaMemset(d, 0xff, 128 * 8 * 4);
    k<<<1, 128>>>(d, c[0], c[1]);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("LBO=%u SBO=%u err=%s\n", c[0], c[1], cudaGetErrorString(e));
    for (int row : {0, 1, 8, 31, 32, 33, 64, 127}) {
      printf("  lane %3d:", row);
      for (int j = 0; j < 8; ++j) printf(" %5u", h[row * 8 + j]);
      printf("\n");
    }
  }
  return 0;
}
