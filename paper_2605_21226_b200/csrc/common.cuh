// common.cuh — shared device helpers for the sm_100a OCTOPUS kernels.
#pragma once
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "codec_params.h"

namespace oqd {

constexpr unsigned kFull = 0xffffffffu;

// ---- exact fp64 primitives (no FMA contraction: every op rounds once, the
// way the reference's scalar C++ does) -------------------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

// v * (+-1) is exact: flip the sign bit when `neg`.
__device__ __forceinline__ double dflip(double v, bool neg) {
  return neg ? __longlong_as_double(__double_as_longlong(v) ^ (long long)0x8000000000000000ull)
             : v;
}

// std::upper_bound count over ascending boundaries (lloydmax.hpp:46-49).
__device__ __forceinline__ uint32_t quantize_ub(const double* b, uint32_t nb, double x) {
  uint32_t lo = 0, hi = nb;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (!(x < b[mid])) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// io.hpp:115-138 f32 -> f16 RNE, bit-identical (including its NaN payload).
__device__ __forceinline__ uint16_t f32_to_f16_ref(float f) {
  const uint32_t x = __float_as_uint(f);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t ex = (x >> 23) & 0xffu;
  uint32_t man = x & 0x7fffffu;
  if (ex == 0xff) return (uint16_t)(sign | 0x7c00u | (man ? 0x200u : 0));
  const int e = (int)ex - 127 + 15;
  if (e >= 31) return (uint16_t)(sign | 0x7c00u);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    man |= 0x800000u;
    const unsigned sh = (unsigned)(14 - e);
    uint32_t half = man >> sh;
    const uint32_t rem = man & ((1u << sh) - 1u);
    const uint32_t mid = 1u << (sh - 1);
    if (rem > mid || (rem == mid && (half & 1u))) ++half;
    return (uint16_t)(sign | half);
  }
  uint32_t half = ((uint32_t)e << 10) | (man >> 13);
  const uint32_t rem = man & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (half & 1u))) ++half;
  return (uint16_t)(sign | half);
}

// Load element i of an input row in any supported dtype, widened exactly.
__device__ __forceinline__ double load_as_double(const void* p, int dtype, size_t i) {
  switch (dtype) {
    case OQ_F32: return (double)static_cast<const float*>(p)[i];
    case OQ_F64: return static_cast<const double*>(p)[i];
    case OQ_F16: return (double)__half2float(static_cast<const __half*>(p)[i]);
    default: {  // OQ_BF16
      const uint16_t b = static_cast<const uint16_t*>(p)[i];
      return (double)__uint_as_float((uint32_t)b << 16);
    }
  }
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel, device
// and size: it costs microseconds, which matters for decode-step launches.
inline cudaError_t set_smem_once(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes set
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{fn, dev}];
  if (have >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}
template <typename F>
inline cudaError_t set_smem_once(F* fn, int bytes) {
  return set_smem_once(reinterpret_cast<const void*>(fn), bytes);
}

// Fill REP consecutive shared copies of NCELL float4 cells, cell i = f(i)
// (f may read global memory): every thread first evaluates all of its cells
// (independent loads in flight together), then stores the replicas.
template <int REP, int NCELL, int PER = 8, typename F>
__device__ __forceinline__ void stage_cells(float4* dst, F f, int tid, int nthreads) {
  for (int c0 = 0; c0 < NCELL; c0 += nthreads * PER) {
    float4 v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int c = c0 + k * nthreads + tid;
      v[k] = c < NCELL ? f(c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int c = c0 + k * nthreads + tid;
      if (c < NCELL)
#pragma unroll
        for (int r = 0; r < REP; ++r) dst[c * REP + r] = v[k];
    }
  }
}

// Element size and exact fp32 widening of the input types the fast K1
// kernels accept (fp32, fp16, bf16); 16-bit elements are in the low half.
template <int DT>
struct InElem {
  static constexpr int BYTES = DT == OQ_F32 ? 4 : 2;
};
template <int DT>
__device__ __forceinline__ float widen16(uint32_t b) {
  if (DT == OQ_BF16) return __uint_as_float(b << 16);
  return __half2float(__ushort_as_half((unsigned short)b));
}
// N consecutive elements of a 16-byte-aligned shared row -> fp32 registers.
template <int DT, int N>
__device__ __forceinline__ void load_elems(float (&y)[N], const void* row, int first = 0) {
  if constexpr (DT == OQ_F32) {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
      const float4 v = reinterpret_cast<const float4*>(row)[i];
      y[first + 4 * i] = v.x;
      y[first + 4 * i + 1] = v.y;
      y[first + 4 * i + 2] = v.z;
      y[first + 4 * i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N / 8; ++i) {
      const uint4 v = reinterpret_cast<const uint4*>(row)[i];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        y[first + 8 * i + 2 * j] = widen16<DT>(w[j] & 0xffffu);
        y[first + 8 * i + 2 * j + 1] = widen16<DT>(w[j] >> 16);
      }
    }
  }
}

// Read `bits` (<= 24) starting at bit `pos` of an LSB-first byte stream.
__device__ __forceinline__ uint32_t read_bits(const uint8_t* s, uint32_t pos, uint32_t bits) {
  const uint32_t byte = pos >> 3, sh = pos & 7;
  uint32_t w = (uint32_t)s[byte] | ((uint32_t)s[byte + 1] << 8) | ((uint32_t)s[byte + 2] << 16) |
               ((uint32_t)s[byte + 3] << 24);
  return (w >> sh) & ((1u << bits) - 1u);
}

// Bounds-safe variant for global buffers: bits <= 8 touches at most 2 bytes.
__device__ __forceinline__ uint32_t read_bits_safe(const uint8_t* s, uint32_t pos, uint32_t bits) {
  const uint32_t byte = pos >> 3, sh = pos & 7;
  uint32_t w = s[byte];
  if (sh + bits > 8) w |= (uint32_t)s[byte + 1] << 8;
  return (w >> sh) & ((1u << bits) - 1u);
}

// 1-D TMA (cp.async.bulk) into shared memory completing on an mbarrier.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace oqd
