// decode.cu — K2: Encoder::decode (codec.hpp:252-275) over OCTO v1 records,
// fp32 on sm_100a.  HBM-bound: reads rec_bytes and writes 4*D bytes per key.
//
// A CTA stages a block of records in shared memory with coalesced 16-byte
// loads.  Each key is decoded by LPV lanes holding EPL contiguous output
// coordinates: the lane gathers the <= 3 triplets covering its coordinates
// (rho_hat * n_hat from fp32 tables in shared memory), runs the inverse
// rotation (WHT butterflies in registers + warp shuffles, then the sign
// flips, rotation.hpp:52-56), scales by the fp32 gamma and stores float4s.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace oqd {

template <int D>
struct DecodeShape {
  static constexpr int EPL = D >= 128 ? D / 32 : 4 < D ? 4 : D;  // elements per lane
  static constexpr int LPV = D / EPL;                               // lanes per vector (<= 32)
  static constexpr int VPW = 32 / LPV;                              // vectors per warp pass
  static constexpr int THREADS = 256;
  static constexpr int VPC = 64;  // vectors staged per CTA iteration
};

template <int D>
__global__ void __launch_bounds__(256) decode_kernel(OqCodecParams p,
                                                     const uint8_t* __restrict__ recs, size_t n,
                                                     float* __restrict__ out, int aligned) {
  using S = DecodeShape<D>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  float4* dirs_s = reinterpret_cast<float4*>(smem_raw);  // K*K
  const uint32_t kk = p.K * p.K;
  const bool dirs_in_smem = kk <= 4096;
  float* rho_s = reinterpret_cast<float*>(smem_raw + (dirs_in_smem ? kk * 16 : 0));
  uint8_t* stage = reinterpret_cast<uint8_t*>(rho_s + 256);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (dirs_in_smem)
    for (uint32_t i = tid; i < kk; i += blockDim.x)
      dirs_s[i] = reinterpret_cast<const float4*>(p.dirs32)[i];
  for (uint32_t i = tid; i < p.KR; i += blockDim.x) rho_s[i] = p.rho32[i];
  const float4* dirs = dirs_in_smem ? dirs_s : reinterpret_cast<const float4*>(p.dirs32);

  const uint32_t rb = p.rec_bytes;
  const int sub = lane % S::LPV;
  const int slot = lane / S::LPV;
  const int e0 = sub * S::EPL;
  const uint32_t smask = p.sign_mask[e0 >> 5] >> (e0 & 31);
  const float scale = (float)p.inv_sqrt_d;
  const size_t nblk = (n + S::VPC - 1) / S::VPC;

  for (size_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    __syncthreads();
    const size_t v0 = blk * S::VPC;
    const size_t nv = min((size_t)S::VPC, n - v0);
    const size_t nbytes = nv * rb;
    const uint8_t* src = recs + v0 * rb;
    if (aligned && (nbytes & 15) == 0) {
      for (size_t i = tid; i < nbytes / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(stage)[i] = reinterpret_cast<const uint4*>(src)[i];
    } else {
      for (size_t i = tid; i < nbytes; i += blockDim.x) stage[i] = src[i];
    }
    __syncthreads();
    for (int vb = warp * S::VPW; vb < (int)nv; vb += (S::THREADS / 32) * S::VPW) {
      const int vl = vb + slot;
      const bool live = vl < (int)nv;
      const uint8_t* r = stage + (live ? vl : 0) * rb;
      float y[S::EPL];
      // reconstruct_rotated for coordinates [e0, e0 + EPL)
      const int t0 = e0 / 3, t1 = (e0 + S::EPL - 1) / 3;
#pragma unroll
      for (int i = 0; i < S::EPL; ++i) y[i] = 0.f;
      constexpr int NTL = (S::EPL + 2) / 3 + 1;  // triplets that can overlap EPL coords
#pragma unroll
      for (int k = 0; k < NTL; ++k) {
        const int t = t0 + k;
        if (t <= t1) {
          const uint32_t a = read_bits(r + 4, 2 * t * p.b_dir, p.b_dir);
          const uint32_t b = read_bits(r + 4, (2 * t + 1) * p.b_dir, p.b_dir);
          const uint32_t ir = read_bits(r + 4 + p.dir_bytes, t * p.b_nrm, p.b_nrm);
          const float4 nv4 = dirs[a * p.K + b];
          const float rho = rho_s[ir];
          const float c0 = rho * nv4.x, c1 = rho * nv4.y, c2 = rho * nv4.z;
          const int rel = 3 * t - e0;  // coordinate of component 0 relative to e0
#pragma unroll
          for (int i = 0; i < S::EPL; ++i) {
            const int j = i - rel;
            if (j >= 0 && j < 3) y[i] = j == 0 ? c0 : (j == 1 ? c1 : c2);
          }
        }
      }
      // inverse rotation: y = s .* (H y) * inv_sqrt_d
#pragma unroll
      for (int len = 1; len < S::EPL; len <<= 1)
#pragma unroll
        for (int i = 0; i < S::EPL; ++i)
          if (!(i & len)) {
            const float a = y[i], b = y[i + len];
            y[i] = a + b;
            y[i + len] = a - b;
          }
#pragma unroll
      for (int lm = 1; lm < S::LPV; lm <<= 1) {
        const bool upper = sub & lm;
#pragma unroll
        for (int i = 0; i < S::EPL; ++i) {
          const float o = __shfl_xor_sync(kFull, y[i], lm);
          y[i] = upper ? o - y[i] : y[i] + o;
        }
      }
      float g;
      {
        const uint32_t gb = (uint32_t)r[0] | ((uint32_t)r[1] << 8) | ((uint32_t)r[2] << 16) |
                            ((uint32_t)r[3] << 24);
        g = __uint_as_float(gb);
      }
      const float gs = g * scale;
#pragma unroll
      for (int i = 0; i < S::EPL; ++i) {
        const float v = y[i] * gs;
        y[i] = ((smask >> i) & 1u) ? -v : v;
      }
      if (live) {
        float* o = out + (v0 + vl) * D + e0;
        if constexpr (S::EPL % 4 == 0) {
#pragma unroll
          for (int i = 0; i < S::EPL; i += 4)
            *reinterpret_cast<float4*>(o + i) = make_float4(y[i], y[i + 1], y[i + 2], y[i + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < S::EPL; ++i) o[i] = y[i];
        }
      }
    }
  }
}

template <int D>
static cudaError_t launch_decode_d(const OqCodecParams& p, const uint8_t* recs, size_t n,
                                   float* out, cudaStream_t st, int num_sms) {
  using S = DecodeShape<D>;
  const uint32_t kk = p.K * p.K;
  const size_t smem = (kk <= 4096 ? kk * 16 : 0) + 256 * 4 + S::VPC * p.rec_bytes + 16;
  cudaError_t e = cudaFuncSetAttribute(decode_kernel<D>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel<D>, S::THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const size_t nblk = (n + S::VPC - 1) / S::VPC;
  size_t grid = (size_t)per_sm * num_sms;
  if (grid > nblk) grid = nblk;
  const int aligned = (reinterpret_cast<uintptr_t>(recs) & 15) == 0;
  decode_kernel<D><<<(unsigned)grid, S::THREADS, smem, st>>>(p, recs, n, out, aligned);
  return cudaGetLastError();
}

cudaError_t launch_decode(const OqCodecParams& p, const uint8_t* recs, size_t n, float* out,
                          cudaStream_t st, int num_sms) {
  if (n == 0) return cudaSuccess;
  switch (p.dim) {
    case 4: return launch_decode_d<4>(p, recs, n, out, st, num_sms);
    case 8: return launch_decode_d<8>(p, recs, n, out, st, num_sms);
    case 16: return launch_decode_d<16>(p, recs, n, out, st, num_sms);
    case 32: return launch_decode_d<32>(p, recs, n, out, st, num_sms);
    case 64: return launch_decode_d<64>(p, recs, n, out, st, num_sms);
    case 128: return launch_decode_d<128>(p, recs, n, out, st, num_sms);
    case 256: return launch_decode_d<256>(p, recs, n, out, st, num_sms);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace oqd
