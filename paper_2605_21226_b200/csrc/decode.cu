// decode.cu — K2: Encoder::decode (codec.hpp:252-275) over OCTO v1 records,
// fp32 on sm_100a.  HBM-bound target: reads rec_bytes and writes 4*D bytes
// per key.
//
// Two kernels: decode128_kernel<b_dir, b_nrm> (d = 128 at the BASELINE bit
// splits (3,1), (4,2), (5,3): one key per thread, records double-buffered by
// TMA, see below) and the generic decode_kernel<D> for every other config.
//
// Generic: a CTA of 256 threads decodes VPC keys per iteration:
//  1. the block of records is staged in shared memory with 16-byte loads;
//  2. LPV = max(1, D/32) lanes per key each take a run of triplets, pull the
//     direction pair and norm index out of the record with two aligned word
//     loads + a funnel shift per field, look up rho_hat and n_hat (fp32
//     tables in shared memory) and write rho_hat*n_hat to a shared row
//     (reconstruct_rotated, codec.hpp:252-266);
//  3. each lane reloads EPL = D/LPV contiguous coordinates and runs the
//     inverse rotation in registers — WHT butterflies in-lane, then
//     log2(LPV) shuffle stages — scales by gamma/sqrt(d), applies the signs
//     (rotation.hpp:52-56) and writes the row back in place;
//  4. the CTA streams its contiguous block of VPC output rows to HBM with
//     coalesced 16-byte streaming stores.
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace oqd {

template <int D>
struct DecodeShape {
  static constexpr int LPV = D <= 32 ? 1 : D / 32;
  static constexpr int EPL = D / LPV;
  static constexpr int NT = (D + 2) / 3;
  static constexpr int TPL = (NT + LPV - 1) / LPV;
  static constexpr int THREADS = 256;
  static constexpr int VPC = THREADS / LPV;
  // 4-float gap after each lane chunk: the LPV lanes of a key start on
  // different banks when they write their triplets.
  __host__ __device__ static constexpr int pidx(int e) { return LPV > 1 ? e + 4 * (e / EPL) : e; }
  static constexpr int NEED = pidx(3 * NT - 1) + 1;
  // float4-aligned rows with STRIDE = 16 (mod 32) floats: the 8 lanes of an
  // LDS.128 phase (2 keys x 4 lanes) land on 8 distinct 16-byte bank groups
  static constexpr int STRIDE = ((NEED + 15) / 32) * 32 + 16;
};

// `bits` (<= 16) at absolute bit position `pos` of a word-aligned smem stream.
__device__ __forceinline__ uint32_t field(const uint32_t* s, uint32_t pos, uint32_t bits) {
  const uint32_t i = pos >> 5, sh = pos & 31;
  return __funnelshift_r(s[i], s[i + 1], sh) & ((1u << bits) - 1u);
}

constexpr int kDecRep = 8;  // direction-table replicas (lane & 7)

template <int D, bool TAB>
__global__ void __launch_bounds__(256) decode_kernel(OqCodecParams p,
                                                     const uint8_t* __restrict__ recs, size_t n,
                                                     float* __restrict__ out, int aligned,
                                                     int aligned_out) {
  using S = DecodeShape<D>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t kk = p.K * p.K;
  uint8_t* sp = smem_raw;
  float4* dirs_s = reinterpret_cast<float4*>(sp);
  if (TAB) sp += (size_t)kk * 16 * kDecRep;
  float* rho_s = reinterpret_cast<float*>(sp);
  sp += 256 * 4;
  float* rows = reinterpret_cast<float*>(sp);
  sp += (size_t)S::VPC * S::STRIDE * 4;
  uint8_t* stage = sp;  // VPC * rec_bytes (+ slack)

  const int tid = threadIdx.x, lane = tid & 31;
  if (TAB)
    for (uint32_t i = tid; i < kk * kDecRep; i += blockDim.x)
      dirs_s[i] = reinterpret_cast<const float4*>(p.dirs32)[i / kDecRep];
  for (uint32_t i = tid; i < p.KR; i += blockDim.x) rho_s[i] = p.rho32[i];
  const float4* dirs = dirs_s + (lane & (kDecRep - 1));
  uint32_t dstride = kDecRep;
  if constexpr (!TAB) {
    dirs = reinterpret_cast<const float4*>(p.dirs32);
    dstride = 1;
  }

  const int sub = S::LPV > 1 ? (lane & (S::LPV - 1)) : 0;
  const int vl = tid / S::LPV;
  const int e0 = sub * S::EPL;
  const uint32_t smask = p.sign_mask[e0 >> 5] >> (e0 & 31);
  const float scale = (float)p.inv_sqrt_d;
  const uint32_t rb = p.rec_bytes;
  const size_t nblk = (n + S::VPC - 1) / S::VPC;
  const uint32_t* stage32 = reinterpret_cast<const uint32_t*>(stage);

  for (size_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    __syncthreads();
    const size_t v0 = blk * S::VPC;
    const size_t nv = min((size_t)S::VPC, n - v0);
    const size_t nbytes = nv * rb;
    const uint8_t* src = recs + v0 * rb;
    if (aligned && (nbytes & 15) == 0) {
      for (size_t i = tid; i < nbytes / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(stage)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
    } else {
      for (size_t i = tid; i < nbytes; i += blockDim.x) stage[i] = src[i];
    }
    __syncthreads();

    const bool live = vl < (int)nv;
    float* row = rows + vl * S::STRIDE;
    float g = 0.f;
    if (live) {
      // ---- reconstruct_rotated for this lane's triplets ---------------------
      const uint32_t base = (uint32_t)vl * rb * 8;  // bit position of the record
      const uint32_t pb = 2 * p.b_dir, nbits = p.b_nrm;
      const uint32_t dpos = base + 32 + pb * sub * S::TPL;
      const uint32_t npos = base + 32 + 8 * p.dir_bytes + nbits * sub * S::TPL;
      g = __uint_as_float(field(stage32, base, 16) | (field(stage32, base + 16, 16) << 16));
      // this lane's TPL field pairs (<= 16 bits each) and norm fields as
      // word-aligned runs: 2 + TPL/2 and 1 + TPL/4 word loads, one funnel
      // shift per word, then static-position extraction
      constexpr int DW = (S::TPL * 16 + 31) / 32, NW = (S::TPL * 8 + 31) / 32;
      uint32_t dr[DW], nr[NW];
      {
        const uint32_t i0 = dpos >> 5, sh = dpos & 31;
        uint32_t prev = stage32[i0];
#pragma unroll
        for (int k = 0; k < DW; ++k) {
          const uint32_t nxt = stage32[i0 + k + 1];
          dr[k] = __funnelshift_r(prev, nxt, sh);
          prev = nxt;
        }
        const uint32_t j0 = npos >> 5, sj = npos & 31;
        prev = stage32[j0];
#pragma unroll
        for (int k = 0; k < NW; ++k) {
          const uint32_t nxt = stage32[j0 + k + 1];
          nr[k] = __funnelshift_r(prev, nxt, sj);
          prev = nxt;
        }
      }
      auto take = [](const uint32_t* w, uint32_t pos, uint32_t bits) {
        const uint32_t i = pos >> 5, sh = pos & 31;
        const uint32_t v = sh + bits <= 32 ? (w[i] >> sh) : __funnelshift_r(w[i], w[i + 1], sh);
        return v & ((1u << bits) - 1u);
      };
#pragma unroll
      for (int u = 0; u < S::TPL; ++u) {
        const int t = sub * S::TPL + u;
        if (t < S::NT) {
          const uint32_t pr = take(dr, pb * u, pb);
          const uint32_t a = pr & (p.K - 1), b = pr >> p.b_dir;
          const uint32_t ir = take(nr, nbits * u, nbits);
          const float4 nv4 = dirs[(a * p.K + b) * dstride];
          const float r = rho_s[ir];
          row[S::pidx(3 * t)] = r * nv4.x;
          if (3 * t + 1 < D) row[S::pidx(3 * t + 1)] = r * nv4.y;
          if (3 * t + 2 < D) row[S::pidx(3 * t + 2)] = r * nv4.z;
        }
      }
    }
    __syncwarp();
    // ---- inverse rotation: y = s .* (H ur) / sqrt(d), times gamma ----------
    float y[S::EPL];
#pragma unroll
    for (int i = 0; i < S::EPL; i += 4) {
      if constexpr (S::EPL % 4 == 0) {
        const float4 f = *reinterpret_cast<const float4*>(row + S::pidx(e0 + i));
        y[i] = f.x;
        y[i + 1] = f.y;
        y[i + 2] = f.z;
        y[i + 3] = f.w;
      } else {
        for (int j = i; j < S::EPL && j < i + 4; ++j) y[j] = row[S::pidx(e0 + j)];
      }
    }
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
    g = S::LPV > 1 ? __shfl_sync(kFull, g, lane & ~(S::LPV - 1)) : g;
    const float gs = g * scale;
#pragma unroll
    for (int i = 0; i < S::EPL; ++i) {
      const float v = y[i] * gs;
      y[i] = ((smask >> i) & 1u) ? -v : v;
    }
    // ---- stage the decoded row in place, then stream the block out --------
    // (a lane's 32 contiguous floats would make every warp store touch 32
    // different 512-byte keys; the block's keys are one contiguous range, so
    // the CTA writes it with fully coalesced 16-byte streaming stores)
#pragma unroll
    for (int i = 0; i < S::EPL; i += 4)
      *reinterpret_cast<float4*>(row + S::pidx(e0 + i)) = make_float4(y[i], y[i + 1], y[i + 2], y[i + 3]);
    __syncthreads();
    float* o = out + v0 * D;
    const int nf4 = (int)nv * (D / 4);
    if (aligned_out) {
      for (int f = tid; f < nf4; f += blockDim.x) {
        const int k = f / (D / 4), e = 4 * (f % (D / 4));
        __stcs(reinterpret_cast<float4*>(o) + f,
               *reinterpret_cast<const float4*>(rows + k * S::STRIDE + S::pidx(e)));
      }
    } else {
      for (int f = tid; f < nf4 * 4; f += blockDim.x) {
        const int k = f / D, e = f % D;
        o[f] = rows[k * S::STRIDE + S::pidx(e)];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// d = 128 fast path: ONE KEY PER THREAD.  The record's fields sit at
// compile-time bit positions (b_dir, b_nrm template parameters), so every
// triplet is extracted with static shifts straight into the thread's 128
// registers; the whole inverse WHT (7 butterfly stages) runs in registers
// with no shuffles, signs and gamma/sqrt(d) are folded into one multiply per
// coordinate, and each warp transposes its 32 decoded keys through shared
// memory (four 32-coordinate quarters) so that global stores are 128-byte
// segments.  Shared traffic per key: record staging, 43 direction + 43 norm
// lookups and the output transpose.
constexpr int kD128Threads = 128;            // 4 warps, 128 keys per block
constexpr int kD128HalfStride = 36;          // floats per staged quarter row (32 + 4)

template <int BD, int BN>
struct D128 {
  static constexpr int NT = 43;
  static constexpr int DIRB = (2 * NT * BD + 7) / 8, NRMB = (NT * BN + 7) / 8;
  static constexpr int BYTES = 4 + DIRB + NRMB;           // without the QJL sidecar
  static constexpr int WORDS = (BYTES + 3) / 4;           // aligned record words used
  static constexpr int NPAIR = 1 << (2 * BD), NRHO = 1 << BN;
  // direction-table replicas (lane & (REP - 1)): 8 keep the 8-lane phases of
  // LDS.128 conflict-free; at b_dir = 5 (1024 directions) 2 keep the table at
  // 32 KB so three CTAs still fit per SM
  static constexpr int REP = BD <= 4 ? 8 : 2;
};

// `bits` (<= 16) at static bit position `pos` of the thread's record words.
template <int N>
__device__ __forceinline__ uint32_t recfield(const uint32_t (&w)[N], int pos, int bits) {
  const int i = pos >> 5, sh = pos & 31;
  const uint32_t v = (sh + bits <= 32) ? (w[i] >> sh) : __funnelshift_r(w[i], w[i + 1], sh);
  return v & ((1u << bits) - 1u);
}

template <int BD, int BN>
__global__ void __launch_bounds__(kD128Threads, 3) decode128_kernel(OqCodecParams p,
                                                                 const uint8_t* __restrict__ recs,
                                                                 size_t n, float* __restrict__ out,
                                                                 int aligned) {
  using S = D128<BD, BN>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  float4* dirs_s = reinterpret_cast<float4*>(smem_raw);                // [NPAIR][S::REP]
  float* rho_s = reinterpret_cast<float*>(dirs_s + S::NPAIR * S::REP);  // [NRHO]
  float* half_s = rho_s + 16;                                           // [4 warps][32][68]
  uint64_t* bars = reinterpret_cast<uint64_t*>(half_s + 4 * 32 * kD128HalfStride);  // [2]
  uint8_t* stage0 = reinterpret_cast<uint8_t*>(bars + 2);  // 2 x [128 records], 16-aligned
  const uint32_t rb = p.rec_bytes;
  const uint32_t stage_bytes = (kD128Threads * rb + 15) & ~15u;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // direction table in field-pair order pr = ixi | ieta << b_dir
  stage_cells<S::REP, S::NPAIR>(
      dirs_s,
      [&](int pr) {
        const int a = pr & ((1 << BD) - 1), b = pr >> BD;
        return __ldg(reinterpret_cast<const float4*>(p.dirs32) + ((a << BD) | b));
      },
      tid, kD128Threads);
  for (int i = tid; i < S::NRHO; i += kD128Threads) rho_s[i] = p.rho32[i];
  const float4* dtab = dirs_s + (lane & (S::REP - 1));
  float* hs = half_s + warp * 32 * kD128HalfStride;
  const float isd = (float)p.inv_sqrt_d;
  const size_t nblk = (n + kD128Threads - 1) / kD128Threads;
  // Records of full blocks arrive by TMA, double-buffered one block ahead;
  // the (single) partial tail block is copied by the threads.
  auto full_block = [&](size_t b) { return aligned && (b + 1) * kD128Threads <= n; };
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x < nblk && full_block(blockIdx.x))
      bulk_g2s(stage0, recs + (size_t)blockIdx.x * kD128Threads * rb, kD128Threads * rb, &bars[0]);
  }

  uint32_t it = 0;
  for (size_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
    const size_t v0 = blk * kD128Threads;
    const int nv = (int)min((size_t)kD128Threads, n - v0);
    uint8_t* stage = stage0 + (it & 1) * stage_bytes;
    __syncthreads();  // every thread is done with the other buffer (and the tables are in)
    if (tid == 0) {
      const size_t nb = blk + gridDim.x;
      if (nb < nblk && full_block(nb)) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bulk_g2s(stage0 + ((it + 1) & 1) * stage_bytes, recs + nb * kD128Threads * rb,
                 kD128Threads * rb, &bars[(it + 1) & 1]);
      }
    }
    if (full_block(blk)) {
      mbar_wait(&bars[it & 1], (it >> 1) & 1);
    } else {
      const size_t nbytes = (size_t)nv * rb;
      const uint8_t* src = recs + v0 * rb;
      for (size_t i = tid; i < nbytes; i += kD128Threads) stage[i] = src[i];
      __syncthreads();
    }

    // ---- this thread's record -> 128 rotated-frame coordinates ---------------
    float y[128];
    float gs = 0.f;
    {
      uint32_t w[S::WORDS + 1];
      const uint32_t off = (uint32_t)tid * rb, wi = off >> 2, sh = 8 * (off & 3);
      const uint32_t* st32 = reinterpret_cast<const uint32_t*>(stage);
      uint32_t prev = st32[wi];
#pragma unroll
      for (int k = 0; k < S::WORDS; ++k) {
        const uint32_t nxt = st32[wi + k + 1];
        w[k] = __funnelshift_r(prev, nxt, sh);
        prev = nxt;
      }
      w[S::WORDS] = 0u;
      gs = __uint_as_float(w[0]) * isd;  // codec.hpp:273 (x float gamma), rotation.hpp:29
#pragma unroll
      for (int t = 0; t < S::NT; ++t) {
        const uint32_t pr = recfield(w, 32 + 2 * BD * t, 2 * BD);
        const uint32_t ir = recfield(w, 32 + 8 * S::DIRB + BN * t, BN);
        const float4 d4 = dtab[pr * S::REP];
        const float r = rho_s[ir];
        y[3 * t] = r * d4.x;  // reconstruct_rotated, codec.hpp:252-266
        if (3 * t + 1 < 128) y[3 * t + 1] = r * d4.y;
        if (3 * t + 2 < 128) y[3 * t + 2] = r * d4.z;
      }
    }
    // ---- inverse rotation: H y, then signs and gamma/sqrt(d) -----------------
#pragma unroll
    for (int len = 1; len < 128; len <<= 1)
#pragma unroll
      for (int i = 0; i < 128; ++i)
        if (!(i & len)) {
          const float a = y[i], b = y[i + len];
          y[i] = a + b;
          y[i + len] = a - b;
        }
#pragma unroll
    for (int i = 0; i < 128; ++i) {
      const bool neg = (p.sign_mask[i >> 5] >> (i & 31)) & 1u;  // uniform
      y[i] *= neg ? -gs : gs;
    }
    // ---- per-warp transpose through shared memory, four quarters -----------
    // (a 32-float staging row per lane keeps the block at 3 CTAs per SM)
    const int kw0 = warp * 32;  // this warp's first key in the block
    const int nkw = min(32, nv - kw0);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        *reinterpret_cast<float4*>(hs + lane * kD128HalfStride + 4 * i) =
            make_float4(y[32 * h + 4 * i], y[32 * h + 4 * i + 1], y[32 * h + 4 * i + 2],
                        y[32 * h + 4 * i + 3]);
      __syncwarp();
      // 32 keys x 8 float4 of this quarter: lane -> (key = it*4 + lane/8, f4 = lane%8)
      if (nkw > 0) {
        float* ob = out + (v0 + kw0) * 128 + 32 * h;
#pragma unroll 4
        for (int it = 0; it < 8; ++it) {
          const int k = 4 * it + (lane >> 3), f = lane & 7;
          if (k < nkw) {
            const float4 v = *reinterpret_cast<const float4*>(hs + k * kD128HalfStride + 4 * f);
            __stcs(reinterpret_cast<float4*>(ob + (size_t)k * 128) + f, v);
          }
        }
      }
      __syncwarp();
    }
  }
}

template <int BD, int BN>
static cudaError_t launch_decode128(const OqCodecParams& p, const uint8_t* recs, size_t n,
                                   float* out, cudaStream_t st, int num_sms) {
  using S = D128<BD, BN>;
  const size_t smem = (size_t)S::NPAIR * S::REP * 16 + 16 * 4 + 4 * 32 * kD128HalfStride * 4 +
                      16 + 2 * (((size_t)kD128Threads * p.rec_bytes + 15) & ~size_t(15)) + 64;
  cudaError_t e = set_smem_once(decode128_kernel<BD, BN>, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode128_kernel<BD, BN>,
                                                    kD128Threads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const size_t nblk = (n + kD128Threads - 1) / kD128Threads;
  size_t grid = (size_t)per_sm * num_sms;
  if (grid > nblk) grid = nblk;
  const int aligned = (reinterpret_cast<uintptr_t>(recs) & 15) == 0;
  decode128_kernel<BD, BN><<<(unsigned)grid, kD128Threads, smem, st>>>(p, recs, n, out, aligned);
  return cudaGetLastError();
}

template <int D, bool TAB>
static cudaError_t launch_decode_dt(const OqCodecParams& p, const uint8_t* recs, size_t n,
                                    float* out, cudaStream_t st, int num_sms) {
  using S = DecodeShape<D>;
  const uint32_t kk = p.K * p.K;
  const size_t smem = (TAB ? kk * 16 * kDecRep : 0) + 256 * 4 +
                      (size_t)S::VPC * S::STRIDE * 4 + (size_t)S::VPC * p.rec_bytes + 64;
  cudaError_t e = set_smem_once(decode_kernel<D, TAB>, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel<D, TAB>, S::THREADS,
                                                    smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const size_t nblk = (n + S::VPC - 1) / S::VPC;
  size_t grid = (size_t)per_sm * num_sms;
  if (grid > nblk) grid = nblk;
  const int aligned = (reinterpret_cast<uintptr_t>(recs) & 15) == 0;
  const int aligned_out = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  decode_kernel<D, TAB><<<(unsigned)grid, S::THREADS, smem, st>>>(p, recs, n, out, aligned,
                                                                  aligned_out);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_decode_d(const OqCodecParams& p, const uint8_t* recs, size_t n,
                                   float* out, cudaStream_t st, int num_sms) {
  return p.K * p.K <= 1024 ? launch_decode_dt<D, true>(p, recs, n, out, st, num_sms)
                           : launch_decode_dt<D, false>(p, recs, n, out, st, num_sms);
}

cudaError_t launch_decode(const OqCodecParams& p, const uint8_t* recs, size_t n, float* out,
                          cudaStream_t st, int num_sms) {
  if (n == 0) return cudaSuccess;
  static const bool generic_only = getenv("OQ_DECODE_GENERIC") != nullptr;  // comparison runs
  if (p.dim == 128 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 && !generic_only) {
    if (p.b_dir == 3 && p.b_nrm == 1) return launch_decode128<3, 1>(p, recs, n, out, st, num_sms);
    if (p.b_dir == 4 && p.b_nrm == 2) return launch_decode128<4, 2>(p, recs, n, out, st, num_sms);
    if (p.b_dir == 5 && p.b_nrm == 3) return launch_decode128<5, 3>(p, recs, n, out, st, num_sms);
  }
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
