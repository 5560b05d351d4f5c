// compress.cu — K1: fused OCTOPUS compress (Encoder::encode, codec.hpp:214-249)
// on sm_100a, bit-exact against the fp64 CPU reference.
//
// A CTA of 128 threads encodes VPC keys per iteration in four phases:
//  A. rotation, LPV = max(1, D/32) lanes per key with EPL = D/LPV contiguous
//     fp64 elements each: sequential norm, normalize, sign flips and WHT in
//     registers (in-lane butterflies, then warp shuffles); the rotated
//     coordinates go to shared memory;
//  B. joint rounding, ONE THREAD PER TRIPLET over all VPC*n_tri triplets:
//     octahedral fold and upper-bound bucketing in exact fp64; the 3x3 (or
//     2x2 / full) window is pre-screened in fp32 and the winner is certified
//     when it beats the runner-up by more than 1e-6 (the fp32 score error is
//     below 3e-7 for |t| <= 1), in which case only the winner's dot product is
//     recomputed in exact fp64 for the norm bucket; near-ties replay the
//     reference's exact strict-'>' scan;
//  C. (QJL) residual norm and second rotation, LPV lanes per key again;
//  D. byte-parallel OCTO v1 record assembly (codec.hpp:381-393) in shared
//     memory, then coalesced 32-bit stores.
// Every fp64 op that can influence a code is an explicitly rounded __d*_rn
// intrinsic in the reference's evaluation order, so codes are bit-exact
// (SURVEY.md §7 H1).  The grid is persistent, so codebook tables are staged
// into shared memory once per CTA.
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "encode_exact.cuh"

namespace oqd {

template <int D>
struct CompressShape {
  static constexpr int LPV = D <= 32 ? 1 : D / 32;
  static constexpr int EPL = D / LPV;
  static constexpr int NT = (D + 2) / 3;
  static constexpr int TPL = (NT + LPV - 1) / LPV;  // triplets per lane
  static constexpr int THREADS = 128;
  static constexpr int VPC = THREADS / LPV;          // vectors per CTA
  // padded element index: a 4-double gap after each lane chunk keeps the
  // 16 lanes of a half-warp on distinct 8-byte banks.
  __host__ __device__ static constexpr int pidx(int e) { return LPV > 1 ? e + 4 * (e / EPL) : e; }
  static constexpr int NEED = pidx(3 * NT - 1) + 1;
  static constexpr int STRIDE = LPV > 1 ? ((NEED + 14) / 16) * 16 + 1 : (NEED | 1);
};

// Vectorized row load of EPL contiguous elements, widened exactly to fp64.
template <int EPL>
__device__ __forceinline__ void load_row(double (&xv)[EPL], const void* x, int dtype, size_t off,
                                         bool live) {
  if (!live) {
#pragma unroll
    for (int i = 0; i < EPL; ++i) xv[i] = 0.0;
    return;
  }
  if (dtype == OQ_F32 && EPL % 4 == 0) {
    const float4* p4 = reinterpret_cast<const float4*>(static_cast<const float*>(x) + off);
#pragma unroll
    for (int i = 0; i < EPL / 4; ++i) {
      const float4 f = __ldg(p4 + i);
      xv[4 * i] = f.x;
      xv[4 * i + 1] = f.y;
      xv[4 * i + 2] = f.z;
      xv[4 * i + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < EPL; ++i) xv[i] = load_as_double(x, dtype, off + i);
  }
}

// ---- in-register rotation: y = H (s .* x) * inv_sqrt_d (rotation.hpp:46-49)
template <int D>
__device__ __forceinline__ void rotate_exact(double (&x)[CompressShape<D>::EPL], uint32_t smask,
                                             int sub, double scale) {
  using S = CompressShape<D>;
#pragma unroll
  for (int i = 0; i < S::EPL; ++i) {  // x * (+-1) is exact: XOR the sign bit
    const uint32_t flip = (i < 31 ? smask << (31 - i) : smask >> (i - 31)) & 0x80000000u;
    x[i] = __hiloint2double(__double2hiint(x[i]) ^ (int)flip, __double2loint(x[i]));
  }
#pragma unroll
  for (int len = 1; len < S::EPL; len <<= 1) {
#pragma unroll
    for (int i = 0; i < S::EPL; ++i)
      if (!(i & len)) {
        const double a = x[i], b = x[i + len];
        x[i] = dadd(a, b);
        x[i + len] = dsub(a, b);
      }
  }
#pragma unroll
  for (int lm = 1; lm < S::LPV; lm <<= 1) {
    const bool upper = sub & lm;
#pragma unroll
    for (int i = 0; i < S::EPL; ++i) {
      const double o = __shfl_xor_sync(kFull, x[i], lm);
      // element j (lower lane) pairs with j+len (upper lane): (a+b, a-b)
      x[i] = upper ? dsub(o, x[i]) : dadd(x[i], o);
    }
  }
#pragma unroll
  for (int i = 0; i < S::EPL; ++i) x[i] = dmul(x[i], scale);
}

// Sequential sum of squares over the whole vector, in element order
// (codec.hpp:219-220 / qjl.hpp:28-29): the chain walks lane 0..LPV-1.
template <int D>
__device__ __forceinline__ double seq_sumsq(const double (&x)[CompressShape<D>::EPL], int sub,
                                            int lane) {
  using S = CompressShape<D>;
  double sq[S::EPL];  // exact squares in parallel; only the adds are serial
#pragma unroll
  for (int i = 0; i < S::EPL; ++i) sq[i] = dmul(x[i], x[i]);
  double run = 0.0;
#pragma unroll
  for (int L = 0; L < S::LPV; ++L) {
    if (sub == L) {
#pragma unroll
      for (int i = 0; i < S::EPL; ++i) run = dadd(run, sq[i]);
    }
    if (S::LPV > 1) run = __shfl_sync(kFull, run, (lane & ~(S::LPV - 1)) + L);
  }
  return run;
}

// TAB: codebook tables staged in shared memory (K^2 <= 1024, i.e. b_dir <= 5);
// otherwise they are read from global memory (L1-cached).
// list != nullptr: encode only the keys list[0 .. *list_n) (the fast path's
// flagged keys), each record written at its own key's slot.
template <int D, bool TAB>
__global__ void __launch_bounds__(128) compress_kernel(OqCodecParams p, const void* __restrict__ x,
                                                       int dtype, size_t n,
                                                       uint8_t* __restrict__ out, int aligned,
                                                       const uint32_t* __restrict__ list,
                                                       const uint32_t* __restrict__ list_n,
                                                       int list_stride) {
  using S = CompressShape<D>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int sub = S::LPV > 1 ? (lane & (S::LPV - 1)) : 0;
  const int vl = tid / S::LPV;  // vector slot within the CTA

  // ---- carve shared memory ------------------------------------------------
  uint8_t* sp = smem_raw;
  double* ur_s = reinterpret_cast<double*>(sp);
  sp += sizeof(double) * S::VPC * S::STRIDE;
  double* xb_s = reinterpret_cast<double*>(sp);
  sp += sizeof(double) * 256;
  double* rb_s = reinterpret_cast<double*>(sp);
  sp += sizeof(double) * 256;
  double* rc_s = reinterpret_cast<double*>(sp);
  sp += sizeof(double) * 256;
  const uint32_t kk = p.K * p.K;
  constexpr bool dirs_in_smem = TAB;
  double* dirs_s = reinterpret_cast<double*>(sp);
  if (dirs_in_smem) sp += sizeof(double) * 3 * kk;
  float4* d32_s = reinterpret_cast<float4*>(sp);
  if (dirs_in_smem) sp += sizeof(float4) * kk;
  uint32_t* xlut_s = reinterpret_cast<uint32_t*>(sp);
  sp += 4096;
  uint32_t* rlut_s = reinterpret_cast<uint32_t*>(sp);
  sp += 4096;
  float* gam_s = reinterpret_cast<float*>(sp);
  sp += sizeof(float) * S::VPC;
  uint32_t* sgn_s = reinterpret_cast<uint32_t*>(sp);  // QJL: D/32 words (>=1) per vector
  constexpr int SGW = D >= 32 ? D / 32 : 1;
  sp += sizeof(uint32_t) * S::VPC * SGW;
  uint16_t* gr_s = reinterpret_cast<uint16_t*>(sp);
  sp += sizeof(uint16_t) * S::VPC;
  uint16_t* dcode_s = reinterpret_cast<uint16_t*>(sp);  // [VPC][2*NT]
  sp += sizeof(uint16_t) * S::VPC * 2 * S::NT;
  uint8_t* ncode_s = sp;  // [VPC][NT]
  sp += S::VPC * S::NT;
  sp = smem_raw + (((sp - smem_raw) + 15) & ~15);  // keep the shared address space
  uint8_t* stage_s = sp;  // [VPC * rec_bytes]

  for (uint32_t i = tid; i < p.K - 1; i += blockDim.x) xb_s[i] = p.xi_bnd[i];
  for (uint32_t i = tid; i < p.KR - 1; i += blockDim.x) rb_s[i] = p.rho_bnd[i];
  for (uint32_t i = tid; i < p.KR; i += blockDim.x) rc_s[i] = p.rho_c[i];
  if (dirs_in_smem) {
    for (uint32_t i = tid; i < 3 * kk; i += blockDim.x) dirs_s[i] = p.dirs64[i];
    for (uint32_t i = tid; i < kk; i += blockDim.x)
      d32_s[i] = reinterpret_cast<const float4*>(p.dirs32)[i];
  }
  for (int c = tid; c < 1024; c += blockDim.x) {
    xlut_s[c] = p.xi_lut[c];
    rlut_s[c] = p.rho_lut[c];
  }
  __syncthreads();
  const double* dirs64 = dirs_s;
  const float4* dirs32 = d32_s;
  if constexpr (!TAB) {
    dirs64 = p.dirs64;
    dirs32 = reinterpret_cast<const float4*>(p.dirs32);
  }
  CompressSmem sm{xb_s, rb_s, rc_s, dirs64, xlut_s, rlut_s};

  const uint32_t smask = p.sign_mask[(sub * S::EPL) >> 5] >> ((sub * S::EPL) & 31);
  const uint32_t qmask = p.qsign_mask[(sub * S::EPL) >> 5] >> ((sub * S::EPL) & 31);
  if (list) n = *list_n;
  const size_t nblocks = (n + S::VPC - 1) / S::VPC;
  const uint32_t rb = p.rec_bytes;

  for (size_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    const size_t v = blk * S::VPC + vl;
    const bool live = v < n;
    const size_t key = list ? (live ? (size_t)list[v * list_stride] : 0) : v;
    double* ur = ur_s + vl * S::STRIDE;

    // ---- load, norm, normalize (codec.hpp:219-225) ------------------------
    double xv[S::EPL];
    load_row<S::EPL>(xv, x, dtype, key * D + sub * S::EPL, live);
    const double g2 = seq_sumsq<D>(xv, sub, lane);
    const double gamma = dsqrt(g2);
    const double inv = ddiv(1.0, gamma > 1e-12 ? gamma : 1e-12);
#pragma unroll
    for (int i = 0; i < S::EPL; ++i) xv[i] = dmul(xv[i], inv);
    // ---- rotate (codec.hpp:227) -------------------------------------------
    rotate_exact<D>(xv, smask, sub, p.inv_sqrt_d);
#pragma unroll
    for (int i = 0; i < S::EPL; ++i) ur[S::pidx(sub * S::EPL + i)] = xv[i];
    if (sub == S::LPV - 1)  // zero pad to 3 * n_tri (codec.hpp:229-230)
      for (int e = D; e < 3 * S::NT; ++e) ur[S::pidx(e)] = 0.0;
    if (sub == 0) gam_s[vl] = (float)gamma;  // codec.hpp:233 (double -> float RN)
    __syncthreads();

    // ---- B: per-triplet joint rounding, one thread per triplet ------------
    // (codec.hpp:236-241; QJL residual r = ur - rho n_hat, codec.hpp:243-246)
    const int ntask = (int)min((size_t)S::VPC, n - blk * S::VPC) * S::NT;
    for (int task = tid; task < ntask; task += blockDim.x) {
      const int w = task / S::NT, t = task - w * S::NT;
      double* uw = ur_s + w * S::STRIDE;
      const double t0 = uw[S::pidx(3 * t)], t1 = uw[S::pidx(3 * t + 1)],
                   t2 = uw[S::pidx(3 * t + 2)];
      const uint32_t code = joint_round(p, sm, dirs32, t0, t1, t2);
      // the triplet's 2*b_dir-bit direction field pair, ixi | ieta << b_dir
      dcode_s[w * 2 * S::NT + t] = (uint16_t)((code & 0xff) | (((code >> 8) & 0xff) << p.b_dir));
      ncode_s[w * S::NT + t] = (uint8_t)(code >> 16);
      if (p.qjl) {
        const uint32_t a = code & 0xff, b = (code >> 8) & 0xff, ir = code >> 16;
        const double* nv = sm.dirs + 3 * (a * p.K + b);
        const double r = sm.rc[ir];
        const double tt[3] = {t0, t1, t2};
#pragma unroll
        for (int j = 0; j < 3; ++j)
          if (3 * t + j < D) uw[S::pidx(3 * t + j)] = dsub(tt[j], dmul(r, nv[j]));
      }
    }
    __syncthreads();

    if (p.qjl) {
      // ---- C: QJL epilogue (qjl.hpp:23-36), LPV lanes per key ---------------
#pragma unroll
      for (int i = 0; i < S::EPL; ++i) xv[i] = ur[S::pidx(sub * S::EPL + i)];
      const double n2 = seq_sumsq<D>(xv, sub, lane);
      rotate_exact<D>(xv, qmask, sub, p.inv_sqrt_d);
      uint32_t bits = 0;
#pragma unroll
      for (int i = 0; i < S::EPL; ++i) bits |= (xv[i] >= 0.0 ? 1u : 0u) << i;
      if (S::EPL >= 32) sgn_s[vl * SGW + sub] = bits;
      else sgn_s[vl * SGW] = bits;
      if (sub == 0) gr_s[vl] = f32_to_f16_ref((float)dsqrt(n2));
    }
    __syncthreads();

    // ---- D: OCTO record assembly (codec.hpp:381-393), word-parallel --------
    // Task (key, k): k = 0 writes gamma (+ the QJL bytes); k in [1, dw] builds
    // 32-bit word k-1 of the direction stream from the <= 6 triplet field
    // pairs overlapping it; the rest build the norm stream words.  Streams
    // are LSB-first with zero padding (io.hpp:66-85).
    const size_t nv = min((size_t)S::VPC, n - blk * S::VPC);
    {
      const int dw = (p.dir_bytes + 3) >> 2, nw = (p.nrm_bytes + 3) >> 2, per = 1 + dw + nw;
      const int pb = 2 * p.b_dir, nb = p.b_nrm;
      for (int task = tid; task < (int)nv * per; task += blockDim.x) {
        const int w = task / per, k = task - w * per;
        uint8_t* rec = stage_s + w * rb;
        if (k == 0) {
          const uint32_t gb = __float_as_uint(gam_s[w]);
#pragma unroll
          for (int j = 0; j < 4; ++j) rec[j] = (uint8_t)(gb >> (8 * j));
          if (p.qjl) {
            uint8_t* q = rec + 4 + p.dir_bytes + p.nrm_bytes;
            q[0] = (uint8_t)gr_s[w];
            q[1] = (uint8_t)(gr_s[w] >> 8);
            for (int j = 0; j < ((D + 7) >> 3); ++j)
              q[2 + j] = (uint8_t)(sgn_s[w * SGW + (j >> 2)] >> (8 * (j & 3)));
          }
          continue;
        }
        const bool dir = k <= dw;
        const int wi = dir ? k - 1 : k - 1 - dw, bits = dir ? pb : nb;
        const int b0 = 32 * wi;
        const int t0 = b0 / bits, t1 = min((b0 + 31) / bits, S::NT - 1);
        uint32_t word = 0;
        for (int t = t0; t <= t1; ++t) {
          const uint32_t c = dir ? (uint32_t)dcode_s[w * 2 * S::NT + t] : (uint32_t)ncode_s[w * S::NT + t];
          const int sh = t * bits - b0;
          word |= sh >= 0 ? (c << sh) : (c >> -sh);
        }
        const int off = dir ? 4 + 4 * wi : 4 + p.dir_bytes + 4 * wi;
        const int nbytes = min(4, (dir ? (int)p.dir_bytes : (int)p.nrm_bytes) - 4 * wi);
        for (int j = 0; j < nbytes; ++j) rec[off + j] = (uint8_t)(word >> (8 * j));
      }
    }
    __syncthreads();
    const size_t nbytes = nv * rb;
    uint8_t* dst = out + blk * S::VPC * (size_t)rb;
    if (list) {
      for (size_t i = tid; i < nbytes; i += blockDim.x) {
        const size_t w = i / rb;
        out[(size_t)list[(blk * S::VPC + w) * list_stride] * rb + (i - w * rb)] = stage_s[i];
      }
    } else if (aligned) {
      const uint32_t* src32 = reinterpret_cast<const uint32_t*>(stage_s);
      uint32_t* dst32 = reinterpret_cast<uint32_t*>(dst);
      for (size_t i = tid; i < nbytes / 4; i += blockDim.x) dst32[i] = src32[i];
      for (size_t i = (nbytes / 4) * 4 + tid; i < nbytes; i += blockDim.x) dst[i] = stage_s[i];
    } else {
      for (size_t i = tid; i < nbytes; i += blockDim.x) dst[i] = stage_s[i];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Small batches (a decode step compresses one key per (batch, kv head)
// stream): one warp per key, latency first (encode_key_warp).
constexpr int kSmallWarps = 4;

__global__ void __launch_bounds__(32 * kSmallWarps) compress_small_kernel(
    OqCodecParams p, const void* __restrict__ x, int dtype, size_t n, uint8_t* __restrict__ out) {
  __shared__ double row_s[kSmallWarps][132];
  __shared__ uint32_t rec_s[kSmallWarps][kRecWords];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const size_t key = blockIdx.x * (size_t)kSmallWarps + wib;
  if (key >= n) return;
  encode_key_warp(p, x, dtype, key, row_s[wib], rec_s[wib], lane);
  if (p.qjl) qjl_key_warp(p, row_s[wib], rec_s[wib], lane, global_tables(p));
  const uint32_t rb = p.rec_bytes;
  uint8_t* dst = out + key * rb;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(rec_s[wib]);
  for (uint32_t b = lane; b < rb; b += 32) dst[b] = src[b];
}

// ---------------------------------------------------------------------------
// Exact fixup of the certified fp32 pass (compress_fast.cu).  Per round a CTA
// takes 16 warps x kFixKeys flagged keys: each warp recomputes its keys'
// reference fp64 rotated coordinates from the stored exact inv
// (rotate_key_warp) and queues the flagged triplets (3 doubles + key + t) in
// shared memory; then every thread re-rounds one queued triplet exactly
// (joint_round: a long dependent chain, so the triplets of many keys run
// side by side instead of one lane per key) and patches its direction-pair
// and norm fields into the record in place — the pass masks every field to
// its width, so the other fields are already final.  Records of different
// keys may share a 32-bit word, hence atomic clear + set on disjoint bits.
// 4 CTAs per SM in the (persistent, strided) grid: b = 3 fixup 518 -> 510 us
// for the whole compress (A/B; b = 2 +0.8 %, b = 4 unchanged; 8 keys per
// warp-round, 4 warps, 6 or 8 CTAs per SM were no better)
constexpr int kFixWarps = 8, kFixKeys = 16, kFixQ = 896, kFixCtasPerSm = 4;

struct FixTriplet {
  double t0, t1, t2;
  uint32_t key, t;
};

__device__ __forceinline__ void patch_field(uint32_t* words, size_t pos, int bits, uint32_t v) {
  const size_t w = pos >> 5;
  const int sh = (int)(pos & 31);
  const uint32_t m = (1u << bits) - 1u;
  atomicAnd(&words[w], ~(m << sh));
  atomicOr(&words[w], (v & m) << sh);
  if (sh + bits > 32) {
    const int hi = sh + bits - 32;
    atomicAnd(&words[w + 1], ~((1u << hi) - 1u));
    atomicOr(&words[w + 1], (v & m) >> (bits - hi));
  }
}

__device__ __forceinline__ void fix_triplet(const OqCodecParams& p, const CompressSmem& tabs,
                                            const float4* d32, uint32_t* words, const FixTriplet& q) {
  const uint32_t code = joint_round(p, tabs, d32, q.t0, q.t1, q.t2);
  const uint32_t pr = (code & 0xff) | (((code >> 8) & 0xff) << p.b_dir), ir = code >> 16;
  const size_t base = (size_t)8 * q.key * p.rec_bytes;
  const int pb = 2 * p.b_dir, nb = p.b_nrm;
  patch_field(words, base + 32 + (size_t)pb * q.t, pb, pr);
  patch_field(words, base + 32 + 8 * (size_t)p.dir_bytes + (size_t)nb * q.t, nb, ir);
}

__global__ void __launch_bounds__(32 * kFixWarps, 2) compress_fixup_kernel(
    OqCodecParams p, const void* __restrict__ x, int dtype, uint8_t* __restrict__ out,
    const FlagEntry* __restrict__ flags, const uint32_t* __restrict__ flag_cnt) {
  extern __shared__ __align__(128) uint8_t fix_stage[];  // [kFixWarps][kFixKeys][row bytes]
  __shared__ double row_s[kFixWarps][132];
  __shared__ FixTriplet queue[kFixQ];
  __shared__ uint32_t qn;
  __shared__ __align__(8) uint64_t bars[kFixWarps];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t n = *flag_cnt;
  const uint32_t rbytes = 128u * (dtype == OQ_F32 ? 4u : 2u);
  uint8_t* stage = fix_stage + (size_t)wib * kFixKeys * rbytes;
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[wib]);
  {
    // warm this SM's L1 with the codebook tables: joint_round's lookups form
    // a dependent chain that would otherwise pay an L2 round trip per step
    const uint32_t kk = p.K * p.K;
    auto pf = [](const void* a) { asm volatile("prefetch.global.L1 [%0];" ::"l"(a)); };
    for (uint32_t l = threadIdx.x; l < (kk * 16 + 127) / 128; l += blockDim.x)
      pf(reinterpret_cast<const uint8_t*>(p.dirs32) + 128 * l);
    for (uint32_t l = threadIdx.x; l < (kk * 24 + 127) / 128; l += blockDim.x)
      pf(reinterpret_cast<const uint8_t*>(p.dirs64) + 128 * l);
    for (uint32_t l = threadIdx.x; l < 32; l += blockDim.x) {
      pf(reinterpret_cast<const uint8_t*>(p.xi_lut) + 128 * l);
      pf(reinterpret_cast<const uint8_t*>(p.rho_lut) + 128 * l);
    }
    if (threadIdx.x == 0) {
      pf(p.xi_bnd);
      pf(p.rho_bnd);
      pf(p.rho_c);
      qn = 0;
    }
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  const CompressSmem tabs = global_tables(p);
  const float4* d32 = reinterpret_cast<const float4*>(p.dirs32);
  uint32_t* words = reinterpret_cast<uint32_t*>(out);
  // keys per warp and round: as many as the list allows up to kFixKeys, so
  // short lists still spread over every warp
  const size_t nwarps = (size_t)gridDim.x * kFixWarps;
  const int kpw = (int)min((size_t)kFixKeys, max((size_t)1, (n + nwarps - 1) / nwarps));
  const size_t per_cta = (size_t)kFixWarps * kpw;
  uint32_t phase = 0;
  for (size_t e0 = blockIdx.x * per_cta; e0 < n; e0 += (size_t)gridDim.x * per_cta) {
    // ---- this warp's keys: flag entries, then their rows by 1-D TMA ------
    const size_t w0 = e0 + (size_t)wib * kpw;
    const int nk = (int)min((size_t)kpw, w0 < n ? n - w0 : (size_t)0);
    FlagEntry f{};
    if (lane < nk) f = flags[w0 + lane];
    if (nk > 0) {
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"(nk * rbytes)
                     : "memory");
      __syncwarp();
      if (lane < nk)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"((uint32_t)__cvta_generic_to_shared(stage + lane * rbytes)),
            "l"(static_cast<const uint8_t*>(x) + (size_t)f.key * rbytes), "r"(rbytes), "r"(bar)
            : "memory");
      asm volatile(
          "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          " @!p bra W_%=;\n}" ::"r"(bar),
          "r"(phase)
          : "memory");
      phase ^= 1u;
    }
    // ---- rotations; flagged triplets -> the queue ---------------------------
#pragma unroll 1
    for (int j = 0; j < nk; ++j) {
      const uint32_t key = __shfl_sync(kFull, f.key, j), mlo = __shfl_sync(kFull, f.mlo, j),
                     mhi = __shfl_sync(kFull, f.mhi, j);
      const double inv = __shfl_sync(kFull, f.inv, j);
      double k[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) k[i] = load_as_double(stage + j * rbytes, dtype, 4 * lane + i);
      rotate_key_warp(p, k, inv, row_s[wib], lane);
      const double* row = row_s[wib];
      for (int t = lane; t < 43; t += 32) {
        if (!(((t < 32 ? mlo >> t : mhi >> (t - 32))) & 1u)) continue;
        const FixTriplet q{row[3 * t], row[3 * t + 1], row[3 * t + 2], key, (uint32_t)t};
        const uint32_t slot = atomicAdd(&qn, 1u);
        if (slot < kFixQ) queue[slot] = q;
        else fix_triplet(p, tabs, d32, words, q);  // queue full: decide it here
      }
      __syncwarp();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staging reused by TMA
    __syncthreads();
    // ---- decisions: one queued triplet per thread -------------------------
    const uint32_t m = min(qn, (uint32_t)kFixQ);
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) fix_triplet(p, tabs, d32, words, queue[i]);
    __syncthreads();
    if (threadIdx.x == 0) qn = 0;
    __syncthreads();
  }
}

cudaError_t launch_compress_fixup(const OqCodecParams& p, const void* x, int dtype, uint8_t* out,
                                  const FlagEntry* flags, const uint32_t* flag_cnt,
                                  cudaStream_t st, int num_sms) {
  // the count lives on the device: a fixed persistent grid strides over it
  const int sm = kFixWarps * kFixKeys * 128 * 4;
  cudaError_t e = set_smem_once(compress_fixup_kernel, sm);
  if (e != cudaSuccess) return e;
  compress_fixup_kernel<<<kFixCtasPerSm * num_sms, 32 * kFixWarps, sm, st>>>(p, x, dtype, out, flags,
                                                                            flag_cnt);
  return cudaGetLastError();
}

// Whole-key exact re-encode of the keys the certified pass flagged, one warp
// per key (used with the QJL sidecar, whose residual depends on every code).
__global__ void __launch_bounds__(32 * kSmallWarps) compress_rekey_kernel(
    OqCodecParams p, const void* __restrict__ x, int dtype, uint8_t* __restrict__ out,
    const FlagEntry* __restrict__ flags, const uint32_t* __restrict__ flag_cnt) {
  __shared__ double row_s[kSmallWarps][132];
  __shared__ uint32_t rec_s[kSmallWarps][kRecWords];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t n = *flag_cnt;
  const uint32_t rb = p.rec_bytes;
  for (size_t i = blockIdx.x * (size_t)kSmallWarps + wib; i < n;
       i += (size_t)gridDim.x * kSmallWarps) {
    const size_t key = flags[i].key;
    encode_key_warp(p, x, dtype, key, row_s[wib], rec_s[wib], lane);
    if (p.qjl) qjl_key_warp(p, row_s[wib], rec_s[wib], lane, global_tables(p));
    uint8_t* dst = out + key * rb;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(rec_s[wib]);
    for (uint32_t b = lane; b < rb; b += 32) dst[b] = src[b];
    __syncwarp();
  }
}

template <int D>
static size_t compress_smem(const OqCodecParams& p) {
  using S = CompressShape<D>;
  const uint32_t kk = p.K * p.K;
  size_t b = sizeof(double) * S::VPC * S::STRIDE + 3 * sizeof(double) * 256;
  if (kk <= 1024) b += sizeof(double) * 3 * kk + sizeof(float4) * kk;
  b += 8192;
  b += sizeof(float) * S::VPC + sizeof(uint32_t) * S::VPC * (D >= 32 ? D / 32 : 1) +
       sizeof(uint16_t) * S::VPC + sizeof(uint16_t) * S::VPC * 2 * S::NT + S::VPC * S::NT;
  b = (b + 15) & ~size_t(15);
  b += (size_t)S::VPC * p.rec_bytes + 16;
  return b;
}

template <int D, bool TAB>
static cudaError_t launch_compress_dt(const OqCodecParams& p, const void* x, int dtype, size_t n,
                                     uint8_t* out, cudaStream_t st, int num_sms,
                                     const uint32_t* list, const uint32_t* list_n,
                                     int list_stride) {
  using S = CompressShape<D>;
  const size_t smem = compress_smem<D>(p);
  cudaError_t e = set_smem_once(compress_kernel<D, TAB>, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, compress_kernel<D, TAB>, S::THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const size_t nblocks = (n + S::VPC - 1) / S::VPC;  // list mode: n = capacity
  size_t grid = (size_t)per_sm * num_sms;
  if (grid > nblocks) grid = nblocks;
  const int aligned = (reinterpret_cast<uintptr_t>(out) & 3) == 0;
  compress_kernel<D, TAB><<<(unsigned)grid, S::THREADS, smem, st>>>(p, x, dtype, n, out, aligned,
                                                                    list, list_n, list_stride);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_compress_d(const OqCodecParams& p, const void* x, int dtype, size_t n,
                                     uint8_t* out, cudaStream_t st, int num_sms,
                                     const uint32_t* list = nullptr,
                                     const uint32_t* list_n = nullptr, int list_stride = 1) {
  return p.K * p.K <= 1024
             ? launch_compress_dt<D, true>(p, x, dtype, n, out, st, num_sms, list, list_n,
                                           list_stride)
             : launch_compress_dt<D, false>(p, x, dtype, n, out, st, num_sms, list, list_n,
                                            list_stride);
}

cudaError_t launch_compress(const OqCodecParams& p, const void* x, int dtype, size_t n,
                            uint8_t* out, cudaStream_t st, int num_sms, uint32_t* flagged) {
  if (n == 0) return cudaSuccess;
  // d = 128 fp32 / fp16 / bf16 keys at the BASELINE bit splits (scalar or
  // local3x3): up to 2048 keys one warp per key (exact), up to 8192 the
  // single-pass two-lanes-per-key kernel (compress_x2.cu), beyond that the
  // certified fp32 pass + the exact fixup of its undecided triplets (or, with
  // QJL, of its flagged keys).  Every other config: the generic exact kernel.
  // OQ_COMPRESS_IMPL=x (x2 only) / e (generic only) select a kernel for
  // comparison runs.
  static const int impl = [] {
    const char* e = getenv("OQ_COMPRESS_IMPL");
    if (!e) return 1;
    return e[0] == 'x' ? 0 : (e[0] == 'e' ? 2 : 1);
  }();
  // small batches (a decode step appends B*Hkv keys): one warp per key,
  // exact, one launch, no table staging
  if (impl == 1 && n <= 2048 && p.dim == 128) {
    cudaError_t e = flagged ? cudaMemsetAsync(flagged, 0, sizeof(uint32_t), st) : cudaSuccess;
    if (e == cudaSuccess) {
      compress_small_kernel<<<(unsigned)((n + kSmallWarps - 1) / kSmallWarps), 32 * kSmallWarps, 0,
                              st>>>(p, x, dtype, n, out);
      e = cudaGetLastError();
    }
    return e;
  }
  if (impl == 1 && n <= 8192 && !p.qjl && compress_fast_ok(p, dtype, x, out)) {
    cudaError_t e = flagged ? cudaMemsetAsync(flagged, 0, sizeof(uint32_t), st) : cudaSuccess;
    if (e == cudaSuccess) e = launch_compress_x2(p, x, dtype, n, out, st, num_sms);
    return e;
  }
  if (impl == 0 && !p.qjl && compress_fast_ok(p, dtype, x, out)) {
    cudaError_t e = flagged ? cudaMemsetAsync(flagged, 0, sizeof(uint32_t), st) : cudaSuccess;
    if (e == cudaSuccess)
      e = launch_compress_x2(p, x, dtype, n, out, st, num_sms);
    return e;
  }
  if (impl == 1 && compress_fast_ok(p, dtype, x, out)) {
    // certified fp32 pass, then the exact re-rounding of the triplets it
    // could not decide
    uint32_t* ws = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws), 32 + n * sizeof(FlagEntry), st);
    if (e != cudaSuccess) return e;
    FlagEntry* fl = reinterpret_cast<FlagEntry*>(ws + 8);
    e = cudaMemsetAsync(ws, 0, sizeof(uint32_t), st);
    if (e == cudaSuccess) e = launch_compress_fast(p, x, dtype, n, out, fl, ws, st, num_sms);
    // with the QJL sidecar a flagged key is re-encoded whole, one warp per
    // key (its residual depends on every triplet's codes)
    if (e == cudaSuccess) {
      if (p.qjl) {
        compress_rekey_kernel<<<num_sms * 16, 32 * kSmallWarps, 0, st>>>(p, x, dtype, out, fl, ws);
        e = cudaGetLastError();
      } else {
        e = launch_compress_fixup(p, x, dtype, out, fl, ws, st, num_sms);
      }
    }
    if (e == cudaSuccess && flagged)
      e = cudaMemcpyAsync(flagged, ws, sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
    const cudaError_t f = cudaFreeAsync(ws, st);
    return e != cudaSuccess ? e : f;
  }
  if (flagged) {
    cudaError_t e = cudaMemsetAsync(flagged, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
  }
  switch (p.dim) {
    case 4: return launch_compress_d<4>(p, x, dtype, n, out, st, num_sms);
    case 8: return launch_compress_d<8>(p, x, dtype, n, out, st, num_sms);
    case 16: return launch_compress_d<16>(p, x, dtype, n, out, st, num_sms);
    case 32: return launch_compress_d<32>(p, x, dtype, n, out, st, num_sms);
    case 64: return launch_compress_d<64>(p, x, dtype, n, out, st, num_sms);
    case 128: return launch_compress_d<128>(p, x, dtype, n, out, st, num_sms);
    case 256: return launch_compress_d<256>(p, x, dtype, n, out, st, num_sms);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace oqd
