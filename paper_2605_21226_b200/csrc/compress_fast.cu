// compress_fast.cu — K1 fast path: Encoder::encode (codec.hpp:214-249) for
// d = 128, fp32 / fp16 / bf16 keys, scalar / local3x3 rounding, no QJL, at the BASELINE bit
// splits (3,1), (4,2), (5,3).  ONE KEY PER THREAD, certified fp32:
//
//  * each warp owns 32 consecutive keys; every lane pulls its 512-byte row
//    into a padded shared-memory row with a 1-D TMA bulk copy (mbarrier per
//    warp), the next block's rows are requested as soon as the current ones
//    sit in registers;
//  * gamma is the reference's sequential fp64 sum of squares, replayed
//    exactly (the fp32 squares are exact in fp64, so fma(k, k, s) == s + k*k)
//    and stored as float(gamma) (codec.hpp:219-233);
//  * the rotation runs in fp32 registers (signs, 7-stage WHT, one scale by
//    float(inv / sqrt(d))).  Its error against the reference's fp64 rotated
//    coordinates is bounded in L2 over the whole vector: each of the 7
//    butterfly stages adds <= u |v_s| (u = 2^-24), |v_s| = 2^((s+1)/2) |k|,
//    and the later stages grow it by 2^((6-s)/2), so after the scale by
//    1/(gamma sqrt d) the butterflies contribute <= 7u, the scale <= 2u per
//    coordinate: for a triplet ||t32 - t64|| <= Et = 7.01u + 2.01u ||t||
//    (see DESIGN.md §2);
//  * every decision of the triplet encoder — octahedral hemisphere and
//    signs (octahedral.hpp:22-31), the xi/eta bucket (lloydmax.hpp:46-49),
//    the 3x3 argmax (codec.hpp:164-189) and the norm bucket — is taken in
//    fp32 and CERTIFIED: it must clear its decision boundary by more than the
//    propagated error bound, otherwise the key is flagged;
//  * a triplet whose decisions miss a margin is marked in the key's 43-bit
//    mask; flagged keys (mask, exact fp64 inv) are appended to a list and
//    only their marked triplets are re-rounded afterwards in exact fp64 and
//    patched into the record (compress.cu, compress_fixup_kernel), so every
//    record is bit-identical to the reference; the flagged key count is
//    reported.
//  * records are assembled in registers at compile-time bit positions,
//    merged across lanes at shared word boundaries with one shuffle, and the
//    warp's 32 records leave with one TMA bulk store.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace oqd {

#ifndef OQ_CF_NW5
#define OQ_CF_NW5 8
#endif
#ifndef OQ_CF_DREP5
#define OQ_CF_DREP5 2
#endif
constexpr int kCFRow = 132;  // floats per staged row (128 + 4 pad: conflict-free LDS.128)
constexpr int kCFCells = 128, kCFLutRep = 8;  // LUT: float4 entries, 8 replicas

template <int BD, int BN, bool QJL = false>
struct CFS {
  static constexpr int K = 1 << BD, KR = 1 << BN, NT = 43;
  static constexpr int DIRB = (2 * NT * BD + 7) / 8, NRMB = (NT * BN + 7) / 8;
  static constexpr int QB = 4 + DIRB + NRMB;            // QJL sidecar offset
  static constexpr int RB = QB + (QJL ? 18 : 0);        // record bytes
  static constexpr int RW = (RB + 3) / 4;               // record words
  // the QJL variants give up direction-table replicas for the larger records
  static constexpr int DREP = QJL ? (BD <= 4 ? 4 : 1) : (BD <= 4 ? 8 : OQ_CF_DREP5);
  // warps per CTA (one CTA per SM): fewer at b_dir = 5 leave room for more
  // direction-table replicas (bank conflicts of the 3x3 window lookups)
  static constexpr int NW = (BD >= 5 && !QJL) ? OQ_CF_NW5 : 8;
  static constexpr int RECBUF_WORDS = (32 * RB) / 4 + 4;
  // shared memory carve (bytes)
  static constexpr int KP = K + 2;  // direction grid padded by a -inf border
  static constexpr int DIRS_BYTES = KP * KP * DREP * 16;
  static constexpr int LUT_BYTES = kCFCells * kCFLutRep * 16;
  static constexpr int BND_BYTES = 64 * 4;
  static constexpr int ROWS_BYTES = NW * 32 * kCFRow * 4;
  static constexpr int RECB_BYTES = NW * RECBUF_WORDS * 4;
  static constexpr int SCR_BYTES = NW * 32 * (RW + 1) * 4;  // per-lane record words
  static constexpr int SMEM =
      DIRS_BYTES + LUT_BYTES + BND_BYTES + ROWS_BYTES + RECB_BYTES + SCR_BYTES + 64;
};

__device__ __forceinline__ uint32_t cf_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Bucket of x among the xi boundaries = std::upper_bound count
// (lloydmax.hpp:46-49), certified when x clears both bracketing boundaries by
// more than g.  One LDS.128 per lookup: cell c of [-1, 1] holds
// (lo, b[lo], b[lo+1], b[lo+2]) with b[0] = -inf, b[K] = b[K+1] = +inf and lo =
// the number of boundaries below the cell; a cell holding two or more
// boundaries stores lo = -1 and flags.
__device__ __forceinline__ uint32_t cf_bucket(float x, float g, const float4* lut, bool& ok) {
  int cell = __float2int_rd((x + 1.f) * (0.5f * kCFCells));
  cell = cell < 0 ? 0 : (cell > kCFCells - 1 ? kCFCells - 1 : cell);
  const float4 e = lut[cell * kCFLutRep];
  const int lo = __float_as_int(e.x);
  const bool upx = x >= e.z;
  const float bl = upx ? e.z : e.y, bh = upx ? e.w : e.z;
  ok = ok && lo >= 0 && (x - bl > g) && (bh - x > g);
  return (uint32_t)lo + (upx ? 1u : 0u);
}

template <int BD, int BN, int MODE, int DT, bool QJL>
__global__ void __launch_bounds__(CFS<BD, BN, QJL>::NW * 32, 1)
    compress_fast_kernel(OqCodecParams p, const void* __restrict__ x, size_t n,
                         uint8_t* __restrict__ out, FlagEntry* __restrict__ flags,
                         uint32_t* __restrict__ flag_cnt) {
  using S = CFS<BD, BN, QJL>;
  constexpr int K = S::K;
  constexpr float U = 5.9604645e-8f;  // 2^-24
  constexpr float E0 = 7.02f * U;     // triplet-independent part of Et (see the header)
  extern __shared__ __align__(128) uint8_t smem[];
  float4* dirs = reinterpret_cast<float4*>(smem);
  float4* lut = reinterpret_cast<float4*>(smem + S::DIRS_BYTES);
  float* bnd = reinterpret_cast<float*>(smem + S::DIRS_BYTES + S::LUT_BYTES);
  float* rows = reinterpret_cast<float*>(smem + S::DIRS_BYTES + S::LUT_BYTES + S::BND_BYTES);
  uint32_t* recb = reinterpret_cast<uint32_t*>(smem + S::DIRS_BYTES + S::LUT_BYTES +
                                               S::BND_BYTES + S::ROWS_BYTES);
  uint32_t* scratch_all = recb + S::NW * S::RECBUF_WORDS;
  __shared__ __align__(8) uint64_t bars[S::NW];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- tables -------------------------------------------------------------
  // cell (a + 1, b + 1) = (n_hat(a, b), bias 0); border cells (0, 0, 0, -inf)
  // so every 3x3 window is 9 loads at immediate offsets and out-of-range
  // candidates score -inf (codec.hpp:164-176 clamps the window)
  stage_cells<S::DREP, S::KP * S::KP>(dirs, [&](int cell) {
    const int a = cell / S::KP - 1, b = cell % S::KP - 1;
    float4 v = make_float4(0.f, 0.f, 0.f, -INFINITY);
    if (a >= 0 && a < K && b >= 0 && b < K) {
      v = __ldg(reinterpret_cast<const float4*>(p.dirs32) + a * K + b);
      v.w = 0.f;
    }
    return v;
  }, tid, S::NW * 32);
  if (tid <= K) bnd[tid] = tid == 0 ? -INFINITY : (tid == K ? INFINITY : (float)p.xi_bnd[tid - 1]);
  float* rho_s = bnd + 40;  // fp32 norm centroids (QJL residual)
  if (QJL && tid < S::KR) rho_s[tid] = p.rho32[tid];
  __syncthreads();
  for (int c = tid; c < kCFCells; c += S::NW * 32) {
    // guard band 1e-6 >> the fp32 error of the cell index
    const float x0 = -1.f + (float)c / (0.5f * kCFCells) - 1e-6f;
    const float x1 = -1.f + (float)(c + 1) / (0.5f * kCFCells) + 1e-6f;
    int l = 0, h = 0;
    for (int i = 1; i < K; ++i) {
      l += bnd[i] < x0 ? 1 : 0;
      h += bnd[i] <= x1 ? 1 : 0;
    }
    auto bb = [&](int i) { return i >= K ? INFINITY : bnd[i]; };
    const float4 v = make_float4(__int_as_float(h - l <= 1 ? l : -1), bb(l), bb(l + 1), bb(l + 2));
    for (int r = 0; r < kCFLutRep; ++r) lut[c * kCFLutRep + r] = v;
  }
  float rbnd[S::KR - 1];
#pragma unroll
  for (int i = 0; i < S::KR - 1; ++i) rbnd[i] = (float)p.rho_bnd[i];
  const float4* dtab = dirs + (lane & (S::DREP - 1));
  const float4* mylut = lut + (lane & (kCFLutRep - 1));
  float* myrow = rows + (warp * 32 + lane) * kCFRow;
  uint32_t* wrec = recb + warp * S::RECBUF_WORDS;
  uint32_t* scratch = scratch_all + warp * 32 * (S::RW + 1);
  uint64_t* bar = &bars[warp];
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cf_smem(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const size_t nblk = (n + 31) / 32;
  const size_t wstride = (size_t)gridDim.x * S::NW;
  auto request = [&](size_t blk) {  // rows of block blk -> this warp's staging rows
    const size_t k0 = blk * 32;
    const int nk = (int)min((size_t)32, n - k0);
    constexpr int RB_IN = 128 * InElem<DT>::BYTES;  // bytes per input row
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cf_smem(bar)),
                   "r"(nk * RB_IN)
                   : "memory");
    __syncwarp();
    if (lane < nk)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(cf_smem(myrow)),
          "l"(static_cast<const uint8_t*>(x) + (k0 + lane) * RB_IN), "n"(RB_IN),
          "r"(cf_smem(bar))
          : "memory");
  };
  size_t blk = (size_t)blockIdx.x * S::NW + warp;
  if (blk < nblk) request(blk);
  uint32_t phase = 0;
  for (; blk < nblk; blk += wstride, phase ^= 1) {
    const size_t k0 = blk * 32;
    const int nk = (int)min((size_t)32, n - k0);
    asm volatile(
        "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W_%=;\n}" ::"r"(cf_smem(bar)),
        "r"(phase)
        : "memory");
    float y[128];
    load_elems<DT, 128>(y, myrow);  // exact widening of fp16 / bf16 keys
    const bool live = lane < nk;

    // ---- rotation in fp32: ur = H (s .* k) * c -------------------------------
    // (the unscaled signs + WHT first: gamma's serial fp64 chain below reads
    // the untouched staging row, so the two interleave)
#pragma unroll
    for (int i = 0; i < 128; ++i)
      if ((p.sign_mask[i >> 5] >> (i & 31)) & 1u) y[i] = -y[i];
#pragma unroll
    for (int len = 1; len < 128; len <<= 1)
#pragma unroll
      for (int i = 0; i < 128; ++i)
        if (!(i & len)) {
          const float a = y[i], b = y[i + len];
          y[i] = a + b;
          y[i + len] = a - b;
        }

    // ---- gamma: sequential fp64 sum of squares (codec.hpp:219-221) -----------
    double g2 = 0.0;
#pragma unroll
    for (int i4 = 0; i4 < 32; ++i4) {
      float k4[4];
      if constexpr (DT == OQ_F32) {
        const float4 v = reinterpret_cast<const float4*>(myrow)[i4];
        k4[0] = v.x; k4[1] = v.y; k4[2] = v.z; k4[3] = v.w;
      } else {
        const uint2 v = reinterpret_cast<const uint2*>(myrow)[i4];
        k4[0] = widen16<DT>(v.x & 0xffffu); k4[1] = widen16<DT>(v.x >> 16);
        k4[2] = widen16<DT>(v.y & 0xffffu); k4[3] = widen16<DT>(v.y >> 16);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double d = (double)k4[j];
        g2 = __fma_rn(d, d, g2);  // the square is exact: == g2 + d*d rounded once
      }
    }
    const double gamma = __dsqrt_rn(g2);
    const float gf = (float)gamma;  // codec.hpp:233
    const double inv = __ddiv_rn(1.0, gamma > 1e-12 ? gamma : 1e-12);
    const float c32 = (float)(inv * p.inv_sqrt_d);
    // outside [2^-60, 2^60] the fp32 rotation could lose range: exact path
    // for every triplet
    const bool ok = gamma > 8.7e-19 && gamma < 1.1e18;
    uint64_t fmask = 0;  // triplets whose decisions missed their margins
#pragma unroll
    for (int i = 0; i < 128; ++i) y[i] *= c32;

    // the rotated row goes back to this lane's staging row; the triplet loop
    // below is rolled (groups of 4 triplets = 3 float4) to keep the code small
#pragma unroll
    for (int i = 0; i < 32; ++i)
      *reinterpret_cast<float4*>(myrow + 4 * i) =
          make_float4(y[4 * i], y[4 * i + 1], y[4 * i + 2], y[4 * i + 3]);

    // ---- per-triplet joint rounding with certified decisions ----------------
    // record bitstream writers into this lane's scratch words (LSB-first,
    // codec.hpp:381-389): direction fields from bit 32, norm fields from bit
    // 32 + 8 * dir_bytes
    uint32_t* scr = scratch + lane;  // word i at scr[32 * i] (lane-interleaved)
#pragma unroll
    for (int i = 0; i <= S::RW; ++i) scr[32 * i] = 0u;
    scr[0] = __float_as_uint(gf);
    uint64_t dacc = 0, nacc = 0;
    int dn = 0, nn = (8 * S::DIRB) & 31, dw = 1, nw = (32 + 8 * S::DIRB) >> 5;
    // completed words are stored directly (the scratch row starts zeroed);
    // only the word the direction and norm streams share is OR-ed
    constexpr int SHARED_W = ((4 + S::DIRB) & 3) ? (4 + S::DIRB) >> 2 : -1;
    auto put = [&](int wi, uint32_t v) {
      if (wi == SHARED_W) scr[32 * wi] |= v;
      else scr[32 * wi] = v;
    };
    // append `bits` (<= 32) to a stream accumulator holding n < 32 bits
    auto append = [&](uint64_t& acc, int& n, int& w, uint64_t v, int bits) {
      acc |= v << n;
      n += bits;
      if (n >= 32) {
        put(w++, (uint32_t)acc);
        acc >>= 32;
        n -= 32;
      }
    };
#pragma unroll 2  // two groups per iteration: more independent triplets in flight
    for (int q = 0; q < 11; ++q) {
      float e[12];
      {
        const float4 v0 = *reinterpret_cast<const float4*>(myrow + 12 * q);
        const float4 v1 = *reinterpret_cast<const float4*>(myrow + 12 * q + 4);
        const float4 v2 = q < 10 ? *reinterpret_cast<const float4*>(myrow + 12 * q + 8)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        e[0] = v0.x; e[1] = v0.y; e[2] = v0.z; e[3] = v0.w;
        e[4] = v1.x; e[5] = v1.y; e[6] = v1.z; e[7] = v1.w;
        e[8] = v2.x; e[9] = v2.y; e[10] = v2.z; e[11] = v2.w;
      }
      uint32_t gmask = 0;  // undecided triplets of this group of 4
      // (4,2): a group's four 8-bit direction pairs are exactly record word
      // q + 1 and its four 2-bit norms record byte 47 + q (stored directly)
      uint32_t gdir = 0, gnrm = 0;
      uint64_t gdir64 = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = 4 * q + j;
        if (t >= S::NT) break;
        const bool pad = t == S::NT - 1;  // elements 126, 127 and the zero pad
        bool okt = true;
        const float t0 = e[3 * j], t1 = e[3 * j + 1], t2 = pad ? 0.f : e[3 * j + 2];
        const float a0 = fabsf(t0), a1 = fabsf(t1), a2 = fabsf(t2);
        const float l1 = a0 + a1 + a2;
        float il;  // rcp.approx: relative error <= 2^-23
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(il) : "f"(l1));
        // Et = E0 + 2.01u |t| <= E0 + 2.01u l1.  xi = t0 / l1 (or 1 - |t1| / l1):
        // |d xi| <= (|dt0| + |xi| |dl1|) / l1 <= (1 + sqrt 3) Et / l1, plus <= 8u
        // of fp32 rounding and u for the fp32 boundaries
        const bool up = pad || t2 >= 0.f;  // octahedral.hpp:28 (pad: pz = 0 exactly)
        // hemisphere and, below it, sgn(px), sgn(py) (octahedral.hpp:29-30):
        // |t_i| > E0 + 2.01u |t_i| is implied by |t_i| > 1.0001 E0
        const float es = 1.0001f * E0;
        // When the signs of t0 and t1 cannot flip under the rotation error
        // (|t_i| > es; t2's sign is certified below, the pad's t2 is exactly
        // 0), l1 is linear in dt and xi' - xi = (w . dt) / l1' with
        // |w|^2 = (1 - |xi|)^2 + 2 xi^2 <= 2: the factor (1 + sqrt 3) drops
        // to sqrt 2 (the same for eta, and in the lower hemisphere with t1
        // and t0 swapped)
        const bool sst = a0 > es && a1 > es;
        const float gx = ((sst ? 1.415f : 2.74f) * E0 * il + (sst ? 2.85f : 5.51f) * U + 9.f * U) * 1.001f;
        okt = l1 > 1e-6f && (pad || a2 > es) && (up || (a0 > es && a1 > es));
        const float xi = up ? t0 * il : copysignf(1.f - a1 * il, t0);
        const float eta = up ? t1 * il : copysignf(1.f - a0 * il, t1);
        const uint32_t sx = cf_bucket(xi, gx, mylut, okt);
        const uint32_t sy = cf_bucket(eta, gx, mylut, okt);
        uint32_t ix = sx, iy = sy;
        float rv, gr;
        if (MODE == 0) {  // scalar: rho of clamp(|t|, 0, 1) (codec.hpp:154-162)
          rv = sqrtf(fmaf(t2, t2, fmaf(t1, t1, t0 * t0)));
          gr = (E0 + 4.6f * U * l1) * 1.001f;  // Et + fp32 sum/sqrt rounding
        } else {  // local3x3 (codec.hpp:164-192): strict '>' argmax over the window
          float b1 = -INFINITY, b2 = -INFINITY;
          uint32_t wi = 0;
          // window corner (sx - 1, sy - 1) = padded cell (sx, sy)
          const float4* wp = dtab + (sx * S::KP + sy) * S::DREP;
#pragma unroll
          for (int da = 0; da < 3; ++da)
#pragma unroll
            for (int db = 0; db < 3; ++db) {
              const float4 nv = wp[(da * S::KP + db) * S::DREP];
              const float sc = fmaf(t2, nv.z, fmaf(t1, nv.y, fmaf(t0, nv.x, nv.w)));
              const bool gt = sc > b1;
              b2 = fmaxf(b2, fminf(b1, sc));
              b1 = fmaxf(b1, sc);
              wi = gt ? (uint32_t)(da * 4 + db) : wi;
            }
          // score error: ||dt|| <= Et (rotation) + |t| u/2 (fp32 table) + 3u |t|
          // (dot rounding), with |t| <= l1
          const float gs = (E0 + 5.53f * U * l1) * 1.001f;
          // the best beats every other candidate c by more than the error of
          // the score difference: |dt| |n_best - n_c| (<= Et dwin, dwin
          // bounding the direction distances within any window) plus the
          // rounding of the two fp32 dot products and table entries (7u |t|)
          okt = okt && (b1 - b2 > (p.dwin * (E0 + 2.02f * U * l1) + 7.02f * U * l1) * 1.002f);
          ix = sx + (wi >> 2) - 1;
          iy = sy + (wi & 3) - 1;
          rv = b1;
          gr = gs;
        }
        rv = fminf(fmaxf(rv, 0.f), 1.f);
        uint32_t ir = 0;
#pragma unroll
        for (int i = 0; i < S::KR - 1; ++i) {
          ir += rv >= rbnd[i] ? 1u : 0u;
          okt = okt && fabsf(rv - rbnd[i]) > gr + U;
        }
        gmask |= (okt ? 0u : 1u) << j;
        if constexpr (QJL) {
          // residual r = t - rho_hat n_hat of the chosen codes (codec.hpp:243-246,
          // 252-266) back into this triplet's slots of the row; the pad
          // coordinate is dropped (qjl.hpp:23-36 works on the d real ones)
          const float4 nv = dtab[(((ix & (K - 1)) + 1) * S::KP + (iy & (K - 1)) + 1) * S::DREP];
          const float rh = rho_s[ir];
          float* rw = myrow + 12 * q + 3 * j;
          rw[0] = t0 - rh * nv.x;
          rw[1] = t1 - rh * nv.y;
          if (!pad) rw[2] = t2 - rh * nv.z;
        }
        // ---- append the fields (masked to their widths: an undecided
        // triplet's fields are patched in place by the exact fixup) ----------
        const uint32_t fpair = (ix & (K - 1)) | ((iy & (K - 1)) << BD);
        if constexpr (BD == 4 && BN == 2) {
          gdir |= fpair << (8 * j);
          gnrm |= ir << (2 * j);
        } else {  // group bits at compile-time offsets, one stream append per group
          gdir64 |= (uint64_t)fpair << (2 * BD * j);
          gnrm |= ir << (BN * j);
        }
      }
      if constexpr (!(BD == 4 && BN == 2)) {
        const int ng = q < 10 ? 4 : S::NT - 40;  // triplets in this group
        if (2 * BD * ng <= 32) {
          append(dacc, dn, dw, gdir64, 2 * BD * ng);
        } else {
          append(dacc, dn, dw, gdir64 & 0xffffffffull, 32);
          append(dacc, dn, dw, gdir64 >> 32, 2 * BD * ng - 32);
        }
        append(nacc, nn, nw, gnrm, BN * ng);
      } else {
        static_assert(S::DIRB == 43, "record layout of (4,2)");
        // word 11 (q = 10) holds dir bytes 44..46 and norm byte 47 (q = 0's)
        if (q < 10) scr[32 * (q + 1)] = gdir;
        else scr[32 * (q + 1)] |= gdir;
        const int nb = 4 + S::DIRB + q;  // record byte of this group's norms
        reinterpret_cast<uint8_t*>(scr + 32 * (nb >> 2))[nb & 3] = (uint8_t)gnrm;
      }
      fmask |= (uint64_t)gmask << (4 * q);
    }
    if constexpr (!(BD == 4 && BN == 2)) {
      if (dn > 0) put(dw, (uint32_t)dacc);
      if (nn > 0) put(nw, (uint32_t)nacc);
    }
    bool okq = true;
    if constexpr (QJL) {
      // ---- QJL sidecar (qjl.hpp:23-36), certified like the codes ----------
      // ||r32 - r64|| <= Er = 13.1u: rotation (9.03u over the whole vector),
      // fp32 tables and product for rho_hat n_hat (1.51u ||u_hat|| <= 3.02u),
      // the subtraction (<= u).
      float y[128];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float4 v = *reinterpret_cast<const float4*>(myrow + 4 * i);
        y[4 * i] = v.x; y[4 * i + 1] = v.y; y[4 * i + 2] = v.z; y[4 * i + 3] = v.w;
      }
      // gamma_r = f16(float(sqrt(sum r^2))), the sum sequential in fp64 (the
      // fp32 squares are exact in fp64).  |sum r32^2 - sum r64^2| <=
      // Er (2 ||r32|| + Er); gamma_r is certified when both ends of that
      // interval round to the same f16 (sqrt, float() and f16() are monotone).
      // w = H (s' .* r) / sqrt(d) in fp32: ||w32 - w64|| <= Er + 7u ||r||
      // (butterflies) + u ||r|| (scale); sign bit i = (w_i >= 0).  The
      // butterflies first: the serial n2 chain reads the row in shared memory
      // and interleaves with them.
#pragma unroll
      for (int i = 0; i < 128; ++i)
        if ((p.qsign_mask[i >> 5] >> (i & 31)) & 1u) y[i] = -y[i];
#pragma unroll
      for (int len = 1; len < 128; len <<= 1)
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (!(i & len)) {
            const float a = y[i], b = y[i + len];
            y[i] = a + b;
            y[i + len] = a - b;
          }
      double n2 = 0.0;
#pragma unroll
      for (int i4 = 0; i4 < 32; ++i4) {
        const float4 v = *reinterpret_cast<const float4*>(myrow + 4 * i4);
        n2 = __fma_rn((double)v.x, (double)v.x, n2);
        n2 = __fma_rn((double)v.y, (double)v.y, n2);
        n2 = __fma_rn((double)v.z, (double)v.z, n2);
        n2 = __fma_rn((double)v.w, (double)v.w, n2);
      }
      constexpr double ER = 13.1 * 5.9604644775390625e-8;
      const double nr = __dsqrt_rn(n2);
      const double en2 = ER * (2.0 * nr + ER) * 1.001 + 1e-13 * n2;
      const uint16_t hlo = f32_to_f16_ref((float)__dsqrt_rn(fmax(n2 - en2, 0.0)));
      const uint16_t hhi = f32_to_f16_ref((float)__dsqrt_rn(n2 + en2));
      okq = hlo == hhi;
      const float isd = (float)p.inv_sqrt_d;
      const float ew = (float)((ER + 8.01 * 5.9604644775390625e-8 * nr) * 1.001 + 1e-14);
      uint32_t sg[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int i = 0; i < 128; ++i) {
        const float wv = y[i] * isd;
        sg[i >> 5] |= (wv >= 0.f ? 1u : 0u) << (i & 31);
        okq = okq && fabsf(wv) > ew;
      }
      // the 18 sidecar bytes (gamma_r, 16 sign bytes, LSB first) at record
      // byte QB, OR-ed into the scratch words (the first one is shared with
      // the norm stream)
      const uint32_t b0 = (uint32_t)hlo | (sg[0] << 16), b1 = (sg[0] >> 16) | (sg[1] << 16),
                     b2 = (sg[1] >> 16) | (sg[2] << 16), b3 = (sg[2] >> 16) | (sg[3] << 16),
                     b4 = sg[3] >> 16;
      constexpr int QW = S::QB >> 2, QO = 8 * (S::QB & 3);
      const uint32_t bw[5] = {b0, b1, b2, b3, b4};
#pragma unroll
      for (int i = 0; i <= 5; ++i) {
        const uint32_t lo = i < 5 ? bw[i] : 0u, hi = i > 0 ? bw[i - 1] : 0u;
        const uint32_t v = QO ? ((lo << QO) | (i > 0 ? hi >> (32 - QO) : 0u)) : lo;
        if (QW + i < S::RW) scr[32 * (QW + i)] |= v;
      }
    }
    __syncwarp();
    if (blk + wstride < nblk) {  // the staging row is consumed: fetch the next block
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      request(blk + wstride);
    }
    uint32_t w[S::RW + 1];
#pragma unroll
    for (int i = 0; i <= S::RW; ++i) w[i] = i < S::RW ? scr[32 * i] : 0u;

    // ---- keys with undecided triplets: exact fixup later ---------------------
    if (!ok || !okq) fmask = (1ull << S::NT) - 1;
    const uint32_t bad = __ballot_sync(kFull, live && fmask != 0);
    if (bad) {
      uint32_t basei = 0;
      if (lane == 0) basei = atomicAdd(flag_cnt, (uint32_t)__popc(bad));
      basei = __shfl_sync(kFull, basei, 0);
      if (live && fmask != 0) {
        FlagEntry fe;
        fe.key = (uint32_t)(k0 + lane);
        fe.mlo = (uint32_t)fmask;
        fe.mhi = (uint32_t)(fmask >> 32);
        fe.pad = 0;
        fe.inv = inv;
        fe.pad2 = 0.0;
        flags[basei + __popc(bad & ((1u << lane) - 1u))] = fe;
      }
    }

    // ---- the warp's 32 records -> shared buffer -> one bulk store ------------
    {
      const uint32_t D = (uint32_t)lane * S::RB, o = 8 * (D & 3), wb = D >> 2;
      const uint32_t last = (D + S::RB - 1) >> 2;  // last word this record touches
      uint32_t prev = 0, mine[S::RW + 1];
#pragma unroll
      for (int j = 0; j <= S::RW; ++j) {
        mine[j] = o ? __funnelshift_l(prev, w[j], o) : w[j];
        prev = w[j];
      }
      // the first word may share bytes with lane-1's last word
      const uint32_t up = __shfl_up_sync(kFull, (last - wb == S::RW) ? mine[S::RW] : mine[S::RW - 1], 1);
      const uint32_t prev_last = __shfl_up_sync(kFull, last, 1);
      if (lane > 0 && prev_last == wb) mine[0] |= up;
      const bool share_end = lane < 31 && ((D + S::RB) & 3);
#pragma unroll
      for (int j = 0; j <= S::RW; ++j) {
        const uint32_t wd = wb + j;
        if (wd < last || (wd == last && !share_end)) wrec[wd] = mine[j];
      }
    }
    __syncwarp();
    uint8_t* dst = out + k0 * S::RB;
    if (nk == 32) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                     "r"(cf_smem(wrec)), "r"(32 * S::RB)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    } else {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(wrec);
      for (int i = lane; i < nk * S::RB; i += 32) dst[i] = src[i];
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int BD, int BN, int MODE, int DT, bool QJL>
static cudaError_t launch_cf_t(const OqCodecParams& p, const void* x, size_t n, uint8_t* out,
                               FlagEntry* flag_idx, uint32_t* flag_cnt, cudaStream_t st,
                               int num_sms) {
  using S = CFS<BD, BN, QJL>;
  static_assert(S::SMEM <= 227 * 1024, "compress_fast shared memory");
  cudaError_t e = set_smem_once(compress_fast_kernel<BD, BN, MODE, DT, QJL>, S::SMEM);
  if (e != cudaSuccess) return e;
  const size_t nblk = (n + 31) / 32;
  size_t grid = (nblk + S::NW - 1) / S::NW;
  if (grid > (size_t)num_sms) grid = num_sms;
  compress_fast_kernel<BD, BN, MODE, DT, QJL>
      <<<(unsigned)grid, S::NW * 32, S::SMEM, st>>>(p, x, n, out, flag_idx, flag_cnt);
  return cudaGetLastError();
}

template <int BD, int BN, int MODE, bool QJL>
static cudaError_t launch_cf(const OqCodecParams& p, const void* x, int dtype, size_t n,
                             uint8_t* out, FlagEntry* flag_idx, uint32_t* flag_cnt,
                             cudaStream_t st, int num_sms) {
  if (dtype == OQ_BF16)
    return launch_cf_t<BD, BN, MODE, OQ_BF16, QJL>(p, x, n, out, flag_idx, flag_cnt, st, num_sms);
  if (dtype == OQ_F16)
    return launch_cf_t<BD, BN, MODE, OQ_F16, QJL>(p, x, n, out, flag_idx, flag_cnt, st, num_sms);
  return launch_cf_t<BD, BN, MODE, OQ_F32, QJL>(p, x, n, out, flag_idx, flag_cnt, st, num_sms);
}

bool compress_fast_ok(const OqCodecParams& p, int dtype, const void* x, const void* out) {
  if (p.dim != 128 || dtype == OQ_F64) return false;
  if (p.rounding != 0 && p.rounding != 2) return false;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(out) & 15)) return false;
  return (p.b_dir == 3 && p.b_nrm == 1) || (p.b_dir == 4 && p.b_nrm == 2) ||
         (p.b_dir == 5 && p.b_nrm == 3);
}

cudaError_t launch_compress_fast(const OqCodecParams& p, const void* x, int dtype, size_t n,
                                 uint8_t* out, FlagEntry* flag_idx, uint32_t* flag_cnt,
                                 cudaStream_t st, int num_sms) {
#define OQ_CF(BD, BN, Q)                                                                         \
  if (p.b_dir == BD && p.b_nrm == BN && (bool)p.qjl == Q)                                       \
    return p.rounding == 0                                                                      \
               ? launch_cf<BD, BN, 0, Q>(p, x, dtype, n, out, flag_idx, flag_cnt, st, num_sms)  \
               : launch_cf<BD, BN, 2, Q>(p, x, dtype, n, out, flag_idx, flag_cnt, st, num_sms);
  OQ_CF(3, 1, false)
  OQ_CF(4, 2, false)
  OQ_CF(5, 3, false)
  OQ_CF(3, 1, true)
  OQ_CF(4, 2, true)
  OQ_CF(5, 3, true)
#undef OQ_CF
  return cudaErrorNotSupported;
}

}  // namespace oqd
