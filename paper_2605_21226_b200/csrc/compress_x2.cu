// compress_x2.cu — K1 for d = 128 (fp32 / fp16 / bf16 keys): Encoder::encode (codec.hpp:214-249), bit-
// exact in ONE pass, two lanes per key.
//
// Per warp, 16 keys at a time:
//  * lane (p, h) = lane 2p + h pulls half h (64 floats) of key p's row into
//    shared memory with a 1-D TMA bulk copy (one mbarrier per warp);
//  * gamma replays the reference's sequential fp64 sum of squares exactly:
//    half 0 sums elements 0..63, hands the partial sum to half 1 with one
//    shuffle, which continues over 64..127 (the fp32 squares are exact in
//    fp64, so fma(k, k, s) == s + k*k rounded once);
//  * u = k * inv, the sign flips and the WHT run in fp64 with the reference's
//    exact operation order — six in-lane butterfly stages and the len = 64
//    stage across the lane pair — then * (1/sqrt d): the rotated coordinates
//    are bit-identical to Rotation::apply (rotation.hpp:46-49);
//  * lane h encodes triplets 21h .. 21h + 20 (+ the padded triplet 42 for
//    h = 1) from its coordinates, written once to a shared work row (lane 1's
//    row starts at element 63).  The octahedral fold, both bucket searches
//    and the norm bucket are exact fp64 (a 128-cell LUT brackets the bucket,
//    one fp64 compare decides it); the 3x3 argmax is screened in fp32 over a
//    -inf-padded direction table and CERTIFIED by a margin larger than the
//    fp32 score error (4.1 u |t|_1), the winner's score then recomputed in
//    fp64; windows that fail the margin rerun the reference's exact strict-'>'
//    scan in fp64 (rare, inline);
//  * each lane writes its fields with two sequential bit writers into its own
//    scratch words; lane 0 of each pair ORs the two halves with gamma into
//    the OCTO v1 record, records are merged at shared word boundaries with
//    one shuffle and the warp's 16 records leave with one TMA bulk store.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace oqd {

constexpr int kX2Warps = 8;
constexpr int kX2Threads = 32 * kX2Warps;
constexpr int kX2Work = 66;  // doubles per lane work row
constexpr int kX2Cells = 128, kX2LutRep = 8;

template <int BD, int BN>
struct X2S {
  static constexpr int K = 1 << BD, KR = 1 << BN, NT = 43, KP = K + 2;
  static constexpr int DIRB = (2 * NT * BD + 7) / 8, NRMB = (NT * BN + 7) / 8;
  static constexpr int RB = 4 + DIRB + NRMB;
  static constexpr int RW = (RB + 3) / 4;
  static constexpr int DREP = BD <= 4 ? 8 : 1;
  static constexpr int DIRS32 = KP * KP * DREP * 16;
  static constexpr int DIRS64 = ((K * K * 3 * 8) + 15) & ~15;
  static constexpr int LUT = kX2Cells * kX2LutRep * 16;
  static constexpr int BND = 64 * 8;
  static constexpr int WBUF = 32 * kX2Work * 8;   // also the TMA staging (16 x 544 B)
  static constexpr int SCR = 32 * (RW + 1) * 4;
  static constexpr int RECB = 16 * RB;             // multiple of 16
  static constexpr int PERWARP = WBUF + SCR + RECB;
  static constexpr int SMEM = DIRS32 + DIRS64 + LUT + BND + kX2Warps * PERWARP + 16;
};

__device__ __forceinline__ uint32_t x2_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// octahedral.hpp:22-31, exact fp64 in the reference's operation order.
__device__ __forceinline__ void x2_oct(double t0, double t1, double t2, double& xi, double& eta) {
  const double l1 = dadd(dadd(fabs(t0), fabs(t1)), fabs(t2));
  const double inv = ddiv(1.0, l1 > 1e-12 ? l1 : 1e-12);
  const double px = dmul(t0, inv), py = dmul(t1, inv), pz = dmul(t2, inv);
  if (pz >= 0.0) {
    xi = px;
    eta = py;
  } else {
    xi = dflip(dsub(1.0, fabs(py)), !(px >= 0.0));
    eta = dflip(dsub(1.0, fabs(px)), !(py >= 0.0));
  }
}

// std::upper_bound count over the xi boundaries (lloydmax.hpp:46-49), exact:
// the LUT cell of float(x) brackets the answer to {lo, lo + 1} (built with a
// 1e-6 guard band), one fp64 compare against b[lo + 1] decides.  b64[0] =
// -inf, b64[i] = boundary i - 1, b64[K] = +inf.  Cells holding two or more
// boundaries (lo < 0) binary-search.
__device__ __forceinline__ uint32_t x2_bucket(double x, const float4* lut, const double* b64,
                                              int K) {
  int cell = __float2int_rd(((float)x + 1.f) * (0.5f * kX2Cells));
  cell = cell < 0 ? 0 : (cell > kX2Cells - 1 ? kX2Cells - 1 : cell);
  const int lo = __float_as_int(lut[cell * kX2LutRep].x);
  if (lo >= 0 && x == x) return (uint32_t)lo + (x >= b64[lo + 1] ? 1u : 0u);
  return quantize_ub(b64 + 1, (uint32_t)(K - 1), x);  // wide cells and NaN (inf keys)
}

// list != nullptr: encode only keys list[0 .. *list_n) (the certified-fp32
// pass's flagged keys), each record stored at its own key slot.
template <int BD, int BN, int MODE, int DT>
__global__ void __launch_bounds__(kX2Threads, 1)
    compress_x2_kernel(OqCodecParams p, const void* __restrict__ x, size_t n,
                       uint8_t* __restrict__ out, const uint32_t* __restrict__ list,
                       const uint32_t* __restrict__ list_n) {
  using S = X2S<BD, BN>;
  constexpr int K = S::K;
  constexpr float U = 5.9604645e-8f;  // 2^-24
  extern __shared__ __align__(128) uint8_t smem[];
  float4* dirs32 = reinterpret_cast<float4*>(smem);
  double* dirs64 = reinterpret_cast<double*>(smem + S::DIRS32);
  float4* lut = reinterpret_cast<float4*>(smem + S::DIRS32 + S::DIRS64);
  double* b64 = reinterpret_cast<double*>(smem + S::DIRS32 + S::DIRS64 + S::LUT);
  uint8_t* perwarp = smem + S::DIRS32 + S::DIRS64 + S::LUT + S::BND;
  __shared__ __align__(8) uint64_t bars[kX2Warps];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = lane & 1, pk = lane >> 1;

  // ---- tables -------------------------------------------------------------
  // padded fp32 direction grid: cell (a + 1, b + 1) = (n_hat(a, b), 0),
  // border cells (0, 0, 0, -inf): out-of-window candidates score -inf
  stage_cells<S::DREP, S::KP * S::KP>(dirs32, [&](int cell) {
    const int a = cell / S::KP - 1, b = cell % S::KP - 1;
    float4 v = make_float4(0.f, 0.f, 0.f, -INFINITY);
    if (a >= 0 && a < K && b >= 0 && b < K) {
      v = __ldg(reinterpret_cast<const float4*>(p.dirs32) + a * K + b);
      v.w = 0.f;
    }
    return v;
  }, tid, kX2Threads);
  {
    constexpr int N64 = K * K * 3, PER = (N64 + kX2Threads - 1) / kX2Threads;
    double v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = k * kX2Threads + tid;
      v[k] = i < N64 ? __ldg(p.dirs64 + i) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = k * kX2Threads + tid;
      if (i < N64) dirs64[i] = v[k];
    }
  }
  if (tid <= K) b64[tid] = tid == 0 ? -INFINITY : (tid == K ? INFINITY : p.xi_bnd[tid - 1]);
  __syncthreads();
  for (int c = tid; c < kX2Cells; c += kX2Threads) {
    const double x0 = -1.0 + (double)c / (0.5 * kX2Cells) - 1e-6;
    const double x1 = -1.0 + (double)(c + 1) / (0.5 * kX2Cells) + 1e-6;
    int l = 0, hh = 0;
    for (int i = 1; i < K; ++i) {
      l += b64[i] < x0 ? 1 : 0;
      hh += b64[i] <= x1 ? 1 : 0;
    }
    const float4 v = make_float4(__int_as_float(hh - l <= 1 ? l : -1), 0.f, 0.f, 0.f);
    for (int r = 0; r < kX2LutRep; ++r) lut[c * kX2LutRep + r] = v;
  }
  double rb[S::KR - 1];
#pragma unroll
  for (int i = 0; i < S::KR - 1; ++i) rb[i] = p.rho_bnd[i];
  const float4* dtab = dirs32 + (lane & (S::DREP - 1));
  const float4* mylut = lut + (lane & (kX2LutRep - 1));
  uint8_t* wb = perwarp + warp * S::PERWARP;
  double* wrow = reinterpret_cast<double*>(wb) + lane * kX2Work;      // work row
  float* half = reinterpret_cast<float*>(wb + pk * 544 + h * 272);   // staging half row
  uint32_t* scr = reinterpret_cast<uint32_t*>(wb + S::WBUF) + lane;  // word i at scr[32 i]
  uint32_t* recb = reinterpret_cast<uint32_t*>(wb + S::WBUF + S::SCR);
  uint64_t* bar = &bars[warp];
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(x2_smem(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (list) n = *list_n;
  const size_t nblk = (n + 15) / 16;
  const size_t wstride = (size_t)gridDim.x * kX2Warps;
  auto key_of = [&](size_t i) -> size_t { return list ? (size_t)list[i] : i; };
  auto request = [&](size_t blk) {
    const size_t k0 = blk * 16;
    const int nk = (int)min((size_t)16, n - k0);
    constexpr int EB = InElem<DT>::BYTES;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(x2_smem(bar)),
                   "r"(nk * 128 * EB)
                   : "memory");
    __syncwarp();
    if (pk < nk)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(x2_smem(half)),
          "l"(static_cast<const uint8_t*>(x) + (key_of(k0 + pk) * 128 + 64 * h) * EB),
          "n"(64 * EB), "r"(x2_smem(bar))
          : "memory");
  };
  size_t blk = (size_t)blockIdx.x * kX2Warps + warp;
  if (blk < nblk) request(blk);
  uint32_t phase = 0;
  for (; blk < nblk; blk += wstride, phase ^= 1) {
    const size_t k0 = blk * 16;
    const int nk = (int)min((size_t)16, n - k0);
    asm volatile(
        "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W_%=;\n}" ::"r"(x2_smem(bar)),
        "r"(phase)
        : "memory");
    float y[64];
    load_elems<DT, 64>(y, half);  // exact widening of fp16 / bf16 keys
    __syncwarp();  // staging consumed: the work rows may overwrite it

    // ---- gamma = sqrt(sequential fp64 sum of squares) (codec.hpp:219-221) ----
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const double d = (double)y[i];
      acc = __fma_rn(d, d, acc);
    }
    double acc2 = __shfl_up_sync(kFull, acc, 1);  // half 1 continues from half 0
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const double d = (double)y[i];
      acc2 = __fma_rn(d, d, acc2);
    }
    const double g2 = __shfl_sync(kFull, acc2, lane | 1);
    const double gamma = dsqrt(g2);
    const double inv = ddiv(1.0, gamma > 1e-12 ? gamma : 1e-12);

    // ---- u = k * inv, signs, WHT (rotation.hpp:20-31, 46-49), exact fp64 -----
    double v[64];
    const uint32_t sm0 = p.sign_mask[2 * h], sm1 = p.sign_mask[2 * h + 1];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const bool neg = ((i < 32 ? sm0 : sm1) >> (i & 31)) & 1u;
      v[i] = dflip(dmul((double)y[i], inv), neg);
    }
#pragma unroll
    for (int len = 1; len < 64; len <<= 1)
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (!(i & len)) {
          const double a = v[i], b = v[i + len];
          v[i] = dadd(a, b);
          v[i + len] = dsub(a, b);
        }
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const double o = __shfl_xor_sync(kFull, v[i], 1);
      v[i] = h ? dsub(o, v[i]) : dadd(v[i], o);  // element i (half 0) with i + 64
      v[i] = dmul(v[i], p.inv_sqrt_d);
    }
    // ---- work row: lane h holds elements 63h .. 63h + 65 ---------------------
    {
      const double e63 = __shfl_sync(kFull, v[63], lane & ~1);
#pragma unroll
      for (int i = 0; i < 64; ++i) wrow[i + h] = v[i];
      if (h) wrow[0] = e63;
      else wrow[64] = 0.0;
      wrow[65] = 0.0;
    }
    __syncwarp();

    // ---- triplets 21h + u ------------------------------------------------------
#pragma unroll
    for (int i = 0; i <= S::RW; ++i) scr[32 * i] = 0u;
    const int t_first = 21 * h;
    uint64_t dacc = 0, nacc = 0;
    int dn = (32 + 2 * BD * t_first) & 31, dw = (32 + 2 * BD * t_first) >> 5;
    int nn = (32 + 8 * S::DIRB + BN * t_first) & 31, nw = (32 + 8 * S::DIRB + BN * t_first) >> 5;
    const int nu = h ? 22 : 21;
#pragma unroll 1
    for (int g = 0; g < 11; ++g) {
      double e[6];
      {
        const double2 q0 = reinterpret_cast<const double2*>(wrow)[3 * g];
        const double2 q1 = reinterpret_cast<const double2*>(wrow)[3 * g + 1];
        const double2 q2 = reinterpret_cast<const double2*>(wrow)[3 * g + 2];
        e[0] = q0.x; e[1] = q0.y; e[2] = q1.x; e[3] = q1.y; e[4] = q2.x; e[5] = q2.y;
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int u = 2 * g + j;
        if (u >= nu) break;
        const double t0 = e[3 * j], t1 = e[3 * j + 1], t2 = e[3 * j + 2];
        double xi, eta;
        x2_oct(t0, t1, t2, xi, eta);
        const uint32_t sx = x2_bucket(xi, mylut, b64, K);
        const uint32_t sy = x2_bucket(eta, mylut, b64, K);
        uint32_t ix = sx, iy = sy;
        double rv;
        if (MODE == 0) {  // scalar (codec.hpp:154-162)
          rv = dsqrt(dadd(dadd(dmul(t0, t0), dmul(t1, t1)), dmul(t2, t2)));
        } else {  // local3x3 (codec.hpp:164-192)
          const float f0 = (float)t0, f1 = (float)t1, f2 = (float)t2;
          float b1 = -INFINITY, b2 = -INFINITY;
          uint32_t wi = 0;
          const float4* wp = dtab + (sx * S::KP + sy) * S::DREP;
#pragma unroll
          for (int da = 0; da < 3; ++da)
#pragma unroll
            for (int db = 0; db < 3; ++db) {
              const float4 nv = wp[(da * S::KP + db) * S::DREP];
              const float sc = fmaf(f2, nv.z, fmaf(f1, nv.y, fmaf(f0, nv.x, nv.w)));
              const bool gt = sc > b1;
              b2 = fmaxf(b2, fminf(b1, sc));
              b1 = fmaxf(b1, sc);
              wi = gt ? (uint32_t)(da * 4 + db) : wi;
            }
          // |s32 - s64| <= (u/2 + u/2 + 3u) |t|_1 (+ the fp64 dot's own ~1e-15)
          const float gs = 4.1f * U * (fabsf(f0) + fabsf(f1) + fabsf(f2)) + 1e-12f;
          if (b1 - b2 > 2.f * gs) {
            ix = sx + (wi >> 2) - 1;
            iy = sy + (wi & 3) - 1;
            const double* nd = dirs64 + 3 * (ix * K + iy);
            rv = dadd(dadd(dmul(t0, nd[0]), dmul(t1, nd[1])), dmul(t2, nd[2]));
          } else {  // near tie: the reference's exact scan, strict '>'
            const uint32_t a0 = sx > 0 ? sx - 1 : 0, a1 = sx + 1 < (uint32_t)K ? sx + 1 : K - 1;
            const uint32_t c0 = sy > 0 ? sy - 1 : 0, c1 = sy + 1 < (uint32_t)K ? sy + 1 : K - 1;
            double best = -INFINITY;
            ix = a0;  // the reference's initial (bx, by) (codec.hpp:180-189)
            iy = c0;
            for (uint32_t a = a0; a <= a1; ++a)
              for (uint32_t b = c0; b <= c1; ++b) {
                const double* nd = dirs64 + 3 * (a * K + b);
                const double sc = dadd(dadd(dmul(t0, nd[0]), dmul(t1, nd[1])), dmul(t2, nd[2]));
                if (sc > best) {
                  best = sc;
                  ix = a;
                  iy = b;
                }
              }
            rv = best;
          }
        }
        rv = rv < 0.0 ? 0.0 : (rv > 1.0 ? 1.0 : rv);
        uint32_t ir = 0;
#pragma unroll
        for (int i = 0; i < S::KR - 1; ++i) ir += (rv < rb[i]) ? 0u : 1u;  // upper_bound
        // ---- append the fields (codec.hpp:381-389) -----------------------------
        dacc |= (uint64_t)(ix | (iy << BD)) << dn;
        dn += 2 * BD;
        if (dn >= 32) {
          scr[32 * dw++] |= (uint32_t)dacc;
          dacc >>= 32;
          dn -= 32;
        }
        nacc |= (uint64_t)ir << nn;
        nn += BN;
        if (nn >= 32) {
          scr[32 * nw++] |= (uint32_t)nacc;
          nacc >>= 32;
          nn -= 32;
        }
      }
    }
    if (dn > 0) scr[32 * dw] |= (uint32_t)dacc;
    if (nn > 0) scr[32 * nw] |= (uint32_t)nacc;
    __syncwarp();
    if (blk + wstride < nblk) {  // work rows (= staging) consumed: fetch the next block
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      request(blk + wstride);
    }

    // ---- lane 0 of each pair: record = gamma | fields of both halves ----------
    {
      uint32_t w[S::RW + 1];
#pragma unroll
      for (int i = 0; i < S::RW; ++i) w[i] = scr[32 * i] | scr[32 * i + 1];
      w[0] = __float_as_uint((float)gamma);  // codec.hpp:233
      w[S::RW] = 0u;
      const uint32_t D = (uint32_t)pk * S::RB, o = 8 * (D & 3), wb0 = D >> 2;
      const uint32_t last = (D + S::RB - 1) >> 2;
      uint32_t prev = 0, mine[S::RW + 1];
#pragma unroll
      for (int j = 0; j <= S::RW; ++j) {
        mine[j] = o ? __funnelshift_l(prev, w[j], o) : w[j];
        prev = w[j];
      }
      const uint32_t up =
          __shfl_up_sync(kFull, (last - wb0 == S::RW) ? mine[S::RW] : mine[S::RW - 1], 2);
      const uint32_t prev_last = __shfl_up_sync(kFull, last, 2);
      if (pk > 0 && prev_last == wb0) mine[0] |= up;
      const bool share_end = pk < 15 && ((D + S::RB) & 3);
      if (!h) {
#pragma unroll
        for (int j = 0; j <= S::RW; ++j) {
          const uint32_t wd = wb0 + j;
          if (wd < last || (wd == last && !share_end)) recb[wd] = mine[j];
        }
      }
    }
    __syncwarp();
    uint8_t* dst = out + k0 * S::RB;
    if (list) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(recb);
      for (int i = lane; i < nk * S::RB; i += 32) {
        const int kp = i / S::RB;
        out[key_of(k0 + kp) * S::RB + (i - kp * S::RB)] = src[i];
      }
    } else if (nk == 16) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                     "r"(x2_smem(recb)), "r"(16 * S::RB)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    } else {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(recb);
      for (int i = lane; i < nk * S::RB; i += 32) dst[i] = src[i];
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int BD, int BN, int MODE, int DT>
static cudaError_t launch_x2_t(const OqCodecParams& p, const void* x, size_t n, uint8_t* out,
                               cudaStream_t st, int num_sms, const uint32_t* list,
                               const uint32_t* list_n) {
  using S = X2S<BD, BN>;
  static_assert(S::SMEM <= 227 * 1024, "shared memory budget");
  cudaError_t e = set_smem_once(compress_x2_kernel<BD, BN, MODE, DT>, S::SMEM);
  if (e != cudaSuccess) return e;
  const size_t nblk = (n + 15) / 16;
  size_t grid = (nblk + kX2Warps - 1) / kX2Warps;
  if (grid > (size_t)num_sms) grid = num_sms;
  compress_x2_kernel<BD, BN, MODE, DT>
      <<<(unsigned)grid, kX2Threads, S::SMEM, st>>>(p, x, n, out, list, list_n);
  return cudaGetLastError();
}

template <int BD, int BN, int MODE>
static cudaError_t launch_x2(const OqCodecParams& p, const void* x, int dtype, size_t n,
                             uint8_t* out, cudaStream_t st, int num_sms, const uint32_t* list,
                             const uint32_t* list_n) {
  if (dtype == OQ_BF16)
    return launch_x2_t<BD, BN, MODE, OQ_BF16>(p, x, n, out, st, num_sms, list, list_n);
  if (dtype == OQ_F16)
    return launch_x2_t<BD, BN, MODE, OQ_F16>(p, x, n, out, st, num_sms, list, list_n);
  return launch_x2_t<BD, BN, MODE, OQ_F32>(p, x, n, out, st, num_sms, list, list_n);
}

cudaError_t launch_compress_x2(const OqCodecParams& p, const void* x, int dtype, size_t n,
                               uint8_t* out, cudaStream_t st, int num_sms, const uint32_t* list,
                               const uint32_t* list_n) {
#define OQ_X2(BD, BN)                                                                             \
  if (p.b_dir == BD && p.b_nrm == BN)                                                             \
    return p.rounding == 0                                                                        \
               ? launch_x2<BD, BN, 0>(p, x, dtype, n, out, st, num_sms, list, list_n)             \
               : launch_x2<BD, BN, 2>(p, x, dtype, n, out, st, num_sms, list, list_n);
  OQ_X2(3, 1)
  OQ_X2(4, 2)
  OQ_X2(5, 3)
#undef OQ_X2
  return cudaErrorNotSupported;
}

}  // namespace oqd
