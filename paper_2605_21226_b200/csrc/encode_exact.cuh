// encode_exact.cuh — the exact (fp64, reference evaluation order) per-triplet
// joint rounding shared by the compress kernels, and encode_key_warp: one
// key encoded by one warp into an OCTO v1 record in shared memory (used by
// the small-batch compress kernel and the fused decode-step append).
#pragma once
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace oqd {

// Record words a warp encoder stages: the largest d = 128 record (b_dir = 8,
// b_nrm = 8, QJL) is 4 + 86 + 43 + 18 = 151 bytes.
constexpr int kRecWords = 40;

struct CompressSmem {
  double* xb;
  double* rb;
  double* rc;
  const double* dirs;
  const uint32_t* xlut;  // 1024 cells of [-1, 1]: (lo | hi << 16) index bracket
  const uint32_t* rlut;  // 1024 cells of [0, 1]
};

// Exact std::upper_bound count (lloydmax.hpp:46-49) via a 1024-cell bracket
// table: for the fp32 cell of x, every boundary below lo is < x and every
// boundary from hi on is > x (the table is built with a 1e-6 guard, far
// above the fp32 cell-position error), so when hi - lo <= 1 one exact fp64
// compare decides; wider brackets (> 1 boundary per cell) binary-search.
__device__ __forceinline__ uint32_t quantize_lut(const double* b, uint32_t nb,
                                                 const uint32_t* lut, double x, float lo,
                                                 float scale) {
  int cell = __float2int_rz(((float)x - lo) * scale);
  cell = cell < 0 ? 0 : (cell > 1023 ? 1023 : cell);
  const uint32_t e = lut[cell], l = e & 0xffff, h = e >> 16;
  if (h - l <= 1u && x == x) return l + ((l < h && !(x < b[l])) ? 1u : 0u);
  return quantize_ub(b, nb, x);
}

__device__ __forceinline__ void oct_encode_exact(double t0, double t1, double t2, double& xi,
                                                 double& eta) {
  // octahedral.hpp:22-31
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

__device__ __forceinline__ double dot3_exact(double t0, double t1, double t2, const double* n) {
  return dadd(dadd(dmul(t0, n[0]), dmul(t1, n[1])), dmul(t2, n[2]));
}

__device__ __forceinline__ uint32_t joint_round(const OqCodecParams& p, const CompressSmem& s,
                                                const float4* dirs32, double t0, double t1,
                                                double t2) {
  double xi, eta;
  oct_encode_exact(t0, t1, t2, xi, eta);
  const uint32_t K = p.K;
  const uint32_t sx = quantize_lut(s.xb, K - 1, s.xlut, xi, -1.f, 512.f);
  const uint32_t sy = quantize_lut(s.xb, K - 1, s.xlut, eta, -1.f, 512.f);
  if (p.rounding == 0) {
    double r = dsqrt(dadd(dadd(dmul(t0, t0), dmul(t1, t1)), dmul(t2, t2)));
    r = r < 0.0 ? 0.0 : (r > 1.0 ? 1.0 : r);
    const uint32_t ir = quantize_lut(s.rb, p.KR - 1, s.rlut, r, 0.f, 1024.f);
    return sx | (sy << 8) | (ir << 16);
  }
  uint32_t ax0 = sx, ax1 = sx, ay0 = sy, ay1 = sy;
  if (p.rounding == 1) {
    ax1 = min(sx + 1, K - 1);
    ay1 = min(sy + 1, K - 1);
  } else if (p.rounding == 2) {
    ax0 = sx > 0 ? sx - 1 : 0;
    ay0 = sy > 0 ? sy - 1 : 0;
    ax1 = min(sx + 1, K - 1);
    ay1 = min(sy + 1, K - 1);
  } else {
    ax0 = ay0 = 0;
    ax1 = ay1 = K - 1;
  }
  const double NINF = -__longlong_as_double(0x7ff0000000000000ll);
  double best = NINF;
  uint32_t bx = ax0, by = ay0;
  {
    // fp32 pre-screen: |s32 - s64| < 3e-7 (|t| <= 1, unit table rows), so a
    // winner ahead by > 1e-6 is the exact strict-'>' argmax as well.
    const float f0 = (float)t0, f1 = (float)t1, f2 = (float)t2;
    float b1 = -INFINITY, b2 = -INFINITY;
    uint32_t wa = ax0, wb = ay0;
    // branch-free running (best, runner-up); strict '>' keeps the first
    // of equal fp32 scores, whose zero margin then forces the exact scan
    auto cand = [&](uint32_t a, uint32_t b, bool valid) {
      const float4 nv = dirs32[valid ? a * K + b : 0];
      const float sc = valid ? fmaf(f2, nv.z, fmaf(f1, nv.y, f0 * nv.x)) : -INFINITY;
      const bool gt = sc > b1;
      b2 = fmaxf(b2, fminf(b1, sc));
      b1 = fmaxf(b1, sc);
      wa = gt ? a : wa;
      wb = gt ? b : wb;
    };
    if (p.rounding == 2) {  // fixed 3x3 window, clamped cells predicated off
      const uint32_t a0 = sx - 1, b0 = sy - 1;  // wrap to huge when sx or sy is 0
      const bool rv[3] = {a0 < K, true, sx + 1 < K}, cv[3] = {b0 < K, true, sy + 1 < K};
      const int base = (int)(sx * K + sy);
#pragma unroll
      for (int da = 0; da < 3; ++da)
#pragma unroll
        for (int db = 0; db < 3; ++db) {
          const bool valid = rv[da] && cv[db];
          const float4 nv = valid ? dirs32[base + (da - 1) * (int)K + (db - 1)]
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
          const float sc = valid ? fmaf(f2, nv.z, fmaf(f1, nv.y, f0 * nv.x)) : -INFINITY;
          const bool gt = sc > b1;
          b2 = fmaxf(b2, fminf(b1, sc));
          b1 = fmaxf(b1, sc);
          wa = gt ? sx + da - 1 : wa;
          wb = gt ? sy + db - 1 : wb;
        }
    } else {
      for (uint32_t a = ax0; a <= ax1; ++a)
        for (uint32_t b = ay0; b <= ay1; ++b) cand(a, b, true);
    }
    if (b1 - b2 > 1e-6f) {  // false for NaN and exact ties
      best = dot3_exact(t0, t1, t2, s.dirs + 3 * (wa * K + wb));
      const double cl = best < 0.0 ? 0.0 : (best > 1.0 ? 1.0 : best);
      const uint32_t ir = quantize_lut(s.rb, p.KR - 1, s.rlut, cl, 0.f, 1024.f);
      return wa | (wb << 8) | (ir << 16);
    }
  }
  if (p.rounding == 2) {
    // the clamped 3x3 window as a fixed 3x3 with invalid cells skipped: the
    // nine exact dot products are independent (issued together), the
    // strict-'>' scan over them stays in row-major order
    double sc[3][3];
#pragma unroll
    for (int da = 0; da < 3; ++da)
#pragma unroll
      for (int db = 0; db < 3; ++db) {
        const uint32_t a = min(ax0 + da, ax1), b = min(ay0 + db, ay1);
        sc[da][db] = dot3_exact(t0, t1, t2, s.dirs + 3 * (a * K + b));
      }
#pragma unroll
    for (int da = 0; da < 3; ++da)
#pragma unroll
      for (int db = 0; db < 3; ++db) {
        const uint32_t a = ax0 + da, b = ay0 + db;
        if (a <= ax1 && b <= ay1 && sc[da][db] > best) {  // strict: first row-major wins
          best = sc[da][db];
          bx = a;
          by = b;
        }
      }
  } else {
    for (uint32_t a = ax0; a <= ax1; ++a)
      for (uint32_t b = ay0; b <= ay1; ++b) {
        const double sc = dot3_exact(t0, t1, t2, s.dirs + 3 * (a * K + b));
        if (sc > best) {  // strict: ties keep the first row-major pair
          best = sc;
          bx = a;
          by = b;
        }
      }
  }
  const double cl = best < 0.0 ? 0.0 : (best > 1.0 ? 1.0 : best);
  const uint32_t ir = quantize_lut(s.rb, p.KR - 1, s.rlut, cl, 0.f, 1024.f);
  return bx | (by << 8) | (ir << 16);
}

// The reference's rotated, padded coordinates of one d = 128 key by one warp
// (Encoder::encode, codec.hpp:222-230): u = k * inv, signs, WHT with the
// reference's butterfly pairs (two in-lane stages, five shuffle stages), *
// 1/sqrt(d) -> row[0 .. 129) (row[128] = 0, the pad).  Lane l holds
// coordinates 4l .. 4l+3.  Ends with a __syncwarp.
__device__ __forceinline__ void rotate_key_warp(const OqCodecParams& p, const double (&k)[4],
                                                double inv, double* row, int lane,
                                                const uint32_t* mask = nullptr) {
  double v[4];
  // u = k * inv, signs, fwht (rotation.hpp:20-31, 46-49)
  const uint32_t sm = (mask ? mask : p.sign_mask)[lane >> 3] >> (4 * (lane & 7));
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = dflip(dmul(k[i], inv), (sm >> i) & 1u);
  {
    double a = v[0], b = v[1];
    v[0] = dadd(a, b); v[1] = dsub(a, b);
    a = v[2]; b = v[3];
    v[2] = dadd(a, b); v[3] = dsub(a, b);
    a = v[0]; b = v[2];
    v[0] = dadd(a, b); v[2] = dsub(a, b);
    a = v[1]; b = v[3];
    v[1] = dadd(a, b); v[3] = dsub(a, b);
  }
#pragma unroll
  for (int lm = 1; lm < 32; lm <<= 1) {
    const bool up = lane & lm;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double o = __shfl_xor_sync(kFull, v[i], lm);
      v[i] = up ? dsub(o, v[i]) : dadd(v[i], o);
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i) row[4 * lane + i] = dmul(v[i], p.inv_sqrt_d);
  if (lane == 0) row[128] = 0.0;  // zero pad to 3 * n_tri (codec.hpp:229-230)
  __syncwarp();
}

// The codebook tables joint_round reads, straight from global memory.
__device__ __forceinline__ CompressSmem global_tables(const OqCodecParams& p) {
  return CompressSmem{const_cast<double*>(p.xi_bnd), const_cast<double*>(p.rho_bnd),
                      const_cast<double*>(p.rho_c), p.dirs64, p.xi_lut, p.rho_lut};
}

// One key (d = 128, no QJL) by one warp, latency first.  gamma is lane 0's
// sequential sum over the shared row (codec.hpp:219-221); rotate_key_warp;
// lane l then rounds triplets l and l + 32 with joint_round reading the codec
// tables straight from global memory (L1-resident: no per-CTA staging), and
// the fields are OR-ed into the record words rec[0 .. 31] (codec.hpp:381-393).
// row: 132 doubles of warp-private shared scratch.  Ends with a __syncwarp.
__device__ __forceinline__ void encode_key_warp(const OqCodecParams& p, const void* __restrict__ x,
                                                int dtype, size_t key, double* row, uint32_t* rec,
                                                int lane) {
  double k[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    k[i] = load_as_double(x, dtype, key * 128 + 4 * lane + i);
    row[4 * lane + i] = dmul(k[i], k[i]);
  }
  rec[lane] = 0u;
  if (lane < kRecWords - 32) rec[32 + lane] = 0u;
  __syncwarp();
  double g2 = 0.0;  // squares are rounded identically in parallel: only the adds chain
  if (lane == 0)
    for (int e = 0; e < 128; ++e) g2 = dadd(g2, row[e]);
  g2 = __shfl_sync(kFull, g2, 0);
  const double gamma = dsqrt(g2);
  const double inv = ddiv(1.0, gamma > 1e-12 ? gamma : 1e-12);
  __syncwarp();
  rotate_key_warp(p, k, inv, row, lane);
  const CompressSmem tabs = global_tables(p);
  const float4* d32 = reinterpret_cast<const float4*>(p.dirs32);
  const int pb = 2 * p.b_dir, nb = p.b_nrm;
  for (int t = lane; t < 43; t += 32) {
    const uint32_t code = joint_round(p, tabs, d32, row[3 * t], row[3 * t + 1], row[3 * t + 2]);
    const uint32_t pr = (code & 0xff) | (((code >> 8) & 0xff) << p.b_dir), ir = code >> 16;
    // dir field pair t at bit 32 + pb t, norm field t at bit 32 + 8 dir_bytes + nb t
    const int dp = 32 + pb * t, np = 32 + 8 * (int)p.dir_bytes + nb * t;
    atomicOr(&rec[dp >> 5], pr << (dp & 31));
    if ((dp & 31) + pb > 32) atomicOr(&rec[(dp >> 5) + 1], pr >> (32 - (dp & 31)));
    atomicOr(&rec[np >> 5], ir << (np & 31));
    if ((np & 31) + nb > 32) atomicOr(&rec[(np >> 5) + 1], ir >> (32 - (np & 31)));
  }
  __syncwarp();
  if (lane == 0) rec[0] = __float_as_uint((float)gamma);  // codec.hpp:233
  __syncwarp();
}

// The QJL sidecar (codec.hpp:243-247, qjl.hpp:23-36) of a key encoded by
// encode_key_warp: its codes are in rec, its reference rotated coordinates in
// row[0 .. 127].  r = ur - rho_hat n_hat (reconstruct_rotated, fp64, in place
// over row), gamma_r = f16(float(sqrt(sum r^2))) with the reference's
// sequential fp64 sum, w = R' r (signs of qjl_seed, WHT, 1/sqrt d); sign bit
// i = (w_i >= 0).  Ends with a __syncwarp.
__device__ __forceinline__ uint32_t rec_bits_w(const uint32_t* w, int pos, int bits) {
  const int i = pos >> 5, sh = pos & 31;
  const uint32_t v = sh + bits > 32 ? __funnelshift_r(w[i], w[i + 1], sh) : w[i] >> sh;
  return v & ((1u << bits) - 1u);
}
__device__ __forceinline__ void qjl_key_warp(const OqCodecParams& p, double* row, uint32_t* rec,
                                             int lane, const CompressSmem& tabs) {
  const int K = (int)p.K, bd = (int)p.b_dir, bn = (int)p.b_nrm;
  double r[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int i = 4 * lane + j, t = i / 3, comp = i - 3 * t;
    const uint32_t pr = rec_bits_w(rec, 32 + 2 * bd * t, 2 * bd);
    const uint32_t ir = rec_bits_w(rec, 32 + 8 * (int)p.dir_bytes + bn * t, bn);
    const uint32_t a = pr & (uint32_t)(K - 1), b = pr >> bd;
    const double uh = dmul(tabs.rc[ir], tabs.dirs[3 * (a * (uint32_t)K + b) + comp]);
    r[j] = dsub(row[i], uh);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 4; ++j) row[4 * lane + j] = r[j];
  __syncwarp();
  double n2 = 0.0;
  if (lane == 0)
    for (int i = 0; i < 128; ++i) n2 = dadd(n2, dmul(row[i], row[i]));
  __syncwarp();
  rotate_key_warp(p, r, 1.0, row, lane, p.qsign_mask);  // w (r * 1.0 is exact)
  const int qb = 8 * (4 + (int)p.dir_bytes + (int)p.nrm_bytes);  // sidecar bit offset
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) bits |= (row[4 * lane + j] >= 0.0 ? 1u : 0u) << j;
  const int sp = qb + 16 + 4 * lane;  // sign bits LSB-first after gamma_r
  atomicOr(&rec[sp >> 5], bits << (sp & 31));
  if (lane == 0) {
    const uint32_t gr = f32_to_f16_ref((float)dsqrt(n2));
    atomicOr(&rec[qb >> 5], gr << (qb & 31));
    if ((qb & 31) > 16) atomicOr(&rec[(qb >> 5) + 1], gr >> (32 - (qb & 31)));
  }
  __syncwarp();
}

}  // namespace oqd
