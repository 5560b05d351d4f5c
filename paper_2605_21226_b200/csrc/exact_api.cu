// exact_api.cu — the reference's per-key Encoder API on the GPU in exact fp64:
//   Encoder::prepare            (codec.hpp:282-292)  -> prepare_f64_kernel
//   Encoder::reconstruct_rotated (codec.hpp:252-266) -> reconstruct_kernel
//   Encoder::decode             (codec.hpp:268-275)  -> decode_f64_kernel
//   Encoder::score(prep, k)     (codec.hpp:295-311)  -> score_prepared_kernel
//   + qjl_estimate              (qjl.hpp:39-48)
// Every fp64 operation is the reference's, in its evaluation order, with no
// FMA contraction (dadd/dmul round once each), so the results are
// bit-identical to the CPU reference.  These serve the drop-in C++ header's
// per-key calls (and oq_decode_f64 for batches that want the reference's
// fp64 output); the throughput paths are K1/K2/K3.
//
// One warp per vector: the row lives in shared memory and each butterfly
// stage of fwht (rotation.hpp:20-31) is split across lanes — every (a + b,
// a - b) pair is computed exactly as the scalar loop computes it.
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace oqd {

namespace {

constexpr int kExWarps = 4;

__device__ __forceinline__ bool sign_bit(const uint32_t* mask, uint32_t i) {
  return (mask[i >> 5] >> (i & 31)) & 1u;
}

// fwht + the final scale multiply (rotation.hpp:20-31) on x[0, d).
__device__ void fwht_warp(double* x, uint32_t d, double scale, int lane) {
  for (uint32_t len = 1; len < d; len <<= 1) {
    __syncwarp();
    for (uint32_t pi = lane; pi < d / 2; pi += 32) {
      const uint32_t j = (pi / len) * 2 * len + pi % len;
      const double a = x[j], b = x[j + len];
      x[j] = dadd(a, b);
      x[j + len] = dsub(a, b);
    }
  }
  __syncwarp();
  for (uint32_t i = lane; i < d; i += 32) x[i] = dmul(x[i], scale);
  __syncwarp();
}

// Rotation::apply (rotation.hpp:46-50): y = signs * x, then fwht.
__device__ void rotate_apply(double* y, const double* x, const uint32_t* mask, uint32_t d,
                             double scale, int lane) {
  for (uint32_t i = lane; i < d; i += 32) y[i] = dflip(x[i], sign_bit(mask, i));
  fwht_warp(y, d, scale, lane);
}

__device__ __forceinline__ uint32_t dir_code(const OqCodecParams& p, const uint8_t* r,
                                             uint32_t idx) {
  return read_bits_safe(r + 4, idx * p.b_dir, p.b_dir);
}
__device__ __forceinline__ uint32_t nrm_code(const OqCodecParams& p, const uint8_t* r, uint32_t t) {
  return read_bits_safe(r + 4 + p.dir_bytes, t * p.b_nrm, p.b_nrm);
}

// reconstruct_rotated (codec.hpp:252-266) of record r into x[0, d).
__device__ void reconstruct_warp(const OqCodecParams& p, const uint8_t* r, double* x, int lane) {
  for (uint32_t t = lane; t < p.nt; t += 32) {
    const double* n = p.dirs64 + 3 * (dir_code(p, r, 2 * t) * p.K + dir_code(p, r, 2 * t + 1));
    const double rho = p.rho_c[nrm_code(p, r, t)];
    for (uint32_t j = 0; j < 3 && 3 * t + j < p.dim; ++j) x[3 * t + j] = dmul(rho, n[j]);
  }
  __syncwarp();
}

__global__ void __launch_bounds__(32 * kExWarps) prepare_f64_kernel(OqCodecParams p,
                                                                    const double* __restrict__ q,
                                                                    size_t nq, double* rot,
                                                                    double* sketch) {
  __shared__ double row[kExWarps][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t i = blockIdx.x * (size_t)kExWarps + w;
  if (i >= nq) return;
  const uint32_t d = p.dim;
  rotate_apply(row[w], q + i * d, p.sign_mask, d, p.inv_sqrt_d, lane);
  for (uint32_t e = lane; e < d; e += 32) rot[i * d + e] = row[w][e];
  if (p.qjl && sketch) {
    __syncwarp();
    // R' (R q) with the QJL rotation (qjl_seed), in place: signs then fwht
    for (uint32_t e = lane; e < d; e += 32) row[w][e] = dflip(row[w][e], sign_bit(p.qsign_mask, e));
    fwht_warp(row[w], d, p.inv_sqrt_d, lane);
    for (uint32_t e = lane; e < d; e += 32) sketch[i * d + e] = row[w][e];
  }
}

__global__ void __launch_bounds__(32 * kExWarps) reconstruct_kernel(OqCodecParams p,
                                                                    const uint8_t* __restrict__ recs,
                                                                    size_t n, double* out,
                                                                    int finish_decode) {
  __shared__ double row[kExWarps][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t i = blockIdx.x * (size_t)kExWarps + w;
  if (i >= n) return;
  const uint8_t* r = recs + i * p.rec_bytes;
  const uint32_t d = p.dim;
  reconstruct_warp(p, r, row[w], lane);
  if (finish_decode) {
    // Encoder::decode: apply_inverse (fwht, then signs; rotation.hpp:52-56),
    // then * double(gamma)
    fwht_warp(row[w], d, p.inv_sqrt_d, lane);
    float g;
    memcpy(&g, r, 4);
    const double gamma = (double)g;
    for (uint32_t e = lane; e < d; e += 32)
      out[i * d + e] = dmul(dflip(row[w][e], sign_bit(p.sign_mask, e)), gamma);
  } else {
    for (uint32_t e = lane; e < d; e += 32) out[i * d + e] = row[w][e];
  }
}

// One thread per (query, key): Encoder::score(prepared, ck), sequential fp64.
__global__ void __launch_bounds__(256) score_prepared_kernel(OqCodecParams p,
                                                             const double* __restrict__ rot,
                                                             const double* __restrict__ sketch,
                                                             size_t nq,
                                                             const uint8_t* __restrict__ recs,
                                                             size_t n, double* out) {
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (idx >= nq * n) return;
  const size_t qi = idx / n, ki = idx % n;
  const uint8_t* r = recs + ki * p.rec_bytes;
  const double* pr = rot + qi * p.dim;
  double acc = 0.0;
  for (uint32_t t = 0; t < p.nt; ++t) {
    const double* nn = p.dirs64 + 3 * (dir_code(p, r, 2 * t) * p.K + dir_code(p, r, 2 * t + 1));
    double dot = 0.0;
    for (uint32_t j = 0; j < 3 && 3 * t + j < p.dim; ++j) dot = dadd(dot, dmul(pr[3 * t + j], nn[j]));
    acc = dadd(acc, dmul(p.rho_c[nrm_code(p, r, t)], dot));
  }
  double est = acc;
  if (p.qjl && sketch) {
    // qjl_estimate (qjl.hpp:39-48)
    const uint8_t* sc = r + 4 + p.dir_bytes + p.nrm_bytes;
    const uint16_t grb = (uint16_t)(sc[0] | (sc[1] << 8));
    const uint8_t* signs = sc + 2;
    const double* sk = sketch + qi * p.dim;
    double a = 0.0;
    for (uint32_t e = 0; e < p.dim; ++e) {
      const bool pos = (signs[e >> 3] >> (e & 7)) & 1u;
      a = dadd(a, pos ? sk[e] : -sk[e]);
    }
    const double gamma_r = (double)__half2float(__ushort_as_half(grb));
    est = dadd(est, dmul(dmul(dsqrt(ddiv(1.5707963267948966, (double)p.dim)), gamma_r), a));
  }
  float g;
  memcpy(&g, r, 4);
  out[idx] = dmul((double)g, est);
}

// attention_decode's softmax read (attention.hpp:20-73) over precomputed
// scores: one thread per (query, value column) replays SoftmaxState::push over
// each of the n_splits chunks in key order and merges the chunks in order —
// the reference's recurrence in fp64 (exp is the device's, so results agree
// to a few ulp rather than bit for bit).
__global__ void __launch_bounds__(128) softmax_read_kernel(const double* __restrict__ scores,
                                                           size_t nq, size_t n,
                                                           const double* __restrict__ values,
                                                           int vdim, int n_splits,
                                                           double inv_sqrt_d, double* out) {
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (idx >= nq * (size_t)vdim) return;
  const size_t qi = idx / vdim;
  const int j = (int)(idx % vdim);
  const double* s = scores + qi * n;
  const double NEG_INF = -__longlong_as_double(0x7ff0000000000000ll);
  const size_t chunk = (n + (size_t)n_splits - 1) / (size_t)n_splits;
  double M = NEG_INF, L = 0.0, A = 0.0;  // total
  for (size_t b0 = 0; b0 < n; b0 += chunk) {
    const size_t e0 = b0 + chunk < n ? b0 + chunk : n;
    double m = NEG_INF, l = 0.0, a = 0.0;  // part
    for (size_t t = b0; t < e0; ++t) {
      const double x = dmul(s[t], inv_sqrt_d);
      const double m_new = x > m ? x : m;
      const double scale = exp(dsub(m, m_new));
      const double w = exp(dsub(x, m_new));
      l = dadd(dmul(l, scale), w);
      a = dadd(dmul(a, scale), dmul(w, values[t * vdim + j]));
      m = m_new;
    }
    if (l == 0.0) continue;  // SoftmaxState::merge skips an empty part
    const double m_new = M > m ? M : m;
    const double sa = exp(dsub(M, m_new)), sb = exp(dsub(m, m_new));
    L = dadd(dmul(L, sa), dmul(l, sb));
    A = dadd(dmul(A, sa), dmul(a, sb));
    M = m_new;
  }
  out[idx] = ddiv(A, L);
}

unsigned blocks_for(size_t n, size_t per) { return (unsigned)((n + per - 1) / per); }

}  // namespace

cudaError_t launch_prepare_f64(const OqCodecParams& p, const double* q, size_t nq, double* rot,
                               double* sketch, cudaStream_t st) {
  if (nq == 0) return cudaSuccess;
  prepare_f64_kernel<<<blocks_for(nq, kExWarps), 32 * kExWarps, 0, st>>>(p, q, nq, rot, sketch);
  return cudaGetLastError();
}

cudaError_t launch_reconstruct_f64(const OqCodecParams& p, const uint8_t* recs, size_t n,
                                   double* out, int finish_decode, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  reconstruct_kernel<<<blocks_for(n, kExWarps), 32 * kExWarps, 0, st>>>(p, recs, n, out,
                                                                        finish_decode);
  return cudaGetLastError();
}

cudaError_t launch_score_prepared(const OqCodecParams& p, const double* rot, const double* sketch,
                                  size_t nq, const uint8_t* recs, size_t n, double* out,
                                  cudaStream_t st) {
  if (nq == 0 || n == 0) return cudaSuccess;
  score_prepared_kernel<<<blocks_for(nq * n, 256), 256, 0, st>>>(p, rot, sketch, nq, recs, n, out);
  return cudaGetLastError();
}

cudaError_t launch_softmax_read(const double* scores, size_t nq, size_t n, const double* values,
                                int vdim, int n_splits, double inv_sqrt_d, double* out,
                                cudaStream_t st) {
  if (nq == 0 || vdim == 0) return cudaSuccess;
  softmax_read_kernel<<<blocks_for(nq * (size_t)vdim, 128), 128, 0, st>>>(
      scores, nq, n, values, vdim, n_splits, inv_sqrt_d, out);
  return cudaGetLastError();
}

}  // namespace oqd
