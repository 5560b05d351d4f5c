// attention_dense.cu — the reference's general attention entry points for
// ANY codec configuration (dim 4..256, b_dir / b_nrm 1..8, QJL), straight
// from OCTO records:
//   * scores:  Encoder::score(prepare(q), k) for nq queries x n keys
//     (codec.hpp:282-316, qjl.hpp:39-48);
//   * attention_decode(enc, q, keys, values, n_splits) with DENSE fp32 values
//     (attention.hpp:50-73): split-K partial SoftmaxStates + an in-order
//     merge (attention.hpp:36-44).
// fp32 arithmetic on CUDA cores; the d=128 compressed-V fast path lives in
// attention.cu.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace oqd {

namespace {

constexpr int kThreads = 128;

// In-place y = H (s .* x) / sqrt(d) over D <= 256 floats in shared memory,
// executed by the whole block (rotation.hpp:46-49).  inverse=true computes
// s .* (H x) / sqrt(d) instead (rotation.hpp:52-56).
__device__ void rotate_smem(float* x, int D, const uint32_t* mask, float scale, bool inverse) {
  if (!inverse)
    for (int i = threadIdx.x; i < D; i += blockDim.x)
      if ((mask[i >> 5] >> (i & 31)) & 1u) x[i] = -x[i];
  __syncthreads();
  for (int len = 1; len < D; len <<= 1) {
    for (int k = threadIdx.x; k < D / 2; k += blockDim.x) {
      const int i = (k / len) * 2 * len + (k % len);
      const float a = x[i], b = x[i + len];
      x[i] = a + b;
      x[i + len] = a - b;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    float v = x[i] * scale;
    if (inverse && ((mask[i >> 5] >> (i & 31)) & 1u)) v = -v;
    x[i] = v;
  }
  __syncthreads();
}

// Factorized score of one record against a prepared query (no 1/sqrt(d)).
__device__ __forceinline__ float score_record(const OqCodecParams& p, const uint8_t* r,
                                              const float* qrot, const float* qsk) {
  float acc = 0.f;
  for (uint32_t t = 0; t < p.nt; ++t) {
    const uint32_t a = read_bits_safe(r + 4, 2 * t * p.b_dir, p.b_dir);
    const uint32_t b = read_bits_safe(r + 4, (2 * t + 1) * p.b_dir, p.b_dir);
    const uint32_t ir = read_bits_safe(r + 4 + p.dir_bytes, t * p.b_nrm, p.b_nrm);
    const float4 n = reinterpret_cast<const float4*>(p.dirs32)[a * p.K + b];
    float dot = qrot[3 * t] * n.x;
    if (3 * t + 1 < p.dim) dot += qrot[3 * t + 1] * n.y;
    if (3 * t + 2 < p.dim) dot += qrot[3 * t + 2] * n.z;
    acc += p.rho32[ir] * dot;
  }
  if (p.qjl) {
    const uint8_t* q = r + 4 + p.dir_bytes + p.nrm_bytes;
    const uint16_t gr = (uint16_t)(q[0] | (q[1] << 8));
    float s = 0.f;
    for (uint32_t i = 0; i < p.dim; ++i) s += ((q[2 + (i >> 3)] >> (i & 7)) & 1u) ? qsk[i] : -qsk[i];
    acc += sqrtf(1.5707963267948966f / (float)p.dim) * __half2float(__ushort_as_half(gr)) * s;
  }
  const uint32_t gb = (uint32_t)r[0] | ((uint32_t)r[1] << 8) | ((uint32_t)r[2] << 16) |
                      ((uint32_t)r[3] << 24);
  return __uint_as_float(gb) * acc;
}

// Prepare query `qi` into shared memory: qrot = R q, qsk = R' qrot.
__device__ void prepare_query(const OqCodecParams& p, const float* q, float* qrot, float* qsk) {
  for (uint32_t i = threadIdx.x; i < p.dim; i += blockDim.x) qrot[i] = q[i];
  for (uint32_t i = p.dim + threadIdx.x; i < 3 * p.nt; i += blockDim.x) qrot[i] = 0.f;
  rotate_smem(qrot, p.dim, p.sign_mask, (float)p.inv_sqrt_d, false);
  if (p.qjl) {
    for (uint32_t i = threadIdx.x; i < p.dim; i += blockDim.x) qsk[i] = qrot[i];
    rotate_smem(qsk, p.dim, p.qsign_mask, (float)p.inv_sqrt_d, false);
  }
}

__global__ void __launch_bounds__(kThreads) scores_kernel(OqCodecParams p, const float* q,
                                                          const uint8_t* recs, size_t n,
                                                          float* out) {
  __shared__ float qrot[260], qsk[256];
  const int qi = blockIdx.y;
  prepare_query(p, q + (size_t)qi * p.dim, qrot, qsk);
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x)
    out[(size_t)qi * n + t] = score_record(p, recs + t * p.rec_bytes, qrot, qsk);
}

// One block per (query, split): chunks of kThreads tokens; each thread
// scores one token, the block updates the running max, then threads own
// value dims and accumulate exp2-weighted rows.  Partial = (m (log2
// domain), l, 0, 0, acc[vdim]).
__global__ void __launch_bounds__(kThreads) dense_partial_kernel(
    OqCodecParams p, const float* q, const uint8_t* recs, size_t n, const float* values,
    int vdim, int n_splits, float* partials, size_t part_stride) {
  __shared__ float qrot[260], qsk[256], w[kThreads];
  __shared__ float red[kThreads / 32];
  const int qi = blockIdx.y, split = blockIdx.x;
  prepare_query(p, q + (size_t)qi * p.dim, qrot, qsk);
  const size_t chunk = (n + n_splits - 1) / n_splits;
  const size_t t0 = (size_t)split * chunk, t1 = min(n, t0 + chunk);
  const float k2 = (float)p.inv_sqrt_d * 1.4426950408889634f;  // 1/sqrt(d) in log2 units
  const float NEG_INF = -__int_as_float(0x7f800000);
  float M = NEG_INF, L = 0.f;
  float acc[2] = {0.f, 0.f};  // dims tid, tid + 128 (vdim <= 256)
  for (size_t c0 = t0; c0 < t1; c0 += kThreads) {
    const size_t t = c0 + threadIdx.x;
    const float s = t < t1 ? score_record(p, recs + t * p.rec_bytes, qrot, qsk) * k2 : NEG_INF;
    float mx = s;
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    float cm = red[0];
    for (int i = 1; i < kThreads / 32; ++i) cm = fmaxf(cm, red[i]);
    const float mn = fmaxf(M, cm);
    const float f = M == NEG_INF ? 0.f : exp2f(M - mn);
    const float e = s == NEG_INF ? 0.f : exp2f(s - mn);
    w[threadIdx.x] = e;
    __syncthreads();
    float ls = e;
    for (int o = 16; o; o >>= 1) ls += __shfl_xor_sync(kFull, ls, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ls;
    __syncthreads();
    float csum = 0.f;
    for (int i = 0; i < kThreads / 32; ++i) csum += red[i];
    L = L * f + csum;
    const int nt = (int)min((size_t)kThreads, t1 - c0);
    for (int h = 0; h < 2; ++h) {
      const int d = threadIdx.x + h * kThreads;
      if (d < vdim) {
        float a = acc[h] * f;
        for (int j = 0; j < nt; ++j) a += w[j] * values[(c0 + j) * vdim + d];
        acc[h] = a;
      }
    }
    M = mn;
    __syncthreads();
  }
  float* out = partials + ((size_t)qi * n_splits + split) * part_stride;
  if (threadIdx.x == 0) {
    out[0] = M;
    out[1] = L;
    out[2] = out[3] = 0.f;
  }
  for (int h = 0; h < 2; ++h) {
    const int d = threadIdx.x + h * kThreads;
    if (d < vdim) out[4 + d] = acc[h];
  }
}

// In-order merge of n_parts partials per row (SoftmaxState::merge) -> acc/l.
__global__ void dense_combine_kernel(const float* partials, int rows, int n_parts,
                                     size_t part_stride, int vdim, float* out) {
  const int row = blockIdx.x;
  const float NEG_INF = -__int_as_float(0x7f800000);
  const float* base = partials + (size_t)row * n_parts * part_stride;
  float M = NEG_INF;
  for (int i = 0; i < n_parts; ++i)
    if (base[i * part_stride + 1] > 0.f) M = fmaxf(M, base[i * part_stride]);
  float L = 0.f;
  for (int i = 0; i < n_parts; ++i) {
    const float* pp = base + i * part_stride;
    if (pp[1] > 0.f) L += pp[1] * exp2f(pp[0] - M);
  }
  for (int d = threadIdx.x; d < vdim; d += blockDim.x) {
    float a = 0.f;
    for (int i = 0; i < n_parts; ++i) {
      const float* pp = base + i * part_stride;
      if (pp[1] > 0.f) a += pp[4 + d] * exp2f(pp[0] - M);
    }
    out[(size_t)row * vdim + d] = L > 0.f ? a / L : 0.f;
  }
}

}  // namespace

cudaError_t launch_scores(const OqCodecParams& p, const float* q, int nq, const uint8_t* recs,
                          size_t n, float* out, cudaStream_t st, int num_sms) {
  if (n == 0 || nq == 0) return cudaSuccess;
  size_t bx = (n + kThreads - 1) / kThreads;
  const size_t cap = (size_t)num_sms * 8;
  if (bx > cap) bx = cap;
  scores_kernel<<<dim3((unsigned)bx, nq), kThreads, 0, st>>>(p, q, recs, n, out);
  return cudaGetLastError();
}

size_t dense_attention_workspace(int nq, int n_splits, int vdim) {
  return (size_t)nq * n_splits * (4 + vdim) * sizeof(float);
}

cudaError_t launch_dense_attention(const OqCodecParams& p, const float* q, int nq,
                                   const uint8_t* recs, size_t n, const float* values, int vdim,
                                   int n_splits, float* workspace, float* out,
                                   cudaStream_t st) {
  const size_t stride = 4 + vdim;
  dense_partial_kernel<<<dim3(n_splits, nq), kThreads, 0, st>>>(p, q, recs, n, values, vdim,
                                                                 n_splits, workspace, stride);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dense_combine_kernel<<<nq, 128, 0, st>>>(workspace, nq, n_splits, stride, vdim, out);
  return cudaGetLastError();
}

}  // namespace oqd
