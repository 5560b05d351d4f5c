// codec_params.h — the plain-old-data view of one codec that the kernels see.
// Built on the host from an oq_codec (capi.cpp) and passed by value.
#pragma once
#include <cstddef>
#include <cstdint>

enum { OQ_F32 = 0, OQ_F64 = 1, OQ_F16 = 2, OQ_BF16 = 3 };

struct OqCodecParams {
  uint32_t dim;       // power of two, 4..256
  uint32_t nt;        // (dim + 2) / 3 triplets
  uint32_t b_dir, b_nrm;
  uint32_t K, KR;     // 2^b_dir, 2^b_nrm
  uint32_t rounding;  // 0 scalar, 1 local2x2, 2 local3x3, 3 full
  uint32_t qjl;
  uint32_t rec_bytes;  // OCTO v1 per-key record size (codec.hpp:381-393)
  uint32_t dir_bytes, nrm_bytes;
  double inv_sqrt_d;   // 1.0 / std::sqrt(double(dim)), host-rounded (rotation.hpp:29)
  uint32_t sign_mask[8];   // rotation signs, bit i = 1 => -1 (rotation.hpp:35-40)
  uint32_t qsign_mask[8];  // QJL rotation signs (qjl_seed)
  // device tables (owned by the codec handle)
  const double* xi_bnd;    // K-1 boundaries (lloydmax.hpp:39-43)
  const double* rho_bnd;   // KR-1
  const double* rho_c;     // KR centroids (fp64)
  const double* dirs64;    // K*K*3 oct_decode(xi_a, xi_b) (codec.hpp:100-107)
  const float* dirs32;     // K*K*4 fp32 copy (x, y, z, 0)
  const float* rho32;      // KR fp32 centroids
  const uint2* jointrep;   // attention table: 2^W codes x REP dithered fp16 replicas of
                           // (rho*x, rho*y | rho*z, 0), W = 2 b_dir + b_nrm, REP = 32 for
                           // W <= 8 else 16 (joint_replicas(), capi.cpp; attention.cu)
  float dwin;              // >= max |n_a - n_b| over the direction pairs of any 3x3 window
                           // (host, fp64, rounded up): certifies the local3x3 argmax
                           // by the score DIFFERENCE's error, |dt| * |n_a - n_b|
  const uint32_t* xi_lut;  // 1024-cell index brackets over [-1, 1] (compress quantize)
  const uint32_t* rho_lut; // 1024-cell index brackets over [0, 1]
};
