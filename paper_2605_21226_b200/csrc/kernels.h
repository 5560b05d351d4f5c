// kernels.h — launcher declarations for the sm_100a kernels (host side).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "codec_params.h"

namespace oqd {

// K1: Encoder::encode -> OCTO v1 records.  d = 128 fp32 keys at the BASELINE
// bit splits take the certified fp32 pass (compress_fast.cu) and re-round the
// triplets it could not decide exactly; `flagged` (device u32, optional)
// receives how many keys had such triplets.
cudaError_t launch_compress(const OqCodecParams& p, const void* x, int dtype, size_t n,
                            uint8_t* out, cudaStream_t st, int num_sms,
                            uint32_t* flagged = nullptr);
bool compress_fast_ok(const OqCodecParams& p, int dtype, const void* x, const void* out);
cudaError_t launch_compress_x2(const OqCodecParams& p, const void* x, int dtype, size_t n,
                               uint8_t* out, cudaStream_t st, int num_sms,
                               const uint32_t* list = nullptr, const uint32_t* list_n = nullptr);
// A key the certified fp32 pass could not fully decide: the triplets whose
// decisions missed their margin (mask bit t; all 43 for a key-level miss)
// and the exact fp64 1 / max(gamma, 1e-12) (codec.hpp:222).
struct FlagEntry {
  uint32_t key, mlo, mhi, pad;
  double inv, pad2;
};
cudaError_t launch_compress_fast(const OqCodecParams& p, const void* x, int dtype, size_t n,
                                 uint8_t* out, FlagEntry* flags, uint32_t* flag_cnt,
                                 cudaStream_t st, int num_sms);
// Exact re-encode of the flagged triplets only (one warp per flagged key:
// fp64 rotation from the stored inv, joint_round per flagged triplet, fields
// patched into the record in place).
cudaError_t launch_compress_fixup(const OqCodecParams& p, const void* x, int dtype, uint8_t* out,
                                  const FlagEntry* flags, const uint32_t* flag_cnt,
                                  cudaStream_t st, int num_sms);
// K2: Encoder::decode of OCTO v1 records -> fp32 [n, dim].
cudaError_t launch_decode(const OqCodecParams& p, const uint8_t* recs, size_t n, float* out,
                          cudaStream_t st, int num_sms);
// Wire validation: zero padding bits in every record (codec.hpp:447,455,459-461).
// Sets *bad (device int) nonzero on any violation.
cudaError_t launch_validate_records(const OqCodecParams& p, const uint8_t* recs, size_t n,
                                    int* bad, cudaStream_t st, int num_sms);

// ---- the per-key Encoder API in exact fp64 (exact_api.cu) -----------------
cudaError_t launch_prepare_f64(const OqCodecParams& p, const double* q, size_t nq, double* rot,
                               double* sketch, cudaStream_t st);
// finish_decode = 0: reconstruct_rotated; 1: Encoder::decode
cudaError_t launch_reconstruct_f64(const OqCodecParams& p, const uint8_t* recs, size_t n,
                                   double* out, int finish_decode, cudaStream_t st);
cudaError_t launch_score_prepared(const OqCodecParams& p, const double* rot, const double* sketch,
                                  size_t nq, const uint8_t* recs, size_t n, double* out,
                                  cudaStream_t st);
cudaError_t launch_softmax_read(const double* scores, size_t nq, size_t n, const double* values,
                                int vdim, int n_splits, double inv_sqrt_d, double* out,
                                cudaStream_t st);

// ---- compressed-cache attention (attention.cu) ----------------------------
struct AttnArgs {
  int B, Hq, Hkv;        // batch, query heads, kv heads (Hq % Hkv == 0)
  size_t T;              // tokens in the cache (per sequence)
  size_t t_begin, t_end; // token range processed by this call (sharding)
  const int32_t* seq_lens;  // optional per-sequence lengths (device), else T
  const float* q;        // [B, Hq, D] fp32 (device)
  const uint8_t* kcache; // K tiles [B][Hkv][T/32][ktile_bytes]
  const uint8_t* vcache; // V tiles [B][Hkv][T/32][vtile_bytes]
  size_t k_tiles_cap, v_tiles_cap;  // tiles allocated per (b, kv head)
  float* partials;       // [B*Hq][n_parts][2 + D] (m, l, acc) scratch
  int n_parts;           // split-K partial slots per (b, q head)
  float* out;            // [B, Hq, D] fp32 (combine output)
  void* qfrag;           // [B*Hkv] fragment scratch (attention_qfrag_bytes each)
  // fused single-launch mode (attention_decode on one GPU): when both are set
  // the attention kernel prepares q itself and writes the final rows to out
  uint32_t* counters = nullptr;  // [B*Hkv*ceil(G/8)] zero on entry, left zero
  int out_partial = 0;  // fused: out rows are merged (m, l, 0, 0, acc[D]) partials
  uint32_t vmask[4] = {0, 0, 0, 0};  // V rotation signs (for the fused combine)
  // fused P2P sequence sharding (oq_attention_decode_p2p); p2p_nranks = 0: off
  int p2p_nranks = 0, p2p_rank = 0;
  uint32_t p2p_epoch = 0;
  uint8_t* p2p_xbuf[8] = {};
  int max_ctas = 0;  // 0: one CTA per SM
};

size_t attention_tile_bytes(const OqCodecParams& p, int role);  // role 0 = K, 1 = V
size_t attention_qfrag_bytes(const OqCodecParams& pk);
// Partial slots per (b, q head): n_splits when > 0, else the stream-K count.
int attention_num_parts(int B, int Hq, int Hkv, uint64_t T, uint64_t t0, uint64_t t1,
                        int n_splits, int num_sms);
bool attention_fast_path_ok(const OqCodecParams& pk, const OqCodecParams& pv);
// records (one (b, kv-head) stream of n tokens) -> tiles
cudaError_t launch_pack_tiles(const OqCodecParams& p, int role, const uint8_t* recs,
                              size_t n_streams, size_t n_tokens, size_t rec_stride_tokens,
                              uint8_t* tiles, size_t tiles_cap, cudaStream_t st);
// decode-step append: record recs[s] -> token slot pos (pos_dev[s] if set)
cudaError_t launch_append_token(const OqCodecParams& p, int role, const uint8_t* recs,
                                size_t n_streams, const int64_t* pos_dev, int64_t pos_scalar,
                                uint8_t* tiles, size_t tiles_cap, cudaStream_t st);
// fused decode-step append of K and V (d = 128, no QJL): encode + tile write
cudaError_t launch_append_fused(const OqCodecParams& pk, const OqCodecParams& pv, const void* xk,
                                const void* xv, int dtype, size_t n_streams,
                                const int64_t* pos_dev, int64_t pos_scalar, uint8_t* rk,
                                uint8_t* rv, uint8_t* tk, uint8_t* tv, size_t tiles_cap,
                                cudaStream_t st);
// K5: query prep -> mma fragments (a.qfrag)
cudaError_t launch_qprep(const OqCodecParams& pk, const AttnArgs& a, cudaStream_t st);
// K3: split-K partials over [t_begin, t_end)
cudaError_t launch_attention_partials(const OqCodecParams& pk, const OqCodecParams& pv,
                                      const AttnArgs& a, int splits, cudaStream_t st,
                                      int num_sms);
// K4: merge n_parts partials in order, inverse V rotation, divide by l.
// partials[row*row_stride + part*part_stride + (m, l, acc[D])]; finalize=0
// writes the merged (m, l, acc) partial instead of the output.
cudaError_t launch_attention_combine(const OqCodecParams& pv, const float* partials, int rows,
                                     int n_parts, size_t row_stride, size_t part_stride,
                                     int finalize, float* out, cudaStream_t st);

// ---- generic (any codec config) scores / dense-V attention (attention_dense.cu)
cudaError_t launch_scores(const OqCodecParams& p, const float* q, int nq, const uint8_t* recs,
                          size_t n, float* out, cudaStream_t st, int num_sms);
size_t dense_attention_workspace(int nq, int n_splits, int vdim);
cudaError_t launch_dense_attention(const OqCodecParams& p, const float* q, int nq,
                                   const uint8_t* recs, size_t n, const float* values, int vdim,
                                   int n_splits, float* workspace, float* out, cudaStream_t st);

}  // namespace oqd
