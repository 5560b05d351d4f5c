/*
 * octoquant_b200.h — C ABI of the B200-native OCTOPUS KV-cache codec hot path.
 *
 * This is the drop-in boundary for the reference's C++ API in
 * /root/reference/proj/include/octoquant (a header-only CPU library).  Every
 * entry point below names the reference interface it replaces.  Signatures
 * carry plain pointers and sizes only (no torch or CUDA types; a CUDA stream
 * is passed as `void*`, NULL = legacy default stream).  Device pointers are
 * caller-owned; an oq_codec owns only its codebook tables.
 *
 * Error behaviour mirrors the reference's exceptions:
 *   OQ_ERR_INVALID_ARGUMENT  <-> std::invalid_argument (config / shape errors)
 *   OQ_ERR_FORMAT            <-> octoquant::FormatError (corrupt codes / wire)
 * plus OQ_ERR_CUDA / OQ_ERR_UNSUPPORTED.  oq_last_error() returns the
 * thread-local message of the last failure.  There is no CPU fallback: with
 * no usable CUDA device the device entry points return OQ_ERR_CUDA.
 */
#ifndef OCTOQUANT_B200_H
#define OCTOQUANT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  OQ_OK = 0,
  OQ_ERR_INVALID_ARGUMENT = 1,
  OQ_ERR_FORMAT = 2,
  OQ_ERR_CUDA = 3,
  OQ_ERR_UNSUPPORTED = 4,
  OQ_ERR_NCCL = 5
} oq_status;

/* Rounding (codec.hpp:34) */
enum { OQ_ROUND_SCALAR = 0, OQ_ROUND_LOCAL2X2 = 1, OQ_ROUND_LOCAL3X3 = 2, OQ_ROUND_FULL = 3 };
/* Input element types accepted by oq_compress. */
enum { OQ_DTYPE_F32 = 0, OQ_DTYPE_F64 = 1, OQ_DTYPE_F16 = 2, OQ_DTYPE_BF16 = 3 };
/* Cache roles for the attention tile formats. */
enum { OQ_ROLE_K = 0, OQ_ROLE_V = 1 };

/* CodecConfig (codec.hpp:54-73), same fields and defaults. */
typedef struct oq_config {
  uint32_t dim;           /* 128 */
  uint8_t b_dir;          /* 3 */
  uint8_t b_nrm;          /* 1 */
  uint8_t rounding;       /* OQ_ROUND_LOCAL3X3 */
  uint8_t qjl;            /* 0 */
  uint64_t rotation_seed; /* 0 */
  uint64_t qjl_seed;      /* 1 */
} oq_config;

typedef struct oq_codec oq_codec;

const char* oq_last_error(void);
const char* oq_version(void);

/* ---- configuration (codec.hpp:34-80, 351-356) ---------------------------- */
oq_status oq_config_default(oq_config* cfg);                       /* CodecConfig{} */
oq_status oq_config_validate(const oq_config* cfg);                /* codec.hpp:65-72 */
oq_status oq_default_bit_split(int b, int* b_dir, int* b_nrm);     /* codec.hpp:77-80 */
oq_status oq_parse_rounding(const char* name, int* rounding);      /* codec.hpp:45-52 */
const char* oq_rounding_name(int rounding);                        /* codec.hpp:36-43 */
double oq_effective_bits_per_coord(const oq_config* cfg);          /* codec.hpp:351-356 */
size_t oq_record_bytes(const oq_config* cfg);                      /* codec.hpp:427-430 */

/* ---- codebook construction (books.hpp:69-95, lloydmax.hpp:84-236) ------- */
/* Host fp64 centroids (2^bits) and boundaries (2^bits - 1), bit-identical
 * to the reference registry. */
oq_status oq_xi_book(int bits, double* centroids, double* boundaries);
oq_status oq_rho_book(uint32_t dim, int bits, double* centroids, double* boundaries);

/* ---- Encoder(cfg) / Encoder(cfg, Books::custom(xi, rho))  codec.hpp:197-212 */
/* Builds (or reuses) the books, derives the device tables and uploads them to
 * the current CUDA device. */
oq_status oq_codec_create(const oq_config* cfg, oq_codec** out);
oq_status oq_codec_create_custom(const oq_config* cfg, const double* xi_centroids, int xi_bits,
                                 const double* rho_centroids, int rho_bits, oq_codec** out);
void oq_codec_destroy(oq_codec* codec);
oq_status oq_codec_config(const oq_codec* codec, oq_config* cfg);

/* ---- compress: Encoder::encode (codec.hpp:214-249) ----------------------
 * x: device [n, dim] of `dtype`; records: device, n * oq_record_bytes bytes,
 * written as the OCTO v1 per-key payload (codec.hpp:381-393) — the bytes
 * pack_keys emits after its 20-byte header.  Codes are bit-exact vs the
 * fp64 reference. */
oq_status oq_compress(const oq_codec* codec, const void* x, int dtype, size_t n, void* records,
                      void* stream);
/* As oq_compress, and *flagged (device uint32, may be NULL) receives how many
 * keys the certified fp32 pass could not decide and re-encoded on the exact
 * fp64 path (0 when the exact kernel ran for every key).  Replaces the same
 * reference entry point as oq_compress (codec.hpp:214-249). */
oq_status oq_compress_ex(const oq_codec* codec, const void* x, int dtype, size_t n,
                         void* records, uint32_t* flagged, void* stream);

/* ---- decode: Encoder::decode (codec.hpp:268-275) -------------------------
 * records -> out device [n, dim] fp32. */
oq_status oq_decode(const oq_codec* codec, const void* records, size_t n, float* out,
                    void* stream);

/* ---- the per-key Encoder API in exact fp64 ------------------------------
 * Bit-identical to the reference (fp64, its evaluation order, no FMA
 * contraction); these back the drop-in C++ header's per-key methods.
 * Direction table (host, no device needed): out fp64 [k*k][3] =
 * oct_decode(xi_a, xi_b) for the k xi centroids — the reference's
 * build_dir_table / Books::dirs (codec.hpp:96-141). */
oq_status oq_dir_table(const double* xi_centroids, int k, double* out);
/* Encoder::prepare (codec.hpp:282-292): q device fp64 [nq, dim] -> rot = R q
 * and, for a QJL codec, sketch = R' R q (device fp64 [nq, dim]; sketch may be
 * NULL without QJL). */
oq_status oq_prepare_f64(const oq_codec* codec, const double* q, size_t nq, double* rot,
                         double* sketch, void* stream);
/* Encoder::reconstruct_rotated (codec.hpp:252-266): records -> device fp64
 * [n, dim], unit scale, rotated frame. */
oq_status oq_reconstruct_rotated(const oq_codec* codec, const void* records, size_t n,
                                 double* out, void* stream);
/* Encoder::decode (codec.hpp:268-275) in exact fp64: records -> device fp64
 * [n, dim].  (oq_decode is the fp32 throughput path, rel. err <= 1e-5.) */
oq_status oq_decode_f64(const oq_codec* codec, const void* records, size_t n, double* out,
                        void* stream);
/* Encoder::score(prepared, k) + qjl_estimate (codec.hpp:295-311,
 * qjl.hpp:39-48): prepared rot/sketch device fp64 [nq, dim] x n records ->
 * out device fp64 [nq][n]. */
oq_status oq_score_prepared(const oq_codec* codec, const double* rot, const double* sketch,
                            size_t nq, const void* records, size_t n, double* out,
                            void* stream);

/* attention_decode(enc, q, keys, values, n_splits) (attention.hpp:50-73) in
 * fp64: Encoder::prepare + Encoder::score bit-exact, then the SoftmaxState
 * push/merge recurrence per value column on the device (device exp: agrees
 * with the reference to a few ulp).  q device fp64 [nq, dim], values device
 * fp64 [n, vdim] -> out device fp64 [nq, vdim].  The drop-in C++ header's
 * attention_decode; the throughput paths are oq_attention_decode (compressed
 * V) and oq_attention_decode_dense (fp32). */
size_t oq_attention_f64_workspace_bytes(const oq_codec* codec, size_t nq, size_t n);
oq_status oq_attention_decode_f64(const oq_codec* codec, const double* q, size_t nq,
                                  const void* records, size_t n, const double* values, int vdim,
                                  int n_splits, double* out, void* workspace, size_t ws_bytes,
                                  void* stream);

/* ---- wire: pack_keys / unpack_keys (codec.hpp:364-478) -------------------
 * An OCTO v1 blob is oq_wire_header(...) followed by the records. */
oq_status oq_wire_header(const oq_config* cfg, uint64_t count, uint8_t header[20]);
/* Checks magic/version/flags/bits/dim and the exact payload size
 * (codec.hpp:411-430); fills cfg (rounding/seeds left at defaults). */
oq_status oq_wire_parse_header(const uint8_t* blob, size_t nbytes, oq_config* cfg,
                               uint64_t* count);
/* Zero-padding checks of every record on the device (codec.hpp:447,455,459-461);
 * synchronizes `stream`; OQ_ERR_FORMAT on a violation. */
oq_status oq_validate_records(const oq_codec* codec, const void* records, size_t n,
                              void* stream);

/* ---- compressed-cache attention (attention.hpp:50-73) --------------------
 * Batched GQA decode: q [B, Hq, dim] fp32 against B x Hkv compressed streams;
 * q head h reads kv head h / (Hq / Hkv).  K and V are each compressed with
 * their own codec (V with the same OCTOPUS codec, no QJL) and stored in the
 * attention tile formats (oq_cache_pack).  out [B, Hq, dim] fp32 =
 * softmax(score(q, k_t) / sqrt(dim)) . decode(v_t), the reference's
 * attention_decode(enc_k, q, keys, Matrix{enc_v.decode(v)}, n_splits). */
typedef struct oq_attn_shape {
  int32_t B, Hq, Hkv;
  uint64_t T;             /* tokens per sequence (max when seq_lens != NULL) */
  uint64_t cap_tokens;    /* tokens allocated per (b, kv head) stream in the caches */
  const int32_t* seq_lens;/* optional device [B] lengths (<= T), NULL = all T */
} oq_attn_shape;

/* Decode-step append (the step beside attention_decode in a decoder): compress
 * one new vector per stream x [n_streams, dim] (Encoder::encode,
 * codec.hpp:214-249) and write it into token slot pos of each stream's tiles
 * (pos_dev: device int64 [n_streams], or NULL for the scalar pos), leaving the
 * stream's other tokens untouched.  records: device scratch of
 * n_streams * oq_record_bytes bytes that receives the OCTO records. */
oq_status oq_cache_append(const oq_codec* codec, int role, const void* x, int dtype,
                          uint64_t n_streams, const int64_t* pos_dev, int64_t pos, void* records,
                          void* tiles, uint64_t cap_tokens, void* stream);
/* Decode step, K and V together: encode k and v (device [n_streams][dim]) and
 * write them at token pos of every stream (as oq_cache_append).  For d = 128
 * this is ONE kernel launch (each warp encodes its stream's vector exactly,
 * QJL sidecar included, into shared memory and writes it into the tile).  k_records / v_records: optional device
 * outputs for the OCTO records (NULL: not written). */
oq_status oq_cache_append_kv(const oq_codec* ck, const oq_codec* cv, const void* k, const void* v,
                             int dtype, uint64_t n_streams, const int64_t* pos_dev, int64_t pos,
                             void* k_records, void* v_records, void* ktiles, void* vtiles,
                             uint64_t cap_tokens, void* stream);
/* Tile formats exist for dim = 128 and 2*b_dir + b_nrm in {7, 10, 13} (b = 2,
 * 3, 4 at the default split); 0 otherwise (use oq_attention_decode_dense). */
size_t oq_cache_tile_bytes(const oq_codec* codec, int role); /* bytes per 32-token tile */
size_t oq_cache_bytes(const oq_codec* codec, int role, uint64_t tokens); /* per stream */
/* records: device [n_streams][rec_stride_tokens] records of n_tokens each
 * -> tiles: device [n_streams][cap_tokens/32 tiles]. */
oq_status oq_cache_pack(const oq_codec* codec, int role, const void* records, uint64_t n_streams,
                        uint64_t n_tokens, uint64_t rec_stride_tokens, void* tiles,
                        uint64_t cap_tokens, void* stream);
/* Device scratch for the attention calls.  Its first 64 KiB hold per-stream
 * arrival counters: they must be zero when the workspace is first used (the
 * kernels leave them zero), so allocate it zero-filled. */
size_t oq_attention_workspace_bytes(const oq_codec* ck, const oq_codec* cv,
                                    const oq_attn_shape* shape, int n_splits);
oq_status oq_attention_decode(const oq_codec* ck, const oq_codec* cv, const oq_attn_shape* shape,
                              const float* q, const void* kcache, const void* vcache,
                              float* out, int n_splits, void* workspace, size_t ws_bytes,
                              void* stream);
/* Sequence sharding: the SoftmaxState (m, l, acc) of tokens [t_begin, t_end)
 * per (b, q head) -> partial [B*Hq][4 + dim] fp32 = (m, l, 0, 0, acc[dim]),
 * m the reference point l and acc are scaled to (logits in log2 units: the
 * running max, or for 2-bit tiles up to 2 below it — the kernel skips
 * rescales of small max moves; the triple stays exact either way) and acc in
 * the rotated V frame.  Chunks merge with oq_attention_combine in token order, which is
 * the reference's SoftmaxState::merge (attention.hpp:36-44). */
oq_status oq_attention_partials(const oq_codec* ck, const oq_codec* cv,
                                const oq_attn_shape* shape, const float* q, const void* kcache,
                                const void* vcache, uint64_t t_begin, uint64_t t_end,
                                float* partial, int n_splits, void* workspace, size_t ws_bytes,
                                void* stream);
/* partials[row * row_stride + part * part_stride + (m, l, 0, 0, acc...)] for
 * rows = B*Hq and n_parts chunks in token order -> out [rows][dim]
 * (finalize: acc/l with the inverse V rotation applied) or, with
 * finalize = 0, the merged partial [rows][4 + dim]. */
oq_status oq_attention_combine(const oq_codec* cv, const float* partials, int rows, int n_parts,
                               size_t row_stride, size_t part_stride, int finalize, float* out,
                               void* stream);

/* ---- sequence-sharded decode attention over NCCL -------------
 * This rank holds tokens [t_begin, t_end) of every stream in kcache/vcache
 * (tile positions as in the full cache); `comm` is an ncclComm_t of nranks
 * ranks.  The rank computes its partials (K5+K3), merges its splits (K4,
 * finalize = 0), ONE ncclAllGather moves the [B*Hq][4 + dim] partials of all
 * ranks, and every rank merges them in rank order — the chunk merge of
 * attention_decode(..., n_splits = nranks) (attention.hpp:60-69) — so out
 * [B, Hq, dim] is identical on all ranks.  NCCL (libnccl.so.2) is loaded on
 * first use; OQ_ERR_NCCL if it is unavailable or a call fails. */
size_t oq_attention_sharded_workspace_bytes(const oq_codec* ck, const oq_codec* cv,
                                            const oq_attn_shape* shape, int n_splits,
                                            int nranks);
oq_status oq_attention_decode_sharded(const oq_codec* ck, const oq_codec* cv,
                                      const oq_attn_shape* shape, const float* q,
                                      const void* kcache, const void* vcache, uint64_t t_begin,
                                      uint64_t t_end, void* nccl_comm, int nranks, float* out,
                                      int n_splits, void* workspace, size_t ws_bytes,
                                      void* stream);
/* ---- the same sequence sharding fused into the attention kernel over peer
 * memory (no collective library) -------------------------------------------
 * Each rank owns an exchange buffer of oq_attention_p2p_exchange_bytes bytes,
 * zeroed once, from oq_device_alloc; xbufs[r] is rank r's buffer as mapped in
 * THIS process (its own pointer for r == rank, oq_ipc_open of rank r's
 * oq_ipc_handle otherwise).  In ONE launch the CTA that finalises a (b, kv
 * head) stream writes this rank's merged (m, l, acc) rows into slot `rank` of
 * every rank's buffer over NVLink, releases a flag there (= epoch), waits for
 * every rank's flag in its own buffer and merges the ranks in rank order —
 * the chunk merge of attention_decode(..., n_splits = nranks)
 * (attention.hpp:60-69) — into out [B, Hq, dim], identical on all ranks.
 * epoch: nonzero, strictly increasing per call (flags are never reset).
 * Every rank must make the call (as with a collective); a missing rank makes
 * the kernel trap after 20 s.  max_ctas: 0 = one CTA per SM (tests running
 * several ranks on one GPU pass SMs / nranks so all ranks are resident).
 * workspace: oq_attention_workspace_bytes(ck, cv, shape, 0), zero-filled. */
size_t oq_attention_p2p_exchange_bytes(const oq_codec* ck, const oq_attn_shape* shape,
                                       int nranks);
oq_status oq_attention_decode_p2p(const oq_codec* ck, const oq_codec* cv,
                                  const oq_attn_shape* shape, const float* q, const void* kcache,
                                  const void* vcache, uint64_t t_begin, uint64_t t_end, int rank,
                                  int nranks, void* const* xbufs, uint32_t epoch, int max_ctas,
                                  float* out, void* workspace, size_t ws_bytes, void* stream);
/* CUDA IPC of device buffers between the ranks' processes (64-byte handles). */
oq_status oq_ipc_handle(void* dev_ptr, uint8_t handle[64]);
oq_status oq_ipc_open(const uint8_t handle[64], void** dev_ptr);
oq_status oq_ipc_close(void* dev_ptr);
/* NCCL helpers for callers without their own NCCL setup (tests, the C++
 * header): unique id (128 bytes) on one rank, broadcast it, then init. */
oq_status oq_nccl_get_unique_id(uint8_t id[128]);
oq_status oq_nccl_comm_init_rank(void** comm, int nranks, const uint8_t id[128], int rank);
oq_status oq_nccl_comm_destroy(void* comm);
/* ncclCommUserRank / ncclCommCount of a communicator (bench.py prints them). */
oq_status oq_nccl_comm_info(void* comm, int* rank, int* nranks);

/* ---- general path: any codec configuration, straight from OCTO records ----
 * Encoder::score(prepare(q), k) (codec.hpp:282-316): out[nq][n] fp32 for q
 * [nq, dim] fp32 against n records. */
oq_status oq_scores(const oq_codec* codec, const float* q, int nq, const void* records, size_t n,
                    float* out, void* stream);
/* attention_decode(enc, q, keys, values, n_splits) (attention.hpp:50-73) with
 * dense fp32 values [n, vdim] (vdim <= 256), one output row per query:
 * out [nq, vdim].  n_splits contiguous chunks merged in order. */
size_t oq_attention_dense_workspace_bytes(int nq, int n_splits, int vdim);
oq_status oq_attention_decode_dense(const oq_codec* codec, const float* q, int nq,
                                    const void* records, size_t n, const float* values,
                                    int vdim, int n_splits, float* out, void* workspace,
                                    size_t ws_bytes, void* stream);

/* ---- device memory helpers (so C/C++ callers need no CUDA headers) ------- */
oq_status oq_device_alloc(size_t bytes, void** ptr);
oq_status oq_device_free(void* ptr);
oq_status oq_device_memset(void* ptr, int value, size_t bytes);  /* synchronizes */
oq_status oq_copy_to_device(void* dst, const void* src, size_t bytes);
oq_status oq_copy_to_host(void* dst, const void* src, size_t bytes);  /* synchronizes */

/* ---- measurement support (bench.py) -------------------------------------
 * When enabled, CUDA events are recorded on the launching stream around each
 * hot kernel ("compress", "decode", "attention"); collect sums them. */
void oq_timing_enable(int on);
oq_status oq_timing_collect(const char* name, double* total_ms, int* count);

#ifdef __cplusplus
}
#endif
#endif
