/*
 * octo_oracle.h — CPU restatement of the OCTOPUS codec hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load liboctoquant_oracle.so, and only as a
 * checker.  The product (paper_2605_21226_b200/) never links or calls it.
 *
 * Parity pinning: every function below restates one reference function
 * (cited as /root/reference/proj/include/octoquant/<file>:<line>).  The
 * restatement is pinned two ways (tests/test_oracle.py):
 *   1. against the known-answer vectors of the reference's own GTest suites
 *      (rng_test.cpp, io_test.cpp, lloydmax_test.cpp, codec_test.cpp);
 *   2. against oracle/_ref/libocto_ref.so, the reference headers compiled
 *      here by oracle/Makefile, bit-for-bit on codebooks and codes.
 *
 * Plain C99 + libm; build with -O2 -ffp-contract=off (no FMA contraction, so
 * every rounding step is the one the reference's scalar code performs).
 */
#ifndef OCTO_ORACLE_H
#define OCTO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp ------------------------------------------------------------ */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_stream_child(uint64_t seed, uint64_t idx);
uint64_t orc_stream_at(uint64_t seed, uint64_t i);
/* Stream(seed).fill_gaussian(out, n) starting at counter `ctr`; returns the
 * counter after the draw. */
uint64_t orc_fill_gaussian(uint64_t seed, uint64_t ctr, double* out, size_t n);
/* rows x cols Gaussian matrix from Stream(seed), cast to fp32. */
void orc_gaussian_f32(uint64_t seed, size_t n, float* out);

/* ---- io.hpp ------------------------------------------------------------- */
uint16_t orc_f32_to_f16(float f);
float orc_f16_to_f32(uint16_t h);

/* ---- rotation.hpp / octahedral.hpp ------------------------------------- */
void orc_rotation_signs(uint32_t dim, uint64_t seed, double* signs);
void orc_fwht(double* x, size_t d);
void orc_oct_encode(const double n[3], double out[2]);
void orc_oct_decode(double xi, double eta, double out[3]);

/* ---- lloydmax.hpp / books.hpp ------------------------------------------ */
/* Codebook centroids + boundaries of the process-wide registry books. */
int orc_xi_book(int bits, double* centroids, double* boundaries);
int orc_rho_book(uint32_t dim, int bits, double* centroids, double* boundaries);
uint32_t orc_quantize(const double* boundaries, uint32_t nb, double x);

/* ---- codec.hpp ---------------------------------------------------------- */
typedef struct {
  uint32_t dim;
  uint8_t b_dir;
  uint8_t b_nrm;
  uint8_t rounding; /* 0 scalar, 1 local2x2, 2 local3x3, 3 full */
  uint8_t qjl;
  uint64_t rotation_seed;
  uint64_t qjl_seed;
} orc_config;

typedef struct orc_encoder orc_encoder;

orc_encoder* orc_encoder_new(const orc_config* cfg);
void orc_encoder_free(orc_encoder* e);
/* Per-key record size in the OCTO v1 payload (codec.hpp:381-393). */
size_t orc_record_bytes(const orc_config* cfg);

/* Encoder::encode on one fp64 key; writes one OCTO payload record. */
void orc_encode_record(const orc_encoder* e, const double* k, uint8_t* rec);
/* Batched fp32 keys -> records (fp32 widened exactly to fp64). */
void orc_encode_f32(const orc_encoder* e, const float* x, size_t n, uint8_t* recs, int threads);
/* Encoder::decode of records (fp64 out); returns 0 ok, -1 FormatError. */
int orc_decode_records(const orc_encoder* e, const uint8_t* recs, size_t n, double* out);
/* Encoder::prepare + Encoder::score(prep, ck) (fp64). */
double orc_score(const orc_encoder* e, const double* q, const uint8_t* rec);
/* attention_decode(enc_k, q, keys, values, n_splits) with values given as a
 * dense fp64 [n, vdim] matrix; returns 0 ok, -1 on invalid argument. */
int orc_attention(const orc_encoder* ek, const double* q, const uint8_t* krecs, size_t n,
                  const double* values, size_t vdim, int n_splits, double* out);
/* SoftmaxState partial of one chunk: m, l, acc[vdim] (attention.hpp:20-45). */
void orc_attention_partial(const orc_encoder* ek, const double* q, const uint8_t* krecs,
                           size_t begin, size_t end, const double* values, size_t vdim,
                           double* m, double* l, double* acc);

/* Wire: the 20-byte OCTO header (codec.hpp:369-375). */
void orc_wire_header(const orc_config* cfg, uint64_t count, uint8_t hdr[20]);
/* unpack_keys validation of a full blob; 0 ok, -1 FormatError. Fills cfg. */
int orc_unpack_check(const uint8_t* blob, size_t n, orc_config* cfg_out, uint64_t* count);

/* Helpers for tests: unpack one record into code arrays. */
int orc_record_codes(const orc_config* cfg, const uint8_t* rec, float* gamma, uint16_t* dir,
                     uint16_t* nrm, uint16_t* gamma_r, uint8_t* signs);

#ifdef __cplusplus
}
#endif
#endif
