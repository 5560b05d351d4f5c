// ref_shim.cpp — extern "C" bridge over the UNMODIFIED reference headers
// (/root/reference/proj/include/octoquant), compiled by oracle/Makefile into
// oracle/_ref/libocto_ref.so.  TEST INFRASTRUCTURE ONLY: used by tests/ to
// pin the C restatement (octo_oracle.c) and by bench.py as the CPU baseline
// ("kind": "reference").  Nothing here re-implements the codec: every entry
// point calls the reference's own functions.
#include <cstdint>
#include <cstring>
#include <span>
#include <thread>
#include <vector>

#include "octoquant/attention.hpp"
#include "octoquant/books.hpp"
#include "octoquant/codec.hpp"

using namespace octoquant;

namespace {

CodecConfig make_cfg(uint32_t dim, int b_dir, int b_nrm, int rounding, uint64_t rot_seed,
                     int qjl, uint64_t qjl_seed) {
  CodecConfig c;
  c.dim = dim;
  c.b_dir = static_cast<uint8_t>(b_dir);
  c.b_nrm = static_cast<uint8_t>(b_nrm);
  c.rounding = static_cast<Rounding>(rounding);
  c.rotation_seed = rot_seed;
  c.qjl = qjl != 0;
  c.qjl_seed = qjl_seed;
  return c;
}

size_t rec_bytes(const CodecConfig& c) {
  const size_t nt = c.n_tri();
  return 4 + (2 * nt * c.b_dir + 7) / 8 + (nt * c.b_nrm + 7) / 8 +
         (c.qjl ? 2 + (c.dim + 7) / 8 : 0);
}

template <typename F>
void fan_out(size_t n, int threads, F&& f) {
  if (threads <= 1 || n < 2) {
    f(size_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] { f(n * t / threads, n * (t + 1) / threads); });
  for (auto& th : pool) th.join();
}

std::vector<CompressedKey> unpack_records(const CodecConfig& c, const uint8_t* recs, size_t n) {
  const size_t rb = rec_bytes(c);
  std::vector<uint8_t> blob(20 + n * rb);
  // Build a v1 header around the records and run the reference unpacker.
  std::memcpy(blob.data(), "OCTO", 4);
  blob[4] = 1;
  blob[5] = c.qjl ? 1 : 0;
  blob[6] = c.b_dir;
  blob[7] = c.b_nrm;
  std::memcpy(blob.data() + 8, &c.dim, 4);
  const uint64_t cnt = n;
  std::memcpy(blob.data() + 12, &cnt, 8);
  std::memcpy(blob.data() + 20, recs, n * rb);
  return unpack_keys(blob).keys;
}

}  // namespace

extern "C" {

int ref_xi_book(int bits, double* c, double* b) {
  const Codebook& bk = xi_book(bits);
  std::memcpy(c, bk.centroids.data(), bk.centroids.size() * 8);
  std::memcpy(b, bk.boundaries.data(), bk.boundaries.size() * 8);
  return 0;
}

int ref_rho_book(uint32_t d, int bits, double* c, double* b) {
  const Codebook& bk = rho_book(d, bits);
  std::memcpy(c, bk.centroids.data(), bk.centroids.size() * 8);
  std::memcpy(b, bk.boundaries.data(), bk.boundaries.size() * 8);
  return 0;
}

void* ref_encoder_new(uint32_t dim, int b_dir, int b_nrm, int rounding, uint64_t rot_seed,
                      int qjl, uint64_t qjl_seed) {
  try {
    return new Encoder(make_cfg(dim, b_dir, b_nrm, rounding, rot_seed, qjl, qjl_seed));
  } catch (...) {
    return nullptr;
  }
}

void ref_encoder_free(void* e) { delete static_cast<Encoder*>(e); }

// Encoder::encode over fp32 keys (widened to fp64), serialized with the
// reference pack_keys; the 20-byte header is stripped so callers get the
// bare per-key records.
void ref_encode_f32(void* h, const float* x, size_t n, uint8_t* out, int threads) {
  const Encoder& enc = *static_cast<Encoder*>(h);
  const CodecConfig& c = enc.config();
  const size_t rb = rec_bytes(c);
  fan_out(n, threads, [&](size_t lo, size_t hi) {
    std::vector<CompressedKey> keys;
    keys.reserve(hi - lo);
    std::vector<double> k(c.dim);
    for (size_t v = lo; v < hi; ++v) {
      for (uint32_t i = 0; i < c.dim; ++i) k[i] = x[v * c.dim + i];
      keys.push_back(enc.encode(k));
    }
    const auto blob = pack_keys(c, keys);
    std::memcpy(out + lo * rb, blob.data() + 20, (hi - lo) * rb);
  });
}

// Encoder::decode of bare records; returns -1 if the reference throws.
int ref_decode(void* h, const uint8_t* recs, size_t n, double* out, int threads) {
  const Encoder& enc = *static_cast<Encoder*>(h);
  const CodecConfig& c = enc.config();
  int bad = 0;
  fan_out(n, threads, [&](size_t lo, size_t hi) {
    try {
      const auto keys = unpack_records(c, recs + lo * rec_bytes(c), hi - lo);
      for (size_t v = lo; v < hi; ++v) {
        const auto u = enc.decode(keys[v - lo]);
        std::memcpy(out + v * c.dim, u.data(), c.dim * 8);
      }
    } catch (...) {
      bad = 1;
    }
  });
  return bad ? -1 : 0;
}

double ref_score(void* h, const double* q, const uint8_t* rec) {
  const Encoder& enc = *static_cast<Encoder*>(h);
  const auto keys = unpack_records(enc.config(), rec, 1);
  return enc.score(std::span<const double>(q, enc.config().dim), keys[0]);
}

// attention_decode(enc_k, q, keys, values, n_splits) for `nq` queries that
// share one key cache (GQA group), fanned out over queries.  values is a
// dense fp64 [n, vdim] matrix (the reference signature, attention.hpp:50-53).
int ref_attention(void* hk, const double* q, size_t nq, const uint8_t* krecs, size_t n,
                  const double* values, size_t vdim, int n_splits, double* out, int threads) {
  const Encoder& enc = *static_cast<Encoder*>(hk);
  const uint32_t d = enc.config().dim;
  int bad = 0;
  try {
    const auto keys = unpack_records(enc.config(), krecs, n);
    Matrix vals(n, vdim);
    std::memcpy(vals.data.data(), values, n * vdim * 8);
    fan_out(nq, threads, [&](size_t lo, size_t hi) {
      try {
        for (size_t i = lo; i < hi; ++i) {
          const auto o = attention_decode(enc, std::span<const double>(q + i * d, d), keys,
                                          vals, n_splits);
          std::memcpy(out + i * vdim, o.data(), vdim * 8);
        }
      } catch (...) {
        bad = 1;
      }
    });
  } catch (...) {
    return -1;
  }
  return bad ? -1 : 0;
}

// Full reference pack_keys / unpack_keys round trip on bare records; returns
// the blob size, or 0 if the reference throws FormatError.
size_t ref_unpack_repack(const uint8_t* blob, size_t n, uint8_t* out) {
  try {
    const PackedBlob pb = unpack_keys(blob, n);
    CodecConfig c;
    c.dim = pb.dim;
    c.b_dir = pb.b_dir;
    c.b_nrm = pb.b_nrm;
    c.qjl = pb.qjl;
    c.qjl_seed = c.rotation_seed + 1;
    const auto re = pack_keys(c, pb.keys);
    std::memcpy(out, re.data(), re.size());
    return re.size();
  } catch (...) {
    return 0;
  }
}



// ---- CPU-resident compressed cache (bench.py's reference arm) --------------
// A reference user holds the cache as CompressedKey vectors; the records are
// unpacked once here (not per step).  Each step then runs what the reference
// needs for decode attention over a compressed K AND V cache:
// Encoder::decode of every V key into the values Matrix, and
// attention_decode(enc_k, q, keys, values) per query of the GQA group.
struct RefCache {
  const Encoder* ek;
  const Encoder* ev;
  std::vector<CompressedKey> keys, vals;
};

void* ref_cache_new(void* hk, void* hv, const uint8_t* krecs, const uint8_t* vrecs, size_t n) {
  try {
    auto* c = new RefCache{static_cast<Encoder*>(hk), static_cast<Encoder*>(hv), {}, {}};
    c->keys = unpack_records(c->ek->config(), krecs, n);
    c->vals = unpack_records(c->ev->config(), vrecs, n);
    return c;
  } catch (...) {
    return nullptr;
  }
}

void ref_cache_free(void* h) { delete static_cast<RefCache*>(h); }

int ref_cache_attention(void* h, const double* q, size_t nq, double* out, int threads) {
  const RefCache& c = *static_cast<RefCache*>(h);
  const uint32_t d = c.ek->config().dim, vd = c.ev->config().dim;
  const size_t n = c.keys.size();
  int bad = 0;
  try {
    Matrix vals(n, vd);
    fan_out(n, threads, [&](size_t lo, size_t hi) {
      try {
        for (size_t i = lo; i < hi; ++i) {
          const auto u = c.ev->decode(c.vals[i]);
          std::memcpy(vals.row(i), u.data(), vd * 8);
        }
      } catch (...) {
        bad = 1;
      }
    });
    fan_out(nq, threads, [&](size_t lo, size_t hi) {
      try {
        for (size_t i = lo; i < hi; ++i) {
          const auto o = attention_decode(*c.ek, std::span<const double>(q + i * d, d), c.keys,
                                          vals, 1);
          std::memcpy(out + i * vd, o.data(), vd * 8);
        }
      } catch (...) {
        bad = 1;
      }
    });
  } catch (...) {
    return -1;
  }
  return bad ? -1 : 0;
}

}  // extern "C"
