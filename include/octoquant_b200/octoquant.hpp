// octoquant_b200/octoquant.hpp — drop-in C++ API for the B200 build.
//
// Mirrors the public names, signatures, value semantics and exception types
// of the reference headers under /root/reference/proj/include/octoquant/
// (codec.hpp, attention.hpp, books.hpp, lloydmax.hpp, qjl.hpp, io.hpp), so
// code written against `octoquant::` compiles unchanged after switching the
// include path and linking liboctoquant_b200.so.  Every data-path method
// runs on the GPU through the C ABI in octoquant_b200.h; the host side only
// (de)serializes codes and codebooks.  The per-key Encoder methods
// (encode, reconstruct_rotated, decode, prepare, score) are bit-identical to
// the reference (exact fp64 kernels) and reuse a per-Encoder device scratch;
// each is still one device round trip, as the reference API is per key, so
// the *_batch methods and the batched C ABI are the fast path.
#pragma once

#include <octoquant_b200.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

namespace octoquant {

// io.hpp:17-20
class FormatError : public std::runtime_error {
 public:
  explicit FormatError(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {
inline void check(oq_status s) {
  if (s == OQ_OK) return;
  const std::string msg = oq_last_error();
  if (s == OQ_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (s == OQ_ERR_FORMAT) throw FormatError(msg);
  throw std::runtime_error(msg);
}

// Device buffer owned by RAII (C-ABI allocation helpers).
class DevBuf {
 public:
  explicit DevBuf(size_t bytes) { check(oq_device_alloc(bytes, &p_)); }
  ~DevBuf() { oq_device_free(p_); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  void* get() const { return p_; }
  template <typename T>
  T* as() const { return static_cast<T*>(p_); }

 private:
  void* p_ = nullptr;
};
}  // namespace detail

// codec.hpp:34-52
enum class Rounding : std::uint8_t { scalar = 0, local2x2 = 1, local3x3 = 2, full = 3 };

inline const char* rounding_name(Rounding r) { return oq_rounding_name(static_cast<int>(r)); }

inline Rounding parse_rounding(const std::string& s) {
  int r = 0;
  detail::check(oq_parse_rounding(s.c_str(), &r));
  return static_cast<Rounding>(r);
}

// codec.hpp:54-73
struct CodecConfig {
  std::uint32_t dim = 128;
  std::uint8_t b_dir = 3;
  std::uint8_t b_nrm = 1;
  Rounding rounding = Rounding::local3x3;
  std::uint64_t rotation_seed = 0;
  bool qjl = false;
  std::uint64_t qjl_seed = 1;

  std::uint32_t n_tri() const { return (dim + 2) / 3; }
  oq_config c() const {
    return oq_config{dim, b_dir, b_nrm, static_cast<std::uint8_t>(rounding),
                     static_cast<std::uint8_t>(qjl ? 1 : 0), rotation_seed, qjl_seed};
  }
  void validate() const {
    const oq_config cc = c();
    detail::check(oq_config_validate(&cc));
  }
};

// codec.hpp:77-80
inline std::pair<int, int> default_bit_split(int b) {
  int bd = 0, bn = 0;
  detail::check(oq_default_bit_split(b, &bd, &bn));
  return {bd, bn};
}

// qjl.hpp:17-20
struct QjlSidecar {
  std::uint16_t gamma_r = 0;
  std::vector<std::uint8_t> signs;
};

// codec.hpp:82-87
struct CompressedKey {
  float gamma = 0.0f;
  std::vector<std::uint16_t> dir;
  std::vector<std::uint16_t> nrm;
  std::optional<QjlSidecar> qjl;
};

// lloydmax.hpp:23
enum class BookKind : std::uint8_t { xi = 0, rho = 1, coord = 2, custom = 3 };

// lloydmax.hpp:28-55 (registry books are host fp64, bit-identical)
struct Codebook {
  BookKind kind = BookKind::custom;
  std::uint8_t bits = 0;
  std::uint32_t dim = 0;  // 0 when the book is dimension-independent
  double lo = 0.0;
  double hi = 0.0;
  std::vector<double> centroids;   // ascending
  std::vector<double> boundaries;  // size 2^bits - 1

  std::uint32_t size() const { return static_cast<std::uint32_t>(centroids.size()); }
  void rebuild_boundaries() {
    boundaries.resize(centroids.size() - 1);
    for (std::size_t i = 0; i + 1 < centroids.size(); ++i)
      boundaries[i] = 0.5 * (centroids[i] + centroids[i + 1]);
  }
  // Count of boundaries <= x (std::upper_bound): a tie goes to the upper cell.
  std::uint32_t quantize(double x) const {
    std::uint32_t lo_i = 0, hi_i = static_cast<std::uint32_t>(boundaries.size());
    while (lo_i < hi_i) {
      const std::uint32_t mid = (lo_i + hi_i) / 2;
      if (!(x < boundaries[mid])) lo_i = mid + 1;
      else hi_i = mid;
    }
    return lo_i;
  }
  double value(std::uint32_t idx) const {
    if (idx >= centroids.size()) throw std::invalid_argument("codebook index out of range");
    return centroids[idx];
  }
};

namespace detail {
inline const Codebook& cached_book(int kind, std::uint32_t dim, int bits) {
  static std::mutex mu;
  static std::map<std::tuple<int, std::uint32_t, int>, std::unique_ptr<Codebook>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto& slot = cache[{kind, dim, bits}];
  if (!slot) {
    if (bits < 1 || bits > 12) throw std::invalid_argument("codebook bits must be in [1,12]");
    auto b = std::make_unique<Codebook>();
    b->centroids.resize(std::size_t{1} << bits);
    b->boundaries.resize((std::size_t{1} << bits) - 1);
    check(kind == 0 ? oq_xi_book(bits, b->centroids.data(), b->boundaries.data())
                    : oq_rho_book(dim, bits, b->centroids.data(), b->boundaries.data()));
    // books.hpp:69-95: xi on [-1, 1] (shared across dims); rho on [0, 1] for
    // dimension d, its domain shaved below the d = 4 pole
    b->kind = kind == 0 ? BookKind::xi : BookKind::rho;
    b->bits = static_cast<std::uint8_t>(bits);
    b->dim = kind == 0 ? 0 : dim;
    b->lo = kind == 0 ? -1.0 : 0.0;
    b->hi = kind == 0 ? 1.0 : (dim == 4 ? 1.0 - 0x1p-40 : 1.0);
    slot = std::move(b);
  }
  return *slot;
}

// little-endian field writer / bounds-checked reader (io.hpp:22-61)
template <typename T>
inline void put_le(std::vector<std::uint8_t>& out, T v) {
  std::uint8_t b[sizeof(T)];
  std::memcpy(b, &v, sizeof(T));
  out.insert(out.end(), b, b + sizeof(T));
}
class ByteReader {
 public:
  ByteReader(const std::uint8_t* p, std::size_t n) : p_(p), n_(n) {}
  template <typename T>
  T get_le() {
    if (pos_ + sizeof(T) > n_) throw FormatError("truncated stream");
    T v;
    std::memcpy(&v, p_ + pos_, sizeof(T));
    pos_ += sizeof(T);
    return v;
  }
  const std::uint8_t* take(std::size_t n) {
    if (pos_ + n > n_) throw FormatError("truncated stream");
    const std::uint8_t* r = p_ + pos_;
    pos_ += n;
    return r;
  }
  std::size_t remaining() const { return n_ - pos_; }

 private:
  const std::uint8_t* p_;
  std::size_t n_;
  std::size_t pos_ = 0;
};
}  // namespace detail

// books.hpp:69-95
inline const Codebook& xi_book(int bits) { return detail::cached_book(0, 0, bits); }
inline const Codebook& rho_book(std::uint32_t d, int bits) { return detail::cached_book(1, d, bits); }

// lloydmax.hpp:256-304 — "OCBK": magic, version 1, kind, bits, reserved 0,
// dim u32, lo / hi f64, then 2^bits f32 centroids (little-endian).
inline std::vector<std::uint8_t> serialize(const Codebook& book) {
  std::vector<std::uint8_t> out = {'O', 'C', 'B', 'K'};
  detail::put_le<std::uint8_t>(out, 1);
  detail::put_le<std::uint8_t>(out, static_cast<std::uint8_t>(book.kind));
  detail::put_le<std::uint8_t>(out, book.bits);
  detail::put_le<std::uint8_t>(out, 0);
  detail::put_le<std::uint32_t>(out, book.dim);
  detail::put_le<double>(out, book.lo);
  detail::put_le<double>(out, book.hi);
  for (double c : book.centroids) detail::put_le<float>(out, static_cast<float>(c));
  return out;
}

inline Codebook deserialize_codebook(const std::uint8_t* p, std::size_t n) {
  detail::ByteReader rd(p, n);
  if (std::memcmp(rd.take(4), "OCBK", 4) != 0) throw FormatError("bad codebook magic");
  if (rd.get_le<std::uint8_t>() != 1) throw FormatError("unsupported codebook version");
  const auto kind = rd.get_le<std::uint8_t>();
  if (kind > 3) throw FormatError("unknown codebook kind");
  const auto bits = rd.get_le<std::uint8_t>();
  if (bits < 1 || bits > 12) throw FormatError("codebook bits out of range");
  if (rd.get_le<std::uint8_t>() != 0) throw FormatError("nonzero reserved byte");
  Codebook book;
  book.kind = static_cast<BookKind>(kind);
  book.bits = bits;
  book.dim = rd.get_le<std::uint32_t>();
  book.lo = rd.get_le<double>();
  book.hi = rd.get_le<double>();
  if (!(book.hi > book.lo)) throw FormatError("bad codebook domain");
  const std::size_t K = std::size_t{1} << bits;
  if (rd.remaining() != K * 4) throw FormatError("codebook payload size mismatch");
  book.centroids.resize(K);
  for (std::size_t i = 0; i < K; ++i) {
    book.centroids[i] = rd.get_le<float>();
    if (i > 0 && !(book.centroids[i] >= book.centroids[i - 1]))
      throw FormatError("centroids not ascending");
  }
  book.rebuild_boundaries();
  return book;
}

inline Codebook deserialize_codebook(const std::vector<std::uint8_t>& bytes) {
  return deserialize_codebook(bytes.data(), bytes.size());
}

// codec.hpp:96-141
using DirTable = std::vector<std::array<double, 3>>;  // [ixi * K + ieta]

namespace detail {
inline std::shared_ptr<const DirTable> build_dir_table(const Codebook& xi) {
  const int K = static_cast<int>(xi.centroids.size());
  std::vector<double> flat(std::size_t(K) * K * 3);
  check(oq_dir_table(xi.centroids.data(), K, flat.data()));
  auto t = std::make_shared<DirTable>(std::size_t(K) * K);
  for (std::size_t i = 0; i < t->size(); ++i) (*t)[i] = {flat[3 * i], flat[3 * i + 1], flat[3 * i + 2]};
  return t;
}
inline std::shared_ptr<const DirTable> cached_dir_table(const Codebook& xi) {
  static std::mutex mu;
  static std::map<const Codebook*, std::shared_ptr<const DirTable>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(&xi);
  if (it == cache.end()) it = cache.emplace(&xi, build_dir_table(xi)).first;
  return it->second;
}
}  // namespace detail

struct Books {
  const Codebook* xi = nullptr;
  const Codebook* rho = nullptr;
  std::shared_ptr<const DirTable> dirs;
  bool custom_books = false;  // (this build: upload the caller's centroids)
  static Books standard(const CodecConfig& cfg) {
    Books b;
    b.xi = &xi_book(cfg.b_dir);
    b.rho = &rho_book(cfg.dim, cfg.b_nrm);
    b.dirs = detail::cached_dir_table(*b.xi);
    return b;
  }
  static Books custom(const Codebook& xi, const Codebook& rho) {
    Books b;
    b.xi = &xi;
    b.rho = &rho;
    b.dirs = detail::build_dir_table(xi);
    b.custom_books = true;
    return b;
  }
};

// codec.hpp:351-356
inline double effective_bits_per_coord(const CodecConfig& cfg) {
  const oq_config c = cfg.c();
  return oq_effective_bits_per_coord(&c);
}

namespace detail {
inline std::size_t record_bytes(const CodecConfig& cfg) {
  const oq_config c = cfg.c();
  return oq_record_bytes(&c);
}

// One OCTO v1 record (codec.hpp:381-393) <-> CompressedKey.
inline void put_bits(std::uint8_t* buf, std::size_t& pos, std::uint32_t v, unsigned bits) {
  for (unsigned i = 0; i < bits; ++i, ++pos)
    if ((v >> i) & 1u) buf[pos >> 3] |= static_cast<std::uint8_t>(1u << (pos & 7));
}
inline std::uint32_t get_bits(const std::uint8_t* buf, std::size_t& pos, unsigned bits) {
  std::uint32_t v = 0;
  for (unsigned i = 0; i < bits; ++i, ++pos)
    if ((buf[pos >> 3] >> (pos & 7)) & 1u) v |= 1u << i;
  return v;
}

inline void to_record(const CodecConfig& cfg, const CompressedKey& ck, std::uint8_t* rec,
                      const char* shape_err) {
  const std::uint32_t nt = cfg.n_tri();
  if (ck.dir.size() != 2 * nt || ck.nrm.size() != nt) throw std::invalid_argument(shape_err);
  if (cfg.qjl != ck.qjl.has_value())
    throw std::invalid_argument("QJL sidecar presence does not match config");
  const std::size_t db = (2 * nt * cfg.b_dir + 7) / 8, nb = (nt * cfg.b_nrm + 7) / 8;
  std::memset(rec, 0, record_bytes(cfg));
  std::memcpy(rec, &ck.gamma, 4);
  std::size_t pos = 0;
  for (auto v : ck.dir) put_bits(rec + 4, pos, v, cfg.b_dir);
  pos = 0;
  for (auto v : ck.nrm) put_bits(rec + 4 + db, pos, v, cfg.b_nrm);
  if (cfg.qjl) {
    if (ck.qjl->signs.size() != (cfg.dim + 7) / 8)
      throw std::invalid_argument("QJL sign bitmap size does not match config");
    std::memcpy(rec + 4 + db + nb, &ck.qjl->gamma_r, 2);
    std::memcpy(rec + 6 + db + nb, ck.qjl->signs.data(), (cfg.dim + 7) / 8);
  }
}

inline CompressedKey from_record(const CodecConfig& cfg, const std::uint8_t* rec) {
  const std::uint32_t nt = cfg.n_tri();
  const std::size_t db = (2 * nt * cfg.b_dir + 7) / 8, nb = (nt * cfg.b_nrm + 7) / 8;
  CompressedKey ck;
  std::memcpy(&ck.gamma, rec, 4);
  std::size_t pos = 0;
  ck.dir.resize(2 * nt);
  for (auto& v : ck.dir) v = static_cast<std::uint16_t>(get_bits(rec + 4, pos, cfg.b_dir));
  for (; pos < db * 8; ++pos)
    if ((rec[4 + (pos >> 3)] >> (pos & 7)) & 1u)
      throw FormatError("nonzero padding in direction stream");
  pos = 0;
  ck.nrm.resize(nt);
  for (auto& v : ck.nrm) v = static_cast<std::uint16_t>(get_bits(rec + 4 + db, pos, cfg.b_nrm));
  for (; pos < nb * 8; ++pos)
    if ((rec[4 + db + (pos >> 3)] >> (pos & 7)) & 1u)
      throw FormatError("nonzero padding in norm stream");
  if (cfg.qjl) {
    QjlSidecar sc;
    std::memcpy(&sc.gamma_r, rec + 4 + db + nb, 2);
    const std::uint8_t* sp = rec + 6 + db + nb;
    sc.signs.assign(sp, sp + (cfg.dim + 7) / 8);
    if (cfg.dim % 8 && (sc.signs.back() & static_cast<std::uint8_t>(0xffu << (cfg.dim % 8))))
      throw FormatError("nonzero padding in sign stream");
    ck.qjl = std::move(sc);
  }
  return ck;
}
}  // namespace detail

// codec.hpp:197-336
class Encoder {
 public:
  explicit Encoder(const CodecConfig& cfg) : cfg_(cfg) {
    cfg_.validate();
    books_ = Books::standard(cfg_);
    init();
  }
  Encoder(const CodecConfig& cfg, const Books& books) : cfg_(cfg), books_(books) {
    cfg_.validate();
    if (!books_.dirs && books_.xi) books_.dirs = detail::build_dir_table(*books_.xi);
    init();
  }

  const CodecConfig& config() const { return cfg_; }
  const Books& books() const { return books_; }
  oq_codec* handle() const { return codec_.get(); }
  std::size_t record_bytes() const { return rb_; }

  // Encoder::encode (codec.hpp:214-249): bit-exact codes from the GPU.
  CompressedKey encode(std::span<const double> k) const {
    if (k.size() != cfg_.dim) throw std::invalid_argument("key dimension mismatch");
    const auto recs = encode_batch(k.data(), 1, OQ_DTYPE_F64);
    return detail::from_record(cfg_, recs.data());
  }

  // Unit-scale reconstruction in the rotated frame (codec.hpp:252-266), exact fp64.
  std::vector<double> reconstruct_rotated(const CompressedKey& ck) const {
    return per_key_f64(ck, &oq_reconstruct_rotated);
  }

  // Encoder::decode (codec.hpp:268-275), exact fp64 (bit-identical).
  std::vector<double> decode(const CompressedKey& ck) const {
    return per_key_f64(ck, &oq_decode_f64);
  }

  // codec.hpp:277-280
  struct PreparedQuery {
    std::vector<double> rot;     // R q
    std::vector<double> sketch;  // R' R q when QJL is enabled
  };

  // Encoder::prepare (codec.hpp:282-292) on the device, exact fp64.
  PreparedQuery prepare(std::span<const double> q) const {
    if (q.size() != cfg_.dim) throw std::invalid_argument("query dimension mismatch");
    const std::size_t d = cfg_.dim, vb = d * sizeof(double);
    PreparedQuery p;
    p.rot.resize(d);
    if (cfg_.qjl) p.sketch.resize(d);
    std::lock_guard<std::mutex> lk(scratch_->mu);
    auto* buf = static_cast<std::uint8_t*>(scratch_->get(3 * vb));
    double* dq = reinterpret_cast<double*>(buf);
    double* drot = reinterpret_cast<double*>(buf + vb);
    double* dsk = reinterpret_cast<double*>(buf + 2 * vb);
    detail::check(oq_copy_to_device(dq, q.data(), vb));
    detail::check(oq_prepare_f64(codec_.get(), dq, 1, drot, dsk, nullptr));
    detail::check(oq_copy_to_host(p.rot.data(), drot, vb));
    if (cfg_.qjl) detail::check(oq_copy_to_host(p.sketch.data(), dsk, vb));
    return p;
  }

  // Factorized estimate of q^T k (codec.hpp:295-311, + qjl_estimate
  // qjl.hpp:39-48) on the device, exact fp64 (bit-identical).
  double score(const PreparedQuery& p, const CompressedKey& ck) const {
    check_codes(ck);
    if (p.rot.size() != cfg_.dim || (cfg_.qjl && ck.qjl && p.sketch.size() != cfg_.dim))
      throw std::invalid_argument("prepared query dimension mismatch");
    const std::size_t d = cfg_.dim, vb = d * sizeof(double);
    const bool use_sketch = cfg_.qjl && ck.qjl;
    std::vector<std::uint8_t> rec(rb_);
    detail::to_record(cfg_, ck, rec.data(), "code stream length mismatch");
    std::lock_guard<std::mutex> lk(scratch_->mu);
    auto* buf = static_cast<std::uint8_t*>(scratch_->get(2 * vb + 8 + rb_));
    double* drot = reinterpret_cast<double*>(buf);
    double* dsk = reinterpret_cast<double*>(buf + vb);
    double* dout = reinterpret_cast<double*>(buf + 2 * vb);
    void* drec = buf + 2 * vb + 8;
    detail::check(oq_copy_to_device(drot, p.rot.data(), vb));
    if (use_sketch) detail::check(oq_copy_to_device(dsk, p.sketch.data(), vb));
    detail::check(oq_copy_to_device(drec, rec.data(), rb_));
    detail::check(oq_score_prepared(codec_.get(), drot, use_sketch ? dsk : nullptr, 1, drec, 1,
                                    dout, nullptr));
    double out = 0.0;
    detail::check(oq_copy_to_host(&out, dout, 8));
    return out;
  }

  double score(std::span<const double> q, const CompressedKey& ck) const {
    return score(prepare(q), ck);
  }

  // ---- batched host-buffer entry points (the fast path) -------------------
  // n keys of `dtype` -> n OCTO records (n * record_bytes()).
  std::vector<std::uint8_t> encode_batch(const void* x, std::size_t n,
                                         int dtype = OQ_DTYPE_F32) const {
    const std::size_t es = dtype == OQ_DTYPE_F64 ? 8 : dtype == OQ_DTYPE_F32 ? 4 : 2;
    const std::size_t xb = n * cfg_.dim * es, xb_al = (xb + 255) & ~std::size_t{255};
    std::vector<std::uint8_t> out(n * rb_);
    std::lock_guard<std::mutex> lk(scratch_->mu);
    auto* buf = static_cast<std::uint8_t*>(scratch_->get(xb_al + out.size()));
    detail::check(oq_copy_to_device(buf, x, xb));
    detail::check(oq_compress(codec_.get(), buf, dtype, n, buf + xb_al, nullptr));
    detail::check(oq_copy_to_host(out.data(), buf + xb_al, out.size()));
    return out;
  }

  // K2 (fp32 throughput decode, rel. err <= 1e-5)
  std::vector<float> decode_batch(const std::uint8_t* recs, std::size_t n) const {
    const std::size_t rbytes = (n * rb_ + 255) & ~std::size_t{255};
    std::vector<float> out(n * cfg_.dim);
    std::lock_guard<std::mutex> lk(scratch_->mu);
    auto* buf = static_cast<std::uint8_t*>(scratch_->get(rbytes + out.size() * 4));
    detail::check(oq_copy_to_device(buf, recs, n * rb_));
    detail::check(oq_decode(codec_.get(), buf, n, reinterpret_cast<float*>(buf + rbytes), nullptr));
    detail::check(oq_copy_to_host(out.data(), buf + rbytes, out.size() * 4));
    return out;
  }

  // exact fp64 decode of n records (Encoder::decode per key, bit-identical)
  std::vector<double> decode_batch_f64(const std::uint8_t* recs, std::size_t n) const {
    const std::size_t rbytes = (n * rb_ + 255) & ~std::size_t{255};
    std::vector<double> out(n * cfg_.dim);
    std::lock_guard<std::mutex> lk(scratch_->mu);
    auto* buf = static_cast<std::uint8_t*>(scratch_->get(rbytes + out.size() * 8));
    detail::check(oq_copy_to_device(buf, recs, n * rb_));
    detail::check(oq_decode_f64(codec_.get(), buf, n, reinterpret_cast<double*>(buf + rbytes),
                                nullptr));
    detail::check(oq_copy_to_host(out.data(), buf + rbytes, out.size() * 8));
    return out;
  }

  std::vector<float> scores_batch(const float* q, int nq, const std::uint8_t* recs,
                                  std::size_t n) const {
    const std::size_t qb = (std::size_t(nq) * cfg_.dim * 4 + 255) & ~std::size_t{255};
    const std::size_t rbytes = (n * rb_ + 255) & ~std::size_t{255};
    std::vector<float> out(std::size_t(nq) * n);
    std::lock_guard<std::mutex> lk(scratch_->mu);
    auto* buf = static_cast<std::uint8_t*>(scratch_->get(qb + rbytes + out.size() * 4));
    detail::check(oq_copy_to_device(buf, q, std::size_t(nq) * cfg_.dim * 4));
    detail::check(oq_copy_to_device(buf + qb, recs, n * rb_));
    detail::check(oq_scores(codec_.get(), reinterpret_cast<float*>(buf), nq, buf + qb, n,
                            reinterpret_cast<float*>(buf + qb + rbytes), nullptr));
    detail::check(oq_copy_to_host(out.data(), buf + qb + rbytes, out.size() * 4));
    return out;
  }

  // Device scratch of this encoder (and its copies), reused across calls and
  // grown on demand, so per-key calls do not allocate; guarded by a mutex so
  // the const methods stay safe to call from several threads, as in the
  // reference.
  struct Scratch {
    std::mutex mu;
    void* buf = nullptr;
    std::size_t cap = 0;
    void* get(std::size_t n) {
      if (n > cap) {
        if (buf) oq_device_free(buf);
        buf = nullptr;
        cap = 0;
        const std::size_t want = std::max(n, std::size_t{1} << 16);
        detail::check(oq_device_alloc(want, &buf));
        cap = want;
      }
      return buf;
    }
    ~Scratch() {
      if (buf) oq_device_free(buf);
    }
  };
  Scratch& scratch() const { return *scratch_; }

 private:
  void init() {
    const oq_config c = cfg_.c();
    oq_codec* h = nullptr;
    if (books_.custom_books)
      detail::check(oq_codec_create_custom(&c, books_.xi->centroids.data(), cfg_.b_dir,
                                           books_.rho->centroids.data(), cfg_.b_nrm, &h));
    else
      detail::check(oq_codec_create(&c, &h));
    codec_ = std::shared_ptr<oq_codec>(h, oq_codec_destroy);
    rb_ = detail::record_bytes(cfg_);
    scratch_ = std::make_shared<Scratch>();
  }

  template <typename Fn>
  std::vector<double> per_key_f64(const CompressedKey& ck, Fn fn) const {
    check_codes(ck);
    std::vector<std::uint8_t> rec(rb_);
    detail::to_record(cfg_, ck, rec.data(), "code stream length mismatch");
    const std::size_t ob = cfg_.dim * sizeof(double);
    std::vector<double> out(cfg_.dim);
    std::lock_guard<std::mutex> lk(scratch_->mu);
    auto* buf = static_cast<std::uint8_t*>(scratch_->get(ob + rb_));
    detail::check(oq_copy_to_device(buf + ob, rec.data(), rb_));
    detail::check(fn(codec_.get(), buf + ob, 1, reinterpret_cast<double*>(buf), nullptr));
    detail::check(oq_copy_to_host(out.data(), buf, ob));
    return out;
  }

  // codec.hpp:319-330
  void check_codes(const CompressedKey& ck) const {
    const std::uint32_t nt = cfg_.n_tri();
    if (ck.dir.size() != 2 * nt || ck.nrm.size() != nt)
      throw FormatError("code stream length mismatch");
    const std::uint32_t kd = 1u << cfg_.b_dir, kn = 1u << cfg_.b_nrm;
    for (std::uint32_t t = 0; t < nt; ++t) {
      if (ck.dir[2 * t] >= kd || ck.dir[2 * t + 1] >= kd)
        throw FormatError("direction index out of range");
      if (ck.nrm[t] >= kn) throw FormatError("norm index out of range");
    }
  }

  CodecConfig cfg_;
  Books books_;
  std::shared_ptr<oq_codec> codec_;
  std::shared_ptr<Scratch> scratch_;
  std::size_t rb_ = 0;
};

// codec.hpp:338-348
inline CompressedKey encode_key(const CodecConfig& cfg, std::span<const double> k) {
  return Encoder(cfg).encode(k);
}
inline std::vector<double> decode_key(const CodecConfig& cfg, const CompressedKey& ck) {
  return Encoder(cfg).decode(ck);
}
inline double score(const CodecConfig& cfg, std::span<const double> q, const CompressedKey& ck) {
  return Encoder(cfg).score(q, ck);
}

// ---- wire format (codec.hpp:358-478) -----------------------------------------
inline std::vector<std::uint8_t> pack_keys(const CodecConfig& cfg,
                                           std::span<const CompressedKey> keys) {
  cfg.validate();
  const oq_config c = cfg.c();
  const std::size_t rb = detail::record_bytes(cfg);
  std::vector<std::uint8_t> out(20 + keys.size() * rb);
  detail::check(oq_wire_header(&c, keys.size(), out.data()));
  for (std::size_t i = 0; i < keys.size(); ++i)
    detail::to_record(cfg, keys[i], out.data() + 20 + i * rb, "key shape does not match config");
  return out;
}

inline std::vector<std::uint8_t> pack(const CodecConfig& cfg, const CompressedKey& ck) {
  return pack_keys(cfg, std::span<const CompressedKey>(&ck, 1));
}

struct PackedBlob {
  std::uint32_t dim = 0;
  std::uint8_t b_dir = 0;
  std::uint8_t b_nrm = 0;
  bool qjl = false;
  std::vector<CompressedKey> keys;
};

inline PackedBlob unpack_keys(const std::uint8_t* p, std::size_t n) {
  oq_config c;
  std::uint64_t count = 0;
  detail::check(oq_wire_parse_header(p, n, &c, &count));
  CodecConfig cfg;
  cfg.dim = c.dim;
  cfg.b_dir = c.b_dir;
  cfg.b_nrm = c.b_nrm;
  cfg.qjl = c.qjl != 0;
  PackedBlob blob{c.dim, c.b_dir, c.b_nrm, c.qjl != 0, {}};
  const std::size_t rb = detail::record_bytes(cfg);
  blob.keys.reserve(count);
  for (std::uint64_t i = 0; i < count; ++i)
    blob.keys.push_back(detail::from_record(cfg, p + 20 + i * rb));
  return blob;
}

inline PackedBlob unpack_keys(const std::vector<std::uint8_t>& bytes) {
  return unpack_keys(bytes.data(), bytes.size());
}

inline CompressedKey unpack(const CodecConfig& cfg, const std::vector<std::uint8_t>& bytes) {
  PackedBlob blob = unpack_keys(bytes);
  if (blob.dim != cfg.dim || blob.b_dir != cfg.b_dir || blob.b_nrm != cfg.b_nrm ||
      blob.qjl != cfg.qjl)
    throw std::invalid_argument("blob header does not match config");
  if (blob.keys.size() != 1) throw std::invalid_argument("expected a single-key blob");
  return std::move(blob.keys[0]);
}

// ---- attention (attention.hpp) ---------------------------------------------------
// io.hpp:168-177
struct Matrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<double> data;
  Matrix() = default;
  Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
  double* row(std::size_t i) { return data.data() + i * cols; }
  const double* row(std::size_t i) const { return data.data() + i * cols; }
};

// attention.hpp:20-45 — the online-softmax accumulator, same recurrence.
struct SoftmaxState {
  double m = -std::numeric_limits<double>::infinity();
  double l = 0.0;
  std::vector<double> acc;

  explicit SoftmaxState(std::size_t width = 0) : acc(width, 0.0) {}

  void push(double s, const double* v, std::size_t width) {
    const double m_new = s > m ? s : m;
    const double scale = std::exp(m - m_new);
    const double w = std::exp(s - m_new);
    l = l * scale + w;
    for (std::size_t j = 0; j < width; ++j) acc[j] = acc[j] * scale + w * v[j];
    m = m_new;
  }

  void merge(const SoftmaxState& o) {
    if (o.l == 0.0) return;
    const double m_new = m > o.m ? m : o.m;
    const double sa = std::exp(m - m_new);
    const double sb = std::exp(o.m - m_new);
    l = l * sa + o.l * sb;
    for (std::size_t j = 0; j < acc.size(); ++j) acc[j] = acc[j] * sa + o.acc[j] * sb;
    m = m_new;
  }
};

// attention.hpp:50-73 — softmax(score / sqrt(d)) . values over the compressed
// cache, n_splits chunks merged in order.  Runs on the GPU in fp64
// (oq_attention_decode_f64: prepare + score bit-exact, SoftmaxState's
// recurrence per value column).  The batched throughput paths are
// oq_attention_decode (compressed V) and oq_attention_decode_dense.
inline std::vector<double> attention_decode(const Encoder& enc, std::span<const double> q,
                                            std::span<const CompressedKey> cache,
                                            const Matrix& values, int n_splits = 1) {
  if (values.rows != cache.size()) throw std::invalid_argument("values/cache length mismatch");
  if (cache.empty()) throw std::invalid_argument("empty cache");
  if (n_splits < 1) throw std::invalid_argument("n_splits must be >= 1");
  if (q.size() != enc.config().dim) throw std::invalid_argument("query dimension mismatch");
  const std::size_t n = cache.size(), rb = enc.record_bytes(), d = enc.config().dim;
  const std::size_t vdim = values.cols;
  std::vector<std::uint8_t> recs(n * rb);
  for (std::size_t i = 0; i < n; ++i)
    detail::to_record(enc.config(), cache[i], recs.data() + i * rb, "code stream length mismatch");
  auto al = [](std::size_t b) { return (b + 255) & ~std::size_t{255}; };
  const std::size_t ws = oq_attention_f64_workspace_bytes(enc.handle(), 1, n);
  const std::size_t o_q = 0, o_r = al(d * 8), o_v = o_r + al(recs.size()),
                    o_o = o_v + al(n * vdim * 8), o_w = o_o + al(vdim * 8);
  std::vector<double> out(vdim);
  std::lock_guard<std::mutex> lk(enc.scratch().mu);
  auto* buf = static_cast<std::uint8_t*>(enc.scratch().get(o_w + ws));
  detail::check(oq_copy_to_device(buf + o_q, q.data(), d * 8));
  detail::check(oq_copy_to_device(buf + o_r, recs.data(), recs.size()));
  detail::check(oq_copy_to_device(buf + o_v, values.data.data(), n * vdim * 8));
  detail::check(oq_attention_decode_f64(enc.handle(), reinterpret_cast<double*>(buf + o_q), 1,
                                        buf + o_r, n, reinterpret_cast<double*>(buf + o_v),
                                        static_cast<int>(vdim), n_splits,
                                        reinterpret_cast<double*>(buf + o_o), buf + o_w, ws,
                                        nullptr));
  detail::check(oq_copy_to_host(out.data(), buf + o_o, vdim * 8));
  return out;
}

}  // namespace octoquant
