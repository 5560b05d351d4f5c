// octoquant_b200/octoquant.hpp — drop-in C++ API for the B200 build.
//
// Mirrors the public names, signatures, value semantics and exception types
// of the reference headers under /root/reference/proj/include/octoquant/
// (codec.hpp, attention.hpp, books.hpp, lloydmax.hpp, qjl.hpp, io.hpp), so
// code written against `octoquant::` compiles unchanged after switching the
// include path and linking liboctoquant_b200.so.  Every data-path method
// runs on the GPU through the C ABI in octoquant_b200.h; the host side only
// (de)serializes codes.  Per-key calls make one device round trip each, as
// the reference API is per key; the *_batch methods are the fast path.
#pragma once

#include <octoquant_b200.h>

#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
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

// lloydmax.hpp:28-55 (registry books are host fp64, bit-identical)
struct Codebook {
  std::vector<double> centroids;
  std::vector<double> boundaries;
  std::uint32_t size() const { return static_cast<std::uint32_t>(centroids.size()); }
  std::uint32_t quantize(double x) const {
    std::uint32_t lo = 0, hi = static_cast<std::uint32_t>(boundaries.size());
    while (lo < hi) {
      const std::uint32_t mid = (lo + hi) / 2;
      if (!(x < boundaries[mid])) lo = mid + 1;
      else hi = mid;
    }
    return lo;
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
    slot = std::move(b);
  }
  return *slot;
}
}  // namespace detail

// books.hpp:69-95
inline const Codebook& xi_book(int bits) { return detail::cached_book(0, 0, bits); }
inline const Codebook& rho_book(std::uint32_t d, int bits) { return detail::cached_book(1, d, bits); }

// codec.hpp:121-141
struct Books {
  const Codebook* xi = nullptr;
  const Codebook* rho = nullptr;
  bool custom_books = false;
  static Books standard(const CodecConfig& cfg) {
    return Books{&xi_book(cfg.b_dir), &rho_book(cfg.dim, cfg.b_nrm), false};
  }
  static Books custom(const Codebook& xi, const Codebook& rho) { return Books{&xi, &rho, true}; }
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
  explicit Encoder(const CodecConfig& cfg) : cfg_(cfg), books_(Books::standard(cfg)) { init(); }
  Encoder(const CodecConfig& cfg, const Books& books) : cfg_(cfg), books_(books) { init(); }

  const CodecConfig& config() const { return cfg_; }
  const Books& books() const { return books_; }
  oq_codec* handle() const { return codec_.get(); }
  std::size_t record_bytes() const { return rb_; }

  CompressedKey encode(std::span<const double> k) const {
    if (k.size() != cfg_.dim) throw std::invalid_argument("key dimension mismatch");
    const auto recs = encode_batch(k.data(), 1, OQ_DTYPE_F64);
    return detail::from_record(cfg_, recs.data());
  }

  std::vector<double> decode(const CompressedKey& ck) const {
    check_codes(ck);
    std::vector<std::uint8_t> rec(rb_);
    detail::to_record(cfg_, ck, rec.data(), "code stream length mismatch");
    const auto f = decode_batch(rec.data(), 1);
    return std::vector<double>(f.begin(), f.end());
  }

  struct PreparedQuery {
    std::vector<double> q;  // the raw query; R q is applied on the device
  };

  PreparedQuery prepare(std::span<const double> q) const {
    if (q.size() != cfg_.dim) throw std::invalid_argument("query dimension mismatch");
    return PreparedQuery{std::vector<double>(q.begin(), q.end())};
  }

  double score(const PreparedQuery& p, const CompressedKey& ck) const {
    check_codes(ck);
    std::vector<std::uint8_t> rec(rb_);
    detail::to_record(cfg_, ck, rec.data(), "code stream length mismatch");
    std::vector<float> qf(p.q.begin(), p.q.end());
    return scores_batch(qf.data(), 1, rec.data(), 1)[0];
  }

  double score(std::span<const double> q, const CompressedKey& ck) const {
    return score(prepare(q), ck);
  }

  // ---- batched host-buffer entry points (the fast path) -------------------
  // n keys of `dtype` -> n OCTO records (n * record_bytes()).
  std::vector<std::uint8_t> encode_batch(const void* x, std::size_t n,
                                         int dtype = OQ_DTYPE_F32) const {
    const std::size_t es = dtype == OQ_DTYPE_F64 ? 8 : dtype == OQ_DTYPE_F32 ? 4 : 2;
    detail::DevBuf dx(n * cfg_.dim * es), dr(n * rb_);
    detail::check(oq_copy_to_device(dx.get(), x, n * cfg_.dim * es));
    detail::check(oq_compress(codec_.get(), dx.get(), dtype, n, dr.get(), nullptr));
    std::vector<std::uint8_t> out(n * rb_);
    detail::check(oq_copy_to_host(out.data(), dr.get(), out.size()));
    return out;
  }

  std::vector<float> decode_batch(const std::uint8_t* recs, std::size_t n) const {
    detail::DevBuf dr(n * rb_), dy(n * cfg_.dim * 4);
    detail::check(oq_copy_to_device(dr.get(), recs, n * rb_));
    detail::check(oq_decode(codec_.get(), dr.get(), n, dy.as<float>(), nullptr));
    std::vector<float> out(n * cfg_.dim);
    detail::check(oq_copy_to_host(out.data(), dy.get(), out.size() * 4));
    return out;
  }

  std::vector<float> scores_batch(const float* q, int nq, const std::uint8_t* recs,
                                  std::size_t n) const {
    detail::DevBuf dq(nq * cfg_.dim * 4), dr(n * rb_), ds(nq * n * 4);
    detail::check(oq_copy_to_device(dq.get(), q, nq * cfg_.dim * 4));
    detail::check(oq_copy_to_device(dr.get(), recs, n * rb_));
    detail::check(oq_scores(codec_.get(), dq.as<float>(), nq, dr.get(), n, ds.as<float>(),
                            nullptr));
    std::vector<float> out(nq * n);
    detail::check(oq_copy_to_host(out.data(), ds.get(), out.size() * 4));
    return out;
  }

 private:
  void init() {
    cfg_.validate();
    const oq_config c = cfg_.c();
    oq_codec* h = nullptr;
    if (books_.custom_books)
      detail::check(oq_codec_create_custom(&c, books_.xi->centroids.data(), cfg_.b_dir,
                                           books_.rho->centroids.data(), cfg_.b_nrm, &h));
    else
      detail::check(oq_codec_create(&c, &h));
    codec_ = std::shared_ptr<oq_codec>(h, oq_codec_destroy);
    rb_ = detail::record_bytes(cfg_);
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

// attention.hpp:50-73 — softmax(score / sqrt(d)) . values over the compressed
// cache, n_splits chunks merged in order; runs on the GPU (fp32).
inline std::vector<double> attention_decode(const Encoder& enc, std::span<const double> q,
                                            std::span<const CompressedKey> cache,
                                            const Matrix& values, int n_splits = 1) {
  if (values.rows != cache.size()) throw std::invalid_argument("values/cache length mismatch");
  if (cache.empty()) throw std::invalid_argument("empty cache");
  if (n_splits < 1) throw std::invalid_argument("n_splits must be >= 1");
  if (q.size() != enc.config().dim) throw std::invalid_argument("query dimension mismatch");
  const std::size_t n = cache.size(), rb = enc.record_bytes();
  std::vector<std::uint8_t> recs(n * rb);
  for (std::size_t i = 0; i < n; ++i)
    detail::to_record(enc.config(), cache[i], recs.data() + i * rb, "code stream length mismatch");
  std::vector<float> qf(q.begin(), q.end()), vf(values.data.begin(), values.data.end());
  const int vdim = static_cast<int>(values.cols);
  const std::size_t ws = oq_attention_dense_workspace_bytes(1, n_splits, vdim);
  detail::DevBuf dq(qf.size() * 4), dr(recs.size()), dv(vf.size() * 4), dout(vdim * 4),
      dws(ws ? ws : 4);
  detail::check(oq_copy_to_device(dq.get(), qf.data(), qf.size() * 4));
  detail::check(oq_copy_to_device(dr.get(), recs.data(), recs.size()));
  detail::check(oq_copy_to_device(dv.get(), vf.data(), vf.size() * 4));
  detail::check(oq_attention_decode_dense(enc.handle(), dq.as<float>(), 1, dr.get(), n,
                                          dv.as<float>(), vdim, n_splits, dout.as<float>(),
                                          dws.get(), ws, nullptr));
  std::vector<float> o(vdim);
  detail::check(oq_copy_to_host(o.data(), dout.get(), vdim * 4));
  return std::vector<double>(o.begin(), o.end());
}

}  // namespace octoquant
