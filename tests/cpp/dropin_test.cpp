// dropin_test.cpp — the reference's codec/attention/wire unit tests
// (/root/reference/proj/tests/codec_test.cpp, cited per case) re-expressed
// against the B200 drop-in header: the same `octoquant::` calls, the same
// exception types, compiled with g++ and linked to liboctoquant_b200.so.
// Prints one line per case and exits non-zero on any failure.
#include <octoquant_b200/octoquant.hpp>

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <functional>
#include <random>
#include <string>
#include <vector>

using namespace octoquant;

static int g_fail = 0;
#define EXPECT(cond)                                                        \
  do {                                                                      \
    if (!(cond)) {                                                          \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
      ++g_fail;                                                             \
    }                                                                       \
  } while (0)
template <typename E>
static bool throws(const std::function<void()>& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
  }
  return false;
}

static std::vector<double> gauss(std::mt19937_64& rng, std::size_t n) {
  std::normal_distribution<double> nd;
  std::vector<double> v(n);
  for (auto& x : v) x = static_cast<float>(nd(rng));  // fp32-representable, like the tests' keys
  return v;
}

static double dot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

static void run(const char* name, const std::function<void()>& f) {
  const int before = g_fail;
  f();
  std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

int main() {
  run("Config.ValidatesFields (codec_test.cpp:40-56)", [] {
    CodecConfig cfg;
    cfg.dim = 96;
    EXPECT(throws<std::invalid_argument>([&] { cfg.validate(); }));
    cfg = CodecConfig{};
    cfg.b_dir = 9;
    EXPECT(throws<std::invalid_argument>([&] { cfg.validate(); }));
    cfg = CodecConfig{};
    cfg.qjl = true;
    cfg.qjl_seed = cfg.rotation_seed;
    EXPECT(throws<std::invalid_argument>([&] { cfg.validate(); }));
    cfg.qjl_seed = cfg.rotation_seed + 1;
    cfg.validate();
  });
  run("Config.DefaultBitSplit (codec_test.cpp:58-63)", [] {
    EXPECT((default_bit_split(3) == std::pair<int, int>{4, 2}));
    EXPECT(throws<std::invalid_argument>([] { default_bit_split(1); }));
  });
  run("Encode.ZeroKeyIsInert (codec_test.cpp:65-73)", [] {
    const Encoder enc(CodecConfig{});
    const std::vector<double> zero(128, 0.0);
    const CompressedKey ck = enc.encode(zero);
    EXPECT(ck.gamma == 0.0f);
    for (double v : enc.decode(ck)) EXPECT(v == 0.0);
  });
  run("Encode.RejectsDimensionMismatch (codec_test.cpp:75-79)", [] {
    const Encoder enc(CodecConfig{});
    const std::vector<double> k(64, 1.0);
    EXPECT(throws<std::invalid_argument>([&] { enc.encode(k); }));
  });
  run("Decode.CodeAssignmentIsIdempotent (codec_test.cpp:190-202)", [] {
    const Encoder enc(CodecConfig{});
    std::mt19937_64 rng(13);
    for (int n = 0; n < 200; ++n) {
      const auto k = gauss(rng, 128);
      const CompressedKey a = enc.encode(k);
      const CompressedKey b = enc.encode(enc.decode(a));
      EXPECT(a.dir == b.dir && a.nrm == b.nrm);
    }
  });
  run("Decode.RejectsMalformedCodes (codec_test.cpp:221-237)", [] {
    const Encoder enc(CodecConfig{});
    CompressedKey ck;
    ck.gamma = 1.0f;
    ck.dir.assign(86, 0);
    ck.nrm.assign(43, 0);
    ck.dir[0] = 8;
    EXPECT(throws<FormatError>([&] { enc.decode(ck); }));
    ck.dir[0] = 0;
    ck.nrm[3] = 2;
    EXPECT(throws<FormatError>([&] { enc.decode(ck); }));
    ck.nrm[3] = 0;
    ck.dir.pop_back();
    EXPECT(throws<FormatError>([&] { enc.decode(ck); }));
  });
  run("Score.EqualsDotWithDecode (codec_test.cpp:239-262)", [] {
    const Encoder enc(CodecConfig{});
    std::mt19937_64 rng(17);
    std::vector<CompressedKey> keys;
    std::vector<std::vector<double>> decoded;
    for (int i = 0; i < 30; ++i) {
      keys.push_back(enc.encode(gauss(rng, 128)));
      decoded.push_back(enc.decode(keys.back()));
    }
    for (int i = 0; i < 10; ++i) {
      const auto q = gauss(rng, 128);
      const auto prep = enc.prepare(q);
      for (int j = 0; j < 30; ++j) {
        const double s = enc.score(prep, keys[j]);
        const double ref = dot(q, decoded[j]);
        EXPECT(std::fabs(s - ref) <= 1e-9 * std::max(1.0, std::sqrt(dot(q, q) * dot(decoded[j], decoded[j]))));
        EXPECT(enc.score(q, keys[j]) == s);  // raw-q entry point
      }
    }
  });
  run("Score.QjlCorrectionIsSeedUnbiased (codec_test.cpp:264-299)", [] {
    // the residual r = R u - reconstruct_rotated(k) of the non-QJL stage; each
    // QJL seed's estimate of q_rot . r is score_qjl / gamma - score / gamma
    const CodecConfig cfg;
    const Encoder enc(cfg);
    std::mt19937_64 rng(19);
    const auto k = gauss(rng, 128), q = gauss(rng, 128);
    const CompressedKey ck = enc.encode(k);
    const double gamma = std::sqrt(dot(k, k));
    std::vector<double> u(128);
    for (int i = 0; i < 128; ++i) u[i] = k[i] / gamma;
    const auto ur = enc.prepare(u).rot;  // R u
    auto r = enc.reconstruct_rotated(ck);
    for (int i = 0; i < 128; ++i) r[i] = ur[i] - r[i];
    const auto q_rot = enc.prepare(q).rot;
    const double truth = dot(q_rot, r);
    const double g = ck.gamma, base = enc.score(q, ck) / g;
    std::vector<double> errs;
    for (std::uint64_t seed = 1; seed <= 512; ++seed) {
      CodecConfig qc = cfg;
      qc.qjl = true;
      qc.qjl_seed = seed;
      const Encoder eq(qc);
      const CompressedKey cq = eq.encode(k);
      EXPECT(cq.dir == ck.dir && cq.nrm == ck.nrm);
      errs.push_back(eq.score(q, cq) / g - base - truth);
    }
    double mean = 0.0;
    for (double e : errs) mean += e;
    mean /= errs.size();
    double var = 0.0;
    for (double e : errs) var += (e - mean) * (e - mean);
    var /= errs.size() - 1;
    EXPECT(std::fabs(mean) <= 3.0 * std::sqrt(var / errs.size()));
  });
  run("PreparedQuery.RotAndSketchAreRotations (codec.hpp:277-292)", [] {
    CodecConfig cfg;
    cfg.qjl = true;
    const Encoder enc(cfg);
    std::mt19937_64 rng(21);
    const auto q = gauss(rng, 128);
    const auto p = enc.prepare(q);
    EXPECT(p.rot.size() == 128 && p.sketch.size() == 128);
    EXPECT(std::fabs(dot(p.rot, p.rot) - dot(q, q)) <= 1e-12 * dot(q, q));
    EXPECT(std::fabs(dot(p.sketch, p.sketch) - dot(q, q)) <= 1e-12 * dot(q, q));
    const Encoder plain(CodecConfig{});
    EXPECT(plain.prepare(q).sketch.empty());
  });
  run("ReconstructRotated.ScoreIsGammaTimesDot (codec.hpp:252-311)", [] {
    const Encoder enc(CodecConfig{});
    std::mt19937_64 rng(22);
    for (int i = 0; i < 20; ++i) {
      const auto k = gauss(rng, 128), q = gauss(rng, 128);
      const CompressedKey ck = enc.encode(k);
      const auto ur = enc.reconstruct_rotated(ck);
      const auto p = enc.prepare(q);
      const double s = enc.score(p, ck), ref = double(ck.gamma) * dot(p.rot, ur);
      EXPECT(std::fabs(s - ref) <= 1e-12 * std::max(1.0, std::fabs(ref)) * 128);
      double n2 = 0.0;
      for (double v : ur) n2 += v * v;
      EXPECT(n2 > 0.5 && n2 < 1.5);  // unit-scale reconstruction
    }
  });
  run("Attention.SplitCountDoesNotChangeOutput (codec_test.cpp:301-336)", [] {
    const Encoder enc(CodecConfig{});
    std::mt19937_64 rng(23);
    std::vector<CompressedKey> cache;
    for (int i = 0; i < 257; ++i) cache.push_back(enc.encode(gauss(rng, 128)));
    Matrix values(257, 16);
    values.data = gauss(rng, 257 * 16);
    const auto q = gauss(rng, 128);
    const auto s1 = attention_decode(enc, q, cache, values, 1);
    const auto s8 = attention_decode(enc, q, cache, values, 8);
    for (int j = 0; j < 16; ++j) EXPECT(std::fabs(s8[j] - s1[j]) <= 1e-6);
    const auto prep = enc.prepare(q);
    std::vector<double> logits(257);
    double m = -1e300;
    for (int t = 0; t < 257; ++t) {
      logits[t] = enc.score(prep, cache[t]) / std::sqrt(128.0);
      m = std::max(m, logits[t]);
    }
    double z = 0;
    std::vector<double> ref(16, 0.0);
    for (int t = 0; t < 257; ++t) {
      const double w = std::exp(logits[t] - m);
      z += w;
      for (int j = 0; j < 16; ++j) ref[j] += w * values.row(t)[j];
    }
    for (int j = 0; j < 16; ++j) EXPECT(std::fabs(s1[j] - ref[j] / z) <= 1e-9);
  });
  run("Attention.SingleKeyReturnsItsValueRow (codec_test.cpp:338-351)", [] {
    const Encoder enc(CodecConfig{});
    std::mt19937_64 rng(29);
    const auto k = gauss(rng, 128), q = gauss(rng, 128);
    const std::vector<CompressedKey> cache = {enc.encode(k)};
    Matrix values(1, 8);
    values.data = gauss(rng, 8);
    const auto out = attention_decode(enc, q, cache, values, 1);
    for (int j = 0; j < 8; ++j) EXPECT(out[j] == values.row(0)[j]);
  });
  run("SoftmaxState.PushMergeMatchesDirect (attention.hpp:20-45)", [] {
    std::mt19937_64 rng(30);
    const auto s = gauss(rng, 40), v = gauss(rng, 40 * 4);
    SoftmaxState all(4), a(4), b(4), empty(4);
    for (int t = 0; t < 40; ++t) all.push(s[t], &v[4 * t], 4);
    for (int t = 0; t < 17; ++t) a.push(s[t], &v[4 * t], 4);
    for (int t = 17; t < 40; ++t) b.push(s[t], &v[4 * t], 4);
    a.merge(b);
    a.merge(empty);  // skipped (l == 0)
    EXPECT(std::fabs(a.l - all.l) <= 1e-12 * all.l && a.m == all.m);
    for (int j = 0; j < 4; ++j) EXPECT(std::fabs(a.acc[j] - all.acc[j]) <= 1e-12 * all.l * 10);
  });
  run("Attention.RejectsBadShapes (codec_test.cpp:353-361)", [] {
    const Encoder enc(CodecConfig{});
    const std::vector<double> q(128, 0.5);
    const Matrix values(2, 8);
    EXPECT(throws<std::invalid_argument>(
        [&] { attention_decode(enc, q, std::span<const CompressedKey>{}, values, 1); }));
  });
  run("Wire.PayloadIs43BytesAtDefaultConfig (codec_test.cpp:412-421)", [] {
    CodecConfig cfg;
    const Encoder enc(cfg);
    std::mt19937_64 rng(53);
    EXPECT(pack(cfg, enc.encode(gauss(rng, 128))).size() == 20u + 43u);
  });
  run("Wire.RoundTripAndHeaderMismatch (codec_test.cpp:423-533)", [] {
    CodecConfig cfg;
    cfg.b_dir = 4;
    cfg.b_nrm = 2;
    cfg.qjl = true;
    const Encoder enc(cfg);
    std::mt19937_64 rng(59);
    std::vector<CompressedKey> keys;
    for (int i = 0; i < 50; ++i) keys.push_back(enc.encode(gauss(rng, 128)));
    const auto blob = pack_keys(cfg, keys);
    const PackedBlob back = unpack_keys(blob);
    EXPECT(back.keys.size() == keys.size() && back.qjl);
    for (std::size_t i = 0; i < keys.size(); ++i)
      EXPECT(back.keys[i].dir == keys[i].dir && back.keys[i].nrm == keys[i].nrm &&
             back.keys[i].qjl->signs == keys[i].qjl->signs);
    CodecConfig other = cfg;
    other.b_dir = 5;
    const auto one = pack(cfg, keys[0]);
    EXPECT(throws<std::invalid_argument>([&] { unpack(other, one); }));
    auto bad = one;
    bad[0] = 'X';
    EXPECT(throws<FormatError>([&] { unpack_keys(bad); }));
    EXPECT(throws<FormatError>([&] { unpack_keys(one.data(), one.size() - 1); }));
  });
  run("Rate.EffectiveBitsPerCoordinate (codec_test.cpp:535-547)", [] {
    CodecConfig cfg;
    EXPECT(effective_bits_per_coord(cfg) == 333.0 / 128.0);
  });
  run("Quantize.CentroidsMapToThemselves (lloydmax_test.cpp:121-127)", [] {
    const Codebook& xi = xi_book(3);
    for (std::uint32_t i = 0; i < xi.size(); ++i) EXPECT(xi.quantize(xi.value(i)) == i);
  });
  run("Books.DirTableAndMetadata (codec.hpp:96-141, lloydmax.hpp:28-43)", [] {
    const CodecConfig cfg;
    const Books bk = Books::standard(cfg);
    EXPECT(bk.dirs && bk.dirs->size() == 64u);
    for (const auto& n : *bk.dirs) EXPECT(std::fabs(n[0] * n[0] + n[1] * n[1] + n[2] * n[2] - 1.0) < 1e-12);
    const Codebook& xi = xi_book(3);
    EXPECT(xi.kind == BookKind::xi && xi.bits == 3 && xi.dim == 0 && xi.lo == -1.0 && xi.hi == 1.0);
    const Codebook& rho = rho_book(128, 2);
    EXPECT(rho.kind == BookKind::rho && rho.bits == 2 && rho.dim == 128 && rho.lo == 0.0 && rho.hi == 1.0);
    Codebook c = xi;
    c.rebuild_boundaries();
    EXPECT(c.boundaries == xi.boundaries);
    const Books custom = Books::custom(xi, rho);
    EXPECT(custom.dirs && *custom.dirs == *bk.dirs);
  });
  run("BookWire.RoundTripIsByteStable (lloydmax_test.cpp:144-167)", [] {
    const Codebook& rho = rho_book(128, 3);
    const auto bytes = serialize(rho);
    const Codebook back = deserialize_codebook(bytes);
    EXPECT(serialize(back) == bytes);
    EXPECT(back.kind == rho.kind && back.bits == rho.bits && back.dim == rho.dim);
    std::mt19937_64 rng(71);
    std::uniform_real_distribution<double> ud(0.0, 1.0);
    for (int n = 0; n < 10000; ++n) {
      const double x = ud(rng);
      std::uint32_t best = 0;
      double bd = 1e300;
      for (std::uint32_t i = 0; i < back.size(); ++i) {
        const double d = std::fabs(x - back.value(i));
        if (d < bd) {
          bd = d;
          best = i;
        }
      }
      EXPECT(back.quantize(x) == best);
    }
  });
  run("BookWire.FiveBitBookStaysSmall (lloydmax_test.cpp:169-171)", [] {
    EXPECT(serialize(xi_book(5)).size() <= 256u);
  });
  run("BookWire.RejectsCorruptBlobs (lloydmax_test.cpp:173-183)", [] {
    auto bytes = serialize(xi_book(2));
    EXPECT(throws<FormatError>([&] { deserialize_codebook(bytes.data(), bytes.size() - 1); }));
    auto bad = bytes;
    bad[0] = 'X';
    EXPECT(throws<FormatError>([&] { deserialize_codebook(bad); }));
    auto unordered = bytes;
    for (int i = 0; i < 4; ++i) std::swap(unordered[28 + i], unordered[32 + i]);
    EXPECT(throws<FormatError>([&] { deserialize_codebook(unordered); }));
  });
  run("Encoder.CustomBooksFromDeserializedCodebooks (codec.hpp:134-140)", [] {
    CodecConfig cfg;
    const Codebook xi = deserialize_codebook(serialize(xi_book(cfg.b_dir)));
    const Codebook rho = deserialize_codebook(serialize(rho_book(cfg.dim, cfg.b_nrm)));
    const Encoder enc(cfg, Books::custom(xi, rho));
    std::mt19937_64 rng(73);
    const auto k = gauss(rng, 128);
    const CompressedKey ck = enc.encode(k);
    const auto dec = enc.decode(ck);
    EXPECT(dot(dec, dec) > 0.5 * dot(k, k));
  });
  std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
