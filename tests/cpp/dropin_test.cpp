// dropin_test.cpp — the reference's codec/attention/wire unit tests
// (/root/reference/proj/tests/codec_test.cpp, cited per case) re-expressed
// against the B200 drop-in header: the same `octoquant::` calls, the same
// exception types, compiled with g++ and linked to liboctoquant_b200.so.
// Prints one line per case and exits non-zero on any failure.
#include <octoquant_b200/octoquant.hpp>

#include <cmath>
#include <cstdio>
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
  run("Score.EqualsDotWithDecode (codec_test.cpp:239-262, fp32 tolerance)", [] {
    const Encoder enc(CodecConfig{});
    std::mt19937_64 rng(17);
    for (int i = 0; i < 20; ++i) {
      const auto k = gauss(rng, 128), q = gauss(rng, 128);
      const CompressedKey ck = enc.encode(k);
      const auto dec = enc.decode(ck);
      const double s = enc.score(q, ck), ref = dot(q, dec);
      EXPECT(std::fabs(s - ref) <= 2e-6 * std::sqrt(dot(q, q) * dot(dec, dec)));
    }
  });
  run("Attention.SplitCountAndDirectSoftmax (codec_test.cpp:301-336, fp32 tolerance)", [] {
    const Encoder enc(CodecConfig{});
    std::mt19937_64 rng(23);
    std::vector<CompressedKey> cache;
    for (int i = 0; i < 257; ++i) cache.push_back(enc.encode(gauss(rng, 128)));
    Matrix values(257, 16);
    values.data = gauss(rng, 257 * 16);
    const auto q = gauss(rng, 128);
    const auto s1 = attention_decode(enc, q, cache, values, 1);
    const auto s8 = attention_decode(enc, q, cache, values, 8);
    for (int j = 0; j < 16; ++j) EXPECT(std::fabs(s8[j] - s1[j]) <= 1e-5);
    std::vector<double> logits(257);
    double m = -1e300;
    for (int t = 0; t < 257; ++t) {
      logits[t] = dot(q, enc.decode(cache[t])) / std::sqrt(128.0);
      m = std::max(m, logits[t]);
    }
    double z = 0;
    std::vector<double> ref(16, 0.0);
    for (int t = 0; t < 257; ++t) {
      const double w = std::exp(logits[t] - m);
      z += w;
      for (int j = 0; j < 16; ++j) ref[j] += w * values.row(t)[j];
    }
    for (int j = 0; j < 16; ++j) EXPECT(std::fabs(s1[j] - ref[j] / z) <= 1e-5);
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
  std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
