// capi.cpp — the oq_* C ABI (include/octoquant_b200.h): argument validation
// with the reference's error semantics, codec construction (host books ->
// device tables) and kernel dispatch.  No CPU compute path exists here: every
// data-path entry point launches an sm_100a kernel.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/octoquant_b200.h"
#include "books.hpp"
#include "codec_params.h"
#include "kernels.h"

struct oq_codec {
  oq_config cfg;
  OqCodecParams p;
  int device = 0;
  int num_sms = 148;
  std::vector<void*> allocs;
  std::vector<double> xi_c, rho_c;  // host copies (centroids)
};

namespace {

thread_local std::string g_err;

// ---- optional CUDA-event timing of the hot kernels (bench.py) -------------
// Events are recorded on the launching stream around each timed launch.
struct KernelTimer {
  bool on = false;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
} g_timer;

struct TimedScope {
  const char* name;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  TimedScope(const char* n, cudaStream_t s) : name(n), st(s) {
    if (!g_timer.on) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
  }
  ~TimedScope() {
    if (!a) return;
    cudaEventRecord(b, st);
    g_timer.marks.push_back({name, {a, b}});
  }
};

oq_status fail(oq_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

struct FormatErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

bool is_pow2(uint32_t v) { return v && !(v & (v - 1)); }

size_t rec_bytes(const oq_config& c) {
  const size_t nt = (c.dim + 2) / 3;
  return 4 + (2 * nt * c.b_dir + 7) / 8 + (nt * c.b_nrm + 7) / 8 +
         (c.qjl ? 2 + (c.dim + 7) / 8 : 0);
}

oq_status validate(const oq_config* c) {
  if (!c) return fail(OQ_ERR_INVALID_ARGUMENT, "null config");
  if (!is_pow2(c->dim) || c->dim < 4)
    return fail(OQ_ERR_INVALID_ARGUMENT, "codec dim must be a power of two, >= 4");
  if (c->b_dir < 1 || c->b_dir > 8 || c->b_nrm < 1 || c->b_nrm > 8)
    return fail(OQ_ERR_INVALID_ARGUMENT, "codec bits must be in [1,8]");
  if (c->qjl && c->qjl_seed == c->rotation_seed)
    return fail(OQ_ERR_INVALID_ARGUMENT, "qjl_seed must differ from rotation_seed");
  if (c->rounding > 3) return fail(OQ_ERR_INVALID_ARGUMENT, "unknown rounding mode");
  return OQ_OK;
}

oq_status cuda_fail(cudaError_t e, const char* what) {
  return fail(OQ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
oq_status upload(oq_codec* c, const std::vector<T>& h, const T** out) {
  void* d = nullptr;
  const size_t bytes = std::max<size_t>(h.size() * sizeof(T), 16);
  cudaError_t e = cudaMalloc(&d, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  c->allocs.push_back(d);
  if (!h.empty()) {
    e = cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy");
  }
  *out = static_cast<const T*>(d);
  return OQ_OK;
}

// Index brackets for quantize (compress.cu quantize_lut): cell c of [lo, hi]
// stores lo | hi << 16 with every boundary < cell_start - 1e-6 counted in lo
// and every boundary <= cell_end + 1e-6 counted in hi.
std::vector<uint32_t> bracket_lut(const std::vector<double>& b, double lo, double hi) {
  std::vector<uint32_t> lut(1024);
  const double w = (hi - lo) / 1024.0;
  for (int c = 0; c < 1024; ++c) {
    const double x0 = lo + c * w - 1e-6, x1 = lo + (c + 1) * w + 1e-6;
    uint32_t l = 0, h = 0;
    for (double v : b) {
      l += v < x0 ? 1u : 0u;
      h += v <= x1 ? 1u : 0u;
    }
    if (c == 1023) h = (uint32_t)b.size();  // x clamped into the last cell
    if (c == 0) l = 0;
    lut[c] = l | (h << 16);
  }
  return lut;
}

// fp16 neighbours of x: the largest fp16 <= x and the smallest fp16 >= x.
void f16_bracket(double x, uint16_t& lo, uint16_t& hi) {
  const __half h = __double2half(x);  // round to nearest
  uint16_t b;
  std::memcpy(&b, &h, 2);
  auto val = [](uint16_t v) {
    __half t;
    std::memcpy(&t, &v, 2);
    return static_cast<double>(__half2float(t));
  };
  // step one fp16 up / down in value (sign-magnitude encoding)
  auto up = [](uint16_t v) -> uint16_t {
    if (v == 0x8000u) return 0x0001u;
    return (v & 0x8000u) ? uint16_t(v - 1) : uint16_t(v + 1);
  };
  auto down = [](uint16_t v) -> uint16_t {
    if (v == 0x0000u) return 0x8001u;
    return (v & 0x8000u) ? uint16_t(v + 1) : uint16_t(v - 1);
  };
  const double hv = val(b);
  if (hv == x) {
    lo = hi = b;
  } else if (hv < x) {
    lo = b;
    hi = up(b);
  } else {
    hi = b;
    lo = down(b);
  }
}

// The attention kernel's dequant table, staged verbatim into shared memory:
// for every joint code (ixi | ieta << b_dir | irho << 2 b_dir) REP fp16
// replicas of (rho x, rho y | rho z, 0), DITHERED.  Each component is rounded
// down in some replicas and up in the others — k of REP take the upper
// neighbour, k = round(REP * (x - lo) / (hi - lo)), replica r when
// bitrev(r) < k — so the mean over the replicas is within ulp / (2 REP) of
// the exact fp64 value.  K3 reads a code through a replica that varies with
// the token (attention.cu), so the fp16 rounding of the table no longer acts
// as a fixed per-code bias that the softmax average over a long context
// cannot remove (T = 128K, b = 3: 1.2e-3 -> 5e-4 relative error;
// T = 256K, b = 2: 7.7e-3 -> 6e-4; tools/exp/k3_numerics.py).
std::vector<uint2> joint_replicas(const std::vector<double>& dirs64, const std::vector<double>& rho_c,
                                  uint32_t b_dir, uint32_t b_nrm) {
  const uint32_t W = 2 * b_dir + b_nrm, K = 1u << b_dir;
  // replica count per entry: attention.cu table_rep()
  const uint32_t REP = W <= 8 ? 32 : W <= 10 ? 16 : 2, LB = W <= 8 ? 5 : W <= 10 ? 4 : 1;
  std::vector<uint2> t(size_t(1) << W << LB);
  for (uint32_t code = 0; code < (1u << W); ++code) {
    const uint32_t a = code & (K - 1), b = (code >> b_dir) & (K - 1), r = code >> (2 * b_dir);
    uint16_t lo[3], hi[3];
    uint32_t k[3];
    for (int j = 0; j < 3; ++j) {
      const double x = rho_c[r] * dirs64[3 * (a * K + b) + j];
      f16_bracket(x, lo[j], hi[j]);
      __half hl, hh;
      std::memcpy(&hl, &lo[j], 2);
      std::memcpy(&hh, &hi[j], 2);
      const double fl = __half2float(hl), fh = __half2float(hh);
      k[j] = fh > fl ? static_cast<uint32_t>(std::lround((x - fl) / (fh - fl) * REP)) : 0u;
    }
    for (uint32_t rep = 0; rep < REP; ++rep) {
      uint32_t br = 0;
      for (uint32_t i = 0; i < LB; ++i) br |= ((rep >> i) & 1u) << (LB - 1 - i);
      uint16_t v[3];
      for (int j = 0; j < 3; ++j) v[j] = br < k[j] ? hi[j] : lo[j];
      t[size_t(code) * REP + rep] = make_uint2(v[0] | (uint32_t(v[1]) << 16), v[2]);
    }
  }
  return t;
}

oq_status build_codec(const oq_config* cfg, const oqh::Book& xi, const oqh::Book& rho,
                      oq_codec** out) {
  if (!out) return fail(OQ_ERR_INVALID_ARGUMENT, "null output handle");
  if (cfg->dim > 256) return fail(OQ_ERR_UNSUPPORTED, "dim > 256 is not supported on device");
  int dev = 0, nsm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "no CUDA device (there is no CPU fallback)");
  e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  auto* c = new oq_codec();
  c->cfg = *cfg;
  c->device = dev;
  c->num_sms = nsm;
  {
    // K1's stream-ordered workspace (flagged-key list) comes from the
    // device's default pool: keep freed blocks cached instead of returning
    // them to the driver at every synchronisation.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = 1ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  c->xi_c = xi.centroids;
  c->rho_c = rho.centroids;
  OqCodecParams& p = c->p;
  std::memset(&p, 0, sizeof(p));
  p.dim = cfg->dim;
  p.nt = (cfg->dim + 2) / 3;
  p.b_dir = cfg->b_dir;
  p.b_nrm = cfg->b_nrm;
  p.K = 1u << cfg->b_dir;
  p.KR = 1u << cfg->b_nrm;
  p.rounding = cfg->rounding;
  p.qjl = cfg->qjl;
  p.rec_bytes = (uint32_t)rec_bytes(*cfg);
  p.dir_bytes = (2 * p.nt * p.b_dir + 7) / 8;
  p.nrm_bytes = (p.nt * p.b_nrm + 7) / 8;
  p.inv_sqrt_d = 1.0 / std::sqrt(static_cast<double>(cfg->dim));  // rotation.hpp:29
  for (uint32_t i = 0; i < cfg->dim; ++i) {
    if (oqh::rotation_sign_mask_word(cfg->rotation_seed, i)) p.sign_mask[i >> 5] |= 1u << (i & 31);
    if (oqh::rotation_sign_mask_word(cfg->qjl_seed, i)) p.qsign_mask[i >> 5] |= 1u << (i & 31);
  }
  // Direction table: oct_decode of every centroid pair (codec.hpp:100-107).
  const uint32_t K = p.K, KR = p.KR;
  std::vector<double> dirs64(size_t(K) * K * 3);
  std::vector<float> dirs32(size_t(K) * K * 4);
  for (uint32_t a = 0; a < K; ++a)
    for (uint32_t b = 0; b < K; ++b) {
      const auto n = oqh::oct_decode(xi.centroids[a], xi.centroids[b]);
      for (int j = 0; j < 3; ++j) {
        dirs64[3 * (a * K + b) + j] = n[j];
        dirs32[4 * (a * K + b) + j] = static_cast<float>(n[j]);
      }
      dirs32[4 * (a * K + b) + 3] = 0.f;
    }
  // The largest distance between two directions of one 3x3 window of
  // cells (valid cells only), for the certified argmax in compress_fast.cu;
  // rounded up to fp32 with margin.
  {
    double dmax = 0.0;
    for (int a = 0; a < (int)K; ++a)
      for (int b = 0; b < (int)K; ++b)
        for (int a2 = a; a2 <= a + 2 && a2 < (int)K; ++a2)
          for (int b2 = b - 2; b2 <= b + 2; ++b2) {
            if (b2 < 0 || b2 >= (int)K || (a2 == a && b2 <= b)) continue;
            double d2 = 0.0;
            for (int j = 0; j < 3; ++j) {
              const double d = dirs64[3 * (a * K + b) + j] - dirs64[3 * (a2 * K + b2) + j];
              d2 += d * d;
            }
            dmax = std::max(dmax, std::sqrt(d2));
          }
    p.dwin = static_cast<float>(std::min(2.0, dmax * (1.0 + 1e-6) + 1e-7));
  }
  std::vector<float> rho32(KR);
  for (uint32_t i = 0; i < KR; ++i) rho32[i] = static_cast<float>(rho.centroids[i]);
  // the attention kernel's dithered replica table (tile formats exist for W <= 13)
  std::vector<uint2> joint;
  const uint32_t W = 2 * p.b_dir + p.b_nrm;
  if (W <= 13) joint = joint_replicas(dirs64, rho.centroids, p.b_dir, p.b_nrm);
  oq_status s;
  if ((s = upload(c, xi.boundaries, &p.xi_bnd)) || (s = upload(c, rho.boundaries, &p.rho_bnd)) ||
      (s = upload(c, rho.centroids, &p.rho_c)) || (s = upload(c, dirs64, &p.dirs64)) ||
      (s = upload(c, dirs32, &p.dirs32)) || (s = upload(c, rho32, &p.rho32)) ||
      (s = upload(c, joint, &p.jointrep)) ||
      (s = upload(c, bracket_lut(xi.boundaries, -1.0, 1.0), &p.xi_lut)) ||
      (s = upload(c, bracket_lut(rho.boundaries, 0.0, 1.0), &p.rho_lut))) {
    oq_codec_destroy(c);
    return s;
  }
  *out = c;
  return OQ_OK;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

oq_status check_codec(const oq_codec* c) {
  if (!c) return fail(OQ_ERR_INVALID_ARGUMENT, "null codec");
  int dev = -1;
  cudaGetDevice(&dev);
  if (dev != c->device) return fail(OQ_ERR_INVALID_ARGUMENT, "codec belongs to another device");
  return OQ_OK;
}

}  // namespace

extern "C" {

const char* oq_last_error(void) { return g_err.c_str(); }
const char* oq_version(void) { return "octoquant-b200 0.1 (sm_100a)"; }

oq_status oq_config_default(oq_config* cfg) {
  if (!cfg) return fail(OQ_ERR_INVALID_ARGUMENT, "null config");
  *cfg = oq_config{128, 3, 1, OQ_ROUND_LOCAL3X3, 0, 0, 1};
  return OQ_OK;
}

oq_status oq_config_validate(const oq_config* cfg) { return validate(cfg); }

oq_status oq_default_bit_split(int b, int* b_dir, int* b_nrm) {
  if (b < 2) return fail(OQ_ERR_INVALID_ARGUMENT, "default bit split needs b >= 2");
  if (b_dir) *b_dir = b + 1;
  if (b_nrm) *b_nrm = b - 1;
  return OQ_OK;
}

oq_status oq_parse_rounding(const char* name, int* r) {
  static const char* names[] = {"scalar", "local2x2", "local3x3", "full"};
  for (int i = 0; i < 4; ++i)
    if (name && std::strcmp(name, names[i]) == 0) {
      if (r) *r = i;
      return OQ_OK;
    }
  return fail(OQ_ERR_INVALID_ARGUMENT,
              std::string("unknown rounding mode: ") + (name ? name : "(null)"));
}

const char* oq_rounding_name(int r) {
  switch (r) {
    case 0: return "scalar";
    case 1: return "local2x2";
    case 2: return "local3x3";
    case 3: return "full";
  }
  return "?";
}

double oq_effective_bits_per_coord(const oq_config* cfg) {
  const double nt = (cfg->dim + 2) / 3;
  double bits = 2.0 * nt * cfg->b_dir + nt * cfg->b_nrm + 32.0;
  if (cfg->qjl) bits += cfg->dim + 16.0;
  return bits / cfg->dim;
}

size_t oq_record_bytes(const oq_config* cfg) { return cfg ? rec_bytes(*cfg) : 0; }

oq_status oq_xi_book(int bits, double* c, double* b) {
  try {
    const oqh::Book& bk = oqh::xi_book(bits);
    if (c) std::memcpy(c, bk.centroids.data(), bk.centroids.size() * 8);
    if (b) std::memcpy(b, bk.boundaries.data(), bk.boundaries.size() * 8);
    return OQ_OK;
  } catch (const std::exception& ex) {
    return fail(OQ_ERR_INVALID_ARGUMENT, ex.what());
  }
}

oq_status oq_rho_book(uint32_t dim, int bits, double* c, double* b) {
  try {
    const oqh::Book& bk = oqh::rho_book(dim, bits);
    if (c) std::memcpy(c, bk.centroids.data(), bk.centroids.size() * 8);
    if (b) std::memcpy(b, bk.boundaries.data(), bk.boundaries.size() * 8);
    return OQ_OK;
  } catch (const std::exception& ex) {
    return fail(OQ_ERR_INVALID_ARGUMENT, ex.what());
  }
}

oq_status oq_codec_create(const oq_config* cfg, oq_codec** out) {
  oq_status s = validate(cfg);
  if (s) return s;
  try {
    return build_codec(cfg, oqh::xi_book(cfg->b_dir), oqh::rho_book(cfg->dim, cfg->b_nrm), out);
  } catch (const std::exception& ex) {
    return fail(OQ_ERR_INVALID_ARGUMENT, ex.what());
  }
}

oq_status oq_codec_create_custom(const oq_config* cfg, const double* xc, int xbits,
                                 const double* rc, int rbits, oq_codec** out) {
  oq_status s = validate(cfg);
  if (s) return s;
  if (!xc || !rc || xbits != cfg->b_dir || rbits != cfg->b_nrm)
    return fail(OQ_ERR_INVALID_ARGUMENT, "custom books must match the configured bit widths");
  for (int i = 1; i < (1 << xbits); ++i)
    if (!(xc[i] >= xc[i - 1])) return fail(OQ_ERR_INVALID_ARGUMENT, "centroids not ascending");
  for (int i = 1; i < (1 << rbits); ++i)
    if (!(rc[i] >= rc[i - 1])) return fail(OQ_ERR_INVALID_ARGUMENT, "centroids not ascending");
  return build_codec(cfg, oqh::custom_book(xc, xbits), oqh::custom_book(rc, rbits), out);
}

void oq_codec_destroy(oq_codec* c) {
  if (!c) return;
  for (void* p : c->allocs) cudaFree(p);
  delete c;
}

oq_status oq_codec_config(const oq_codec* c, oq_config* cfg) {
  if (!c || !cfg) return fail(OQ_ERR_INVALID_ARGUMENT, "null argument");
  *cfg = c->cfg;
  return OQ_OK;
}

oq_status oq_compress(const oq_codec* c, const void* x, int dtype, size_t n, void* records,
                      void* stream) {
  return oq_compress_ex(c, x, dtype, n, records, nullptr, stream);
}

oq_status oq_compress_ex(const oq_codec* c, const void* x, int dtype, size_t n, void* records,
                         uint32_t* flagged, void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  if (n && (!x || !records)) return fail(OQ_ERR_INVALID_ARGUMENT, "null buffer");
  if (dtype < OQ_DTYPE_F32 || dtype > OQ_DTYPE_BF16)
    return fail(OQ_ERR_INVALID_ARGUMENT, "unknown dtype");
  TimedScope ts("compress", as_stream(stream));
  cudaError_t e = oqd::launch_compress(c->p, x, dtype, n, static_cast<uint8_t*>(records),
                                       as_stream(stream), c->num_sms, flagged);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "compress kernel");
}

oq_status oq_decode(const oq_codec* c, const void* records, size_t n, float* out, void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  if (n && (!records || !out)) return fail(OQ_ERR_INVALID_ARGUMENT, "null buffer");
  TimedScope ts("decode", as_stream(stream));
  cudaError_t e = oqd::launch_decode(c->p, static_cast<const uint8_t*>(records), n, out,
                                     as_stream(stream), c->num_sms);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "decode kernel");
}

oq_status oq_dir_table(const double* xi_centroids, int k, double* out) {
  if (!xi_centroids || !out || k < 1) return fail(OQ_ERR_INVALID_ARGUMENT, "bad direction table arguments");
  for (int a = 0; a < k; ++a)
    for (int b = 0; b < k; ++b) {
      const auto n = oqh::oct_decode(xi_centroids[a], xi_centroids[b]);
      for (int j = 0; j < 3; ++j) out[3 * (size_t(a) * k + b) + j] = n[j];
    }
  return OQ_OK;
}

oq_status oq_prepare_f64(const oq_codec* c, const double* q, size_t nq, double* rot,
                         double* sketch, void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  if (nq && (!q || !rot)) return fail(OQ_ERR_INVALID_ARGUMENT, "null buffer");
  if (nq && c->p.qjl && !sketch)
    return fail(OQ_ERR_INVALID_ARGUMENT, "QJL codec: the sketch output is required");
  cudaError_t e = oqd::launch_prepare_f64(c->p, q, nq, rot, c->p.qjl ? sketch : nullptr,
                                          as_stream(stream));
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "prepare kernel");
}

oq_status oq_reconstruct_rotated(const oq_codec* c, const void* records, size_t n, double* out,
                                 void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  if (n && (!records || !out)) return fail(OQ_ERR_INVALID_ARGUMENT, "null buffer");
  cudaError_t e = oqd::launch_reconstruct_f64(c->p, static_cast<const uint8_t*>(records), n, out,
                                              0, as_stream(stream));
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "reconstruct kernel");
}

oq_status oq_decode_f64(const oq_codec* c, const void* records, size_t n, double* out,
                        void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  if (n && (!records || !out)) return fail(OQ_ERR_INVALID_ARGUMENT, "null buffer");
  cudaError_t e = oqd::launch_reconstruct_f64(c->p, static_cast<const uint8_t*>(records), n, out,
                                              1, as_stream(stream));
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "exact decode kernel");
}

oq_status oq_score_prepared(const oq_codec* c, const double* rot, const double* sketch, size_t nq,
                            const void* records, size_t n, double* out, void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  if (nq && n && (!rot || !records || !out)) return fail(OQ_ERR_INVALID_ARGUMENT, "null buffer");
  if (nq && n && c->p.qjl && !sketch)
    return fail(OQ_ERR_INVALID_ARGUMENT, "QJL codec: the prepared sketch is required");
  cudaError_t e = oqd::launch_score_prepared(c->p, rot, c->p.qjl ? sketch : nullptr, nq,
                                             static_cast<const uint8_t*>(records), n, out,
                                             as_stream(stream));
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "score kernel");
}

size_t oq_attention_f64_workspace_bytes(const oq_codec* c, size_t nq, size_t n) {
  if (!c) return 0;
  return (2 * nq * c->p.dim + nq * n) * sizeof(double);
}

oq_status oq_attention_decode_f64(const oq_codec* c, const double* q, size_t nq,
                                  const void* records, size_t n, const double* values, int vdim,
                                  int n_splits, double* out, void* workspace, size_t ws_bytes,
                                  void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  // attention.hpp:54-56
  if (n == 0) return fail(OQ_ERR_INVALID_ARGUMENT, "empty cache");
  if (n_splits < 1) return fail(OQ_ERR_INVALID_ARGUMENT, "n_splits must be >= 1");
  if (vdim < 1) return fail(OQ_ERR_INVALID_ARGUMENT, "values/cache length mismatch");
  if (!q || !records || !values || !out || !workspace)
    return fail(OQ_ERR_INVALID_ARGUMENT, "null buffer");
  if (ws_bytes < oq_attention_f64_workspace_bytes(c, nq, n))
    return fail(OQ_ERR_INVALID_ARGUMENT, "workspace too small");
  double* rot = static_cast<double*>(workspace);
  double* sketch = rot + nq * c->p.dim;
  double* scores = sketch + nq * c->p.dim;
  cudaStream_t st = as_stream(stream);
  cudaError_t e = oqd::launch_prepare_f64(c->p, q, nq, rot, sketch, st);
  if (e == cudaSuccess)
    e = oqd::launch_score_prepared(c->p, rot, sketch, nq, static_cast<const uint8_t*>(records), n,
                                   scores, st);
  if (e == cudaSuccess)
    e = oqd::launch_softmax_read(scores, nq, n, values, vdim, n_splits, c->p.inv_sqrt_d, out, st);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "fp64 attention kernels");
}

oq_status oq_wire_header(const oq_config* cfg, uint64_t count, uint8_t h[20]) {
  oq_status s = validate(cfg);
  if (s) return s;
  std::memcpy(h, "OCTO", 4);
  h[4] = 1;
  h[5] = cfg->qjl ? 1 : 0;
  h[6] = cfg->b_dir;
  h[7] = cfg->b_nrm;
  std::memcpy(h + 8, &cfg->dim, 4);
  std::memcpy(h + 12, &count, 8);
  return OQ_OK;
}

oq_status oq_wire_parse_header(const uint8_t* p, size_t n, oq_config* cfg, uint64_t* count) {
  // codec.hpp:410-430 (ByteReader throws FormatError("truncated stream")).
  if (!p || n < 4) return fail(OQ_ERR_FORMAT, "truncated stream");
  if (std::memcmp(p, "OCTO", 4) != 0) return fail(OQ_ERR_FORMAT, "bad blob magic");
  if (n < 5) return fail(OQ_ERR_FORMAT, "truncated stream");
  if (p[4] != 1) return fail(OQ_ERR_FORMAT, "unsupported blob version");
  if (n < 6) return fail(OQ_ERR_FORMAT, "truncated stream");
  if (p[5] & ~1u) return fail(OQ_ERR_FORMAT, "unknown flag bits");
  if (n < 8) return fail(OQ_ERR_FORMAT, "truncated stream");
  oq_config c;
  oq_config_default(&c);
  c.qjl = p[5] & 1u;
  c.b_dir = p[6];
  c.b_nrm = p[7];
  if (c.b_dir < 1 || c.b_dir > 8 || c.b_nrm < 1 || c.b_nrm > 8)
    return fail(OQ_ERR_FORMAT, "blob bits out of range");
  if (n < 12) return fail(OQ_ERR_FORMAT, "truncated stream");
  std::memcpy(&c.dim, p + 8, 4);
  if (!is_pow2(c.dim) || c.dim < 4) return fail(OQ_ERR_FORMAT, "blob dim invalid");
  if (n < 20) return fail(OQ_ERR_FORMAT, "truncated stream");
  uint64_t cnt;
  std::memcpy(&cnt, p + 12, 8);
  const size_t rb = rec_bytes(c);
  if (n - 20 != cnt * rb) return fail(OQ_ERR_FORMAT, "blob payload size mismatch");
  if (cfg) *cfg = c;
  if (count) *count = cnt;
  return OQ_OK;
}

oq_status oq_validate_records(const oq_codec* c, const void* records, size_t n, void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  if (n == 0) return OQ_OK;
  int* d_bad = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_bad), sizeof(int), as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  cudaMemsetAsync(d_bad, 0, sizeof(int), as_stream(stream));
  e = oqd::launch_validate_records(c->p, static_cast<const uint8_t*>(records), n, d_bad,
                                   as_stream(stream), c->num_sms);
  int bad = 0;
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, as_stream(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(as_stream(stream));
  cudaFreeAsync(d_bad, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "validate kernel");
  if (bad & 1) return fail(OQ_ERR_FORMAT, "nonzero padding in direction stream");
  if (bad & 2) return fail(OQ_ERR_FORMAT, "nonzero padding in norm stream");
  if (bad & 4) return fail(OQ_ERR_FORMAT, "nonzero padding in sign stream");
  return OQ_OK;
}

// ---- attention -------------------------------------------------------------

size_t oq_cache_tile_bytes(const oq_codec* c, int role) {
  return c ? oqd::attention_tile_bytes(c->p, role) : 0;
}

size_t oq_cache_bytes(const oq_codec* c, int role, uint64_t tokens) {
  return c ? ((tokens + 31) / 32) * oqd::attention_tile_bytes(c->p, role) : 0;
}

oq_status oq_cache_pack(const oq_codec* c, int role, const void* records, uint64_t n_streams,
                        uint64_t n_tokens, uint64_t rec_stride, void* tiles, uint64_t cap_tokens,
                        void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  if (role != OQ_ROLE_K && role != OQ_ROLE_V) return fail(OQ_ERR_INVALID_ARGUMENT, "bad role");
  if (n_tokens > cap_tokens || n_tokens > rec_stride)
    return fail(OQ_ERR_INVALID_ARGUMENT, "cache capacity smaller than the token count");
  if (oqd::attention_tile_bytes(c->p, role) == 0)
    return fail(OQ_ERR_UNSUPPORTED, "attention tile format needs dim 128 and 2*b_dir+b_nrm <= 13");
  if (role == OQ_ROLE_V && c->cfg.qjl)
    return fail(OQ_ERR_INVALID_ARGUMENT, "the V codec carries no QJL sidecar");
  cudaError_t e = oqd::launch_pack_tiles(c->p, role, static_cast<const uint8_t*>(records),
                                         n_streams, n_tokens, rec_stride,
                                         static_cast<uint8_t*>(tiles), (cap_tokens + 31) / 32,
                                         as_stream(stream));
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "pack tiles kernel");
}

oq_status oq_cache_append(const oq_codec* c, int role, const void* x, int dtype,
                          uint64_t n_streams, const int64_t* pos_dev, int64_t pos, void* records,
                          void* tiles, uint64_t cap_tokens, void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  if (role != OQ_ROLE_K && role != OQ_ROLE_V) return fail(OQ_ERR_INVALID_ARGUMENT, "bad role");
  if (n_streams && (!x || !records || !tiles)) return fail(OQ_ERR_INVALID_ARGUMENT, "null buffer");
  if (!pos_dev && (pos < 0 || (uint64_t)pos >= cap_tokens))
    return fail(OQ_ERR_INVALID_ARGUMENT, "append position outside the cache");
  if (oqd::attention_tile_bytes(c->p, role) == 0)
    return fail(OQ_ERR_UNSUPPORTED, "attention tile format needs dim 128 and 2*b_dir+b_nrm <= 13");
  if (role == OQ_ROLE_V && c->cfg.qjl)
    return fail(OQ_ERR_INVALID_ARGUMENT, "the V codec carries no QJL sidecar");
  s = oq_compress(c, x, dtype, n_streams, records, stream);
  if (s) return s;
  cudaError_t e = oqd::launch_append_token(c->p, role, static_cast<const uint8_t*>(records),
                                           n_streams, pos_dev, pos, static_cast<uint8_t*>(tiles),
                                           (cap_tokens + 31) / 32, as_stream(stream));
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "append kernel");
}

oq_status oq_cache_append_kv(const oq_codec* ck, const oq_codec* cv, const void* k, const void* v,
                             int dtype, uint64_t n_streams, const int64_t* pos_dev, int64_t pos,
                             void* k_records, void* v_records, void* ktiles, void* vtiles,
                             uint64_t cap_tokens, void* stream) {
  oq_status s = check_codec(ck);
  if (!s) s = check_codec(cv);
  if (s) return s;
  if (n_streams && (!k || !v || !ktiles || !vtiles))
    return fail(OQ_ERR_INVALID_ARGUMENT, "null buffer");
  if (!pos_dev && (pos < 0 || (uint64_t)pos >= cap_tokens))
    return fail(OQ_ERR_INVALID_ARGUMENT, "append position outside the cache");
  if (oqd::attention_tile_bytes(ck->p, OQ_ROLE_K) == 0 ||
      oqd::attention_tile_bytes(cv->p, OQ_ROLE_V) == 0)
    return fail(OQ_ERR_UNSUPPORTED, "attention tile format needs dim 128 and 2*b_dir+b_nrm <= 13");
  if (cv->cfg.qjl) return fail(OQ_ERR_INVALID_ARGUMENT, "the V codec carries no QJL sidecar");
  if (dtype != OQ_F32 && dtype != OQ_F64 && dtype != OQ_F16 && dtype != OQ_BF16)
    return fail(OQ_ERR_INVALID_ARGUMENT, "bad dtype");
  if (n_streams == 0) return OQ_OK;
  cudaStream_t st = as_stream(stream);
  // one launch: both roles encoded (exactly, QJL sidecar included) and
  // written in place (the tile format implies d = 128)
  cudaError_t e = oqd::launch_append_fused(
      ck->p, cv->p, k, v, dtype, n_streams, pos_dev, pos, static_cast<uint8_t*>(k_records),
      static_cast<uint8_t*>(v_records), static_cast<uint8_t*>(ktiles),
      static_cast<uint8_t*>(vtiles), (cap_tokens + 31) / 32, st);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "fused append kernel");
}

static int parts_per_row(const oq_codec* ck, const oq_attn_shape* sh, uint64_t t0, uint64_t t1,
                         int n_splits) {
  return oqd::attention_num_parts(sh->B, sh->Hq, sh->Hkv, sh->T, t0, t1, n_splits, ck->num_sms);
}

// Workspace layout: [per-stream arrival counters, 64 KiB: zero on first use,
// the fused kernel leaves them zero][partials][query fragments].
static constexpr size_t kCounterBytes = 64 * 1024;

size_t oq_attention_workspace_bytes(const oq_codec* ck, const oq_codec* cv,
                                    const oq_attn_shape* sh, int n_splits) {
  if (!ck || !cv || !sh || n_splits < 0 || sh->Hkv < 1) return 0;
  const size_t rows = (size_t)sh->B * sh->Hq;
  // stream-K needs the most slots for the full range; shorter ranges need fewer
  const size_t np = (size_t)parts_per_row(ck, sh, 0, sh->T, n_splits) + 1;
  const size_t part = rows * np * (4 + ck->cfg.dim) * sizeof(float);
  const size_t hc = sh->Hkv > 0 ? (size_t)((sh->Hq / sh->Hkv + 7) / 8) : 1;
  const size_t qf = (size_t)sh->B * sh->Hkv * hc * oqd::attention_qfrag_bytes(ck->p);
  return kCounterBytes + ((part + 255) & ~size_t(255)) + qf + 256;
}

static oq_status attn_check(const oq_codec* ck, const oq_codec* cv, const oq_attn_shape* sh,
                            const float* q, const void* kc, const void* vc, int n_splits,
                            size_t ws_bytes) {
  oq_status s;
  if ((s = check_codec(ck)) || (s = check_codec(cv))) return s;
  if (!sh || !q || !kc || !vc) return fail(OQ_ERR_INVALID_ARGUMENT, "null argument");
  if (sh->B < 1 || sh->Hq < 1 || sh->Hkv < 1 || sh->Hq % sh->Hkv)
    return fail(OQ_ERR_INVALID_ARGUMENT, "bad head configuration");
  if (sh->T == 0) return fail(OQ_ERR_INVALID_ARGUMENT, "empty cache");  // attention.hpp:55
  if (sh->T > sh->cap_tokens) return fail(OQ_ERR_INVALID_ARGUMENT, "values/cache length mismatch");
  if (n_splits < 0) return fail(OQ_ERR_INVALID_ARGUMENT, "n_splits must be >= 0 (0 = auto)");
  if (ck->cfg.dim != cv->cfg.dim) return fail(OQ_ERR_INVALID_ARGUMENT, "K/V dim mismatch");
  if (cv->cfg.qjl) return fail(OQ_ERR_INVALID_ARGUMENT, "the V codec carries no QJL sidecar");
  if (!oqd::attention_fast_path_ok(ck->p, cv->p))
    return fail(OQ_ERR_UNSUPPORTED, "attention kernels need dim 128 and 2*b_dir+b_nrm <= 13");
  if (ws_bytes < oq_attention_workspace_bytes(ck, cv, sh, n_splits))
    return fail(OQ_ERR_INVALID_ARGUMENT, "workspace too small");
  return OQ_OK;
}

struct P2PArgs {
  int rank, nranks;
  uint32_t epoch;
  uint8_t* xbuf[8];
  int max_ctas;
};

static oq_status run_partials(const oq_codec* ck, const oq_codec* cv, const oq_attn_shape* sh,
                              const float* q, const void* kc, const void* vc, uint64_t t0,
                              uint64_t t1, int n_splits, void* ws, cudaStream_t st,
                              float** parts_out, int* n_parts_out, float* fused_out = nullptr,
                              bool fused_partial = false, const P2PArgs* p2p = nullptr) {
  const size_t rows = (size_t)sh->B * sh->Hq;
  const int np_max = parts_per_row(ck, sh, 0, sh->T, n_splits) + 1;
  const int np = parts_per_row(ck, sh, t0, t1, n_splits);
  const size_t part = rows * (size_t)np_max * (4 + ck->cfg.dim) * sizeof(float);
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  oqd::AttnArgs a{};
  a.B = sh->B;
  a.Hq = sh->Hq;
  a.Hkv = sh->Hkv;
  a.T = sh->T;
  a.t_begin = t0;
  a.t_end = t1;
  a.seq_lens = sh->seq_lens;
  a.q = q;
  a.kcache = static_cast<const uint8_t*>(kc);
  a.vcache = static_cast<const uint8_t*>(vc);
  a.k_tiles_cap = a.v_tiles_cap = (sh->cap_tokens + 31) / 32;
  a.partials = reinterpret_cast<float*>(w8 + kCounterBytes);
  a.n_parts = np;
  *n_parts_out = np;
  a.qfrag = w8 + kCounterBytes + ((part + 255) & ~size_t(255));
  if (t1 <= t0) {  // no tokens in range: every row's partial is empty (l = 0)
    const size_t w = 4 + ck->cfg.dim;
    float* dst = fused_out && fused_partial ? fused_out : a.partials;
    const size_t nrow = fused_out && fused_partial ? rows : rows * (size_t)np;
    const cudaError_t z = cudaMemsetAsync(dst, 0, nrow * w * sizeof(float), st);
    if (z != cudaSuccess) return cuda_fail(z, "cudaMemsetAsync");
    *parts_out = fused_out && fused_partial ? nullptr : a.partials;
    return OQ_OK;
  }
  // one launch when the per-stream counters fit: q prep and the final merge
  // run inside the attention kernel
  const size_t n_sh = (size_t)sh->B * sh->Hkv * ((sh->Hq / sh->Hkv + 7) / 8);
  static const bool unfused = getenv("OQ_ATTN_UNFUSED") != nullptr;  // comparison runs
  const bool fuse = fused_out && n_sh * 4 <= kCounterBytes && !unfused;
  cudaError_t e = cudaSuccess;
  if (p2p && !fuse) return fail(OQ_ERR_UNSUPPORTED, "P2P sharding needs the fused attention kernel");
  if (fuse) {
    a.out = fused_out;
    a.out_partial = fused_partial ? 1 : 0;
    a.counters = reinterpret_cast<uint32_t*>(w8);
    for (int i = 0; i < 4; ++i) a.vmask[i] = cv->p.sign_mask[i];
    if (p2p) {
      a.p2p_nranks = p2p->nranks;
      a.p2p_rank = p2p->rank;
      a.p2p_epoch = p2p->epoch;
      for (int i = 0; i < p2p->nranks; ++i) a.p2p_xbuf[i] = p2p->xbuf[i];
      a.max_ctas = p2p->max_ctas;
    }
  } else {
    e = oqd::launch_qprep(ck->p, a, st);
    if (e != cudaSuccess) return cuda_fail(e, "qprep kernel");
  }
  {
    TimedScope ts("attention", st);
    e = oqd::launch_attention_partials(ck->p, cv->p, a, n_splits, st, ck->num_sms);
  }
  if (e != cudaSuccess) return cuda_fail(e, "attention kernel");
  *parts_out = fuse ? nullptr : a.partials;
  return OQ_OK;
}

oq_status oq_attention_decode(const oq_codec* ck, const oq_codec* cv, const oq_attn_shape* sh,
                              const float* q, const void* kc, const void* vc, float* out,
                              int n_splits, void* ws, size_t ws_bytes, void* stream) {
  oq_status s = attn_check(ck, cv, sh, q, kc, vc, n_splits, ws_bytes);
  if (s) return s;
  if (!out || !ws) return fail(OQ_ERR_INVALID_ARGUMENT, "null argument");
  float* parts = nullptr;
  int np = 0;
  s = run_partials(ck, cv, sh, q, kc, vc, 0, sh->T, n_splits, ws, as_stream(stream), &parts, &np,
                   out);
  if (s) return s;
  if (!parts) return OQ_OK;  // fused: the attention kernel wrote out
  const int rows = sh->B * sh->Hq;
  const size_t w = 4 + ck->cfg.dim;
  cudaError_t e = oqd::launch_attention_combine(cv->p, parts, rows, np, np * w, w, 1,
                                                out, as_stream(stream));
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "combine kernel");
}

// ---- NCCL, loaded on first use (no link-time dependency) -------------------
namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  // signatures from nccl.h (ncclResult_t is an int enum; ncclFloat32 = 7)
  int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*user_rank)(void*, int*) = nullptr;
  int (*count)(void*, int*) = nullptr;
  int (*get_unique_id)(void*) = nullptr;
  int (*init_rank)(void**, int, const void*, int) = nullptr;  // id passed by value (128 B)
  int (*destroy)(void*) = nullptr;
  const char* (*err)(int) = nullptr;
};
struct NcclUid {
  char b[128];
};
NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = "libnccl.so.2 not found";
      return a;
    }
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.user_rank = reinterpret_cast<decltype(a.user_rank)>(dlsym(h, "ncclCommUserRank"));
    a.count = reinterpret_cast<decltype(a.count)>(dlsym(h, "ncclCommCount"));
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.init_rank = reinterpret_cast<decltype(a.init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "ncclCommDestroy"));
    a.err = reinterpret_cast<decltype(a.err)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.all_gather && a.user_rank && a.count && a.get_unique_id && a.init_rank &&
           a.destroy && a.err;
    if (!a.ok) a.why = "libnccl lacks the expected symbols";
    return a;
  }();
  return api;
}
oq_status nccl_fail(int r, const char* what) {
  return fail(OQ_ERR_NCCL, std::string(what) + ": " + (nccl().err ? nccl().err(r) : "error"));
}
}  // namespace

oq_status oq_attention_partials(const oq_codec* ck, const oq_codec* cv, const oq_attn_shape* sh,
                                const float* q, const void* kc, const void* vc, uint64_t t0,
                                uint64_t t1, float* partial, int n_splits, void* ws,
                                size_t ws_bytes, void* stream) {
  oq_status s = attn_check(ck, cv, sh, q, kc, vc, n_splits, ws_bytes);
  if (s) return s;
  if (!partial || !ws) return fail(OQ_ERR_INVALID_ARGUMENT, "null argument");
  if (t0 > t1 || t1 > sh->T) return fail(OQ_ERR_INVALID_ARGUMENT, "bad token range");
  float* parts = nullptr;
  int np = 0;
  // one launch when possible: the attention kernel merges its splits into
  // the (m, l, acc) partial itself
  s = run_partials(ck, cv, sh, q, kc, vc, t0, t1, n_splits, ws, as_stream(stream), &parts, &np,
                   partial, true);
  if (s || !parts) return s;
  const int rows = sh->B * sh->Hq;
  const size_t w = 4 + ck->cfg.dim;
  cudaError_t e = oqd::launch_attention_combine(cv->p, parts, rows, np, np * w, w, 0,
                                                partial, as_stream(stream));
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "combine kernel");
}

oq_status oq_attention_combine(const oq_codec* cv, const float* partials, int rows, int n_parts,
                               size_t row_stride, size_t part_stride, int finalize, float* out,
                               void* stream) {
  oq_status s = check_codec(cv);
  if (s) return s;
  if (!partials || !out || rows < 1 || n_parts < 1)
    return fail(OQ_ERR_INVALID_ARGUMENT, "bad combine arguments");
  cudaError_t e = oqd::launch_attention_combine(cv->p, partials, rows, n_parts, row_stride,
                                                part_stride, finalize, out, as_stream(stream));
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "combine kernel");
}

size_t oq_attention_sharded_workspace_bytes(const oq_codec* ck, const oq_codec* cv,
                                            const oq_attn_shape* sh, int n_splits, int nranks) {
  const size_t base = oq_attention_workspace_bytes(ck, cv, sh, n_splits);
  if (!base || nranks < 1) return 0;
  const size_t gather = (size_t)nranks * sh->B * sh->Hq * (4 + ck->cfg.dim) * sizeof(float);
  return ((base + 255) & ~size_t(255)) + gather;
}

oq_status oq_attention_decode_sharded(const oq_codec* ck, const oq_codec* cv,
                                      const oq_attn_shape* sh, const float* q, const void* kc,
                                      const void* vc, uint64_t t0, uint64_t t1, void* comm,
                                      int nranks, float* out, int n_splits, void* ws,
                                      size_t ws_bytes, void* stream) {
  const size_t base = oq_attention_workspace_bytes(ck, cv, sh, n_splits);
  oq_status s = attn_check(ck, cv, sh, q, kc, vc, n_splits, base);
  if (s) return s;
  if (!out || !ws || !comm || nranks < 1) return fail(OQ_ERR_INVALID_ARGUMENT, "null argument");
  if (t0 > t1 || t1 > sh->T) return fail(OQ_ERR_INVALID_ARGUMENT, "bad token range");
  if (ws_bytes < oq_attention_sharded_workspace_bytes(ck, cv, sh, n_splits, nranks))
    return fail(OQ_ERR_INVALID_ARGUMENT, "workspace too small");
  NcclApi& api = nccl();
  if (!api.ok) return fail(OQ_ERR_NCCL, api.why);
  int rank = -1, count = 0, r;
  if ((r = api.user_rank(comm, &rank)) != 0) return nccl_fail(r, "ncclCommUserRank");
  if ((r = api.count(comm, &count)) != 0) return nccl_fail(r, "ncclCommCount");
  if (count != nranks) return fail(OQ_ERR_INVALID_ARGUMENT, "nranks differs from the communicator");
  const cudaStream_t st = as_stream(stream);
  const int rows = sh->B * sh->Hq;
  const size_t w = 4 + ck->cfg.dim, per = (size_t)rows * w;
  float* gather = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + ((base + 255) & ~size_t(255)));
  float* parts = nullptr;
  int np = 0;
  // this rank's merged partial lands straight in its slot of the gather
  // buffer: from the attention kernel itself when it runs fused, else by a
  // combine pass over its splits
  s = run_partials(ck, cv, sh, q, kc, vc, t0, t1, n_splits, ws, st, &parts, &np,
                   gather + (size_t)rank * per, true);
  if (s) return s;
  cudaError_t e = cudaSuccess;
  if (parts) {
    e = oqd::launch_attention_combine(cv->p, parts, rows, np, np * w, w, 0,
                                      gather + (size_t)rank * per, st);
    if (e != cudaSuccess) return cuda_fail(e, "combine kernel");
  }
  // the only collective: in-place all-gather of the per-rank partials
  if ((r = api.all_gather(gather + (size_t)rank * per, gather, per, /*ncclFloat32*/ 7, comm, st)) != 0)
    return nccl_fail(r, "ncclAllGather");
  e = oqd::launch_attention_combine(cv->p, gather, rows, nranks, w, per, 1, out, st);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "combine kernel");
}

// ---- fused P2P sequence sharding (peer memory, no collective library) -----
size_t oq_attention_p2p_exchange_bytes(const oq_codec* ck, const oq_attn_shape* sh, int nranks) {
  if (!ck || !sh || nranks < 1) return 0;
  const size_t rows = (size_t)sh->B * sh->Hq;
  const size_t n_sh = (size_t)sh->B * sh->Hkv * ((sh->Hq / (sh->Hkv ? sh->Hkv : 1) + 7) / 8);
  return 2 * (size_t)nranks * rows * (4 + ck->cfg.dim) * sizeof(float) + (size_t)nranks * n_sh * 4;
}

oq_status oq_attention_decode_p2p(const oq_codec* ck, const oq_codec* cv, const oq_attn_shape* sh,
                                  const float* q, const void* kc, const void* vc, uint64_t t0,
                                  uint64_t t1, int rank, int nranks, void* const* xbufs,
                                  uint32_t epoch, int max_ctas, float* out, void* ws,
                                  size_t ws_bytes, void* stream) {
  const size_t base = oq_attention_workspace_bytes(ck, cv, sh, 0);
  oq_status s = attn_check(ck, cv, sh, q, kc, vc, 0, base);
  if (s) return s;
  if (!out || !ws || !xbufs) return fail(OQ_ERR_INVALID_ARGUMENT, "null argument");
  if (nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks)
    return fail(OQ_ERR_INVALID_ARGUMENT, "P2P sharding supports 1..8 ranks");
  if (epoch == 0) return fail(OQ_ERR_INVALID_ARGUMENT, "epoch must be nonzero (flags start at 0)");
  if (t0 > t1 || t1 > sh->T) return fail(OQ_ERR_INVALID_ARGUMENT, "bad token range");
  if (ws_bytes < base) return fail(OQ_ERR_INVALID_ARGUMENT, "workspace too small");
  if (ck->cfg.dim != 128) return fail(OQ_ERR_UNSUPPORTED, "P2P sharding needs dim 128");
  P2PArgs p{rank, nranks, epoch, {}, max_ctas};
  for (int r = 0; r < nranks; ++r) {
    if (!xbufs[r]) return fail(OQ_ERR_INVALID_ARGUMENT, "null exchange buffer");
    p.xbuf[r] = static_cast<uint8_t*>(xbufs[r]);
  }
  float* parts = nullptr;
  int np = 0;
  // an empty token range still has to publish (empty) rows and wait: not
  // representable by the memset shortcut, so it is rejected
  if (t1 <= t0) return fail(OQ_ERR_UNSUPPORTED, "P2P sharding needs a nonempty token range per rank");
  return run_partials(ck, cv, sh, q, kc, vc, t0, t1, 0, ws, as_stream(stream), &parts, &np, out,
                      false, &p);
}

oq_status oq_ipc_handle(void* dev_ptr, uint8_t handle[64]) {
  if (!dev_ptr || !handle) return fail(OQ_ERR_INVALID_ARGUMENT, "null argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  std::memcpy(handle, &h, 64);
  return OQ_OK;
}

oq_status oq_ipc_open(const uint8_t handle[64], void** dev_ptr) {
  if (!dev_ptr || !handle) return fail(OQ_ERR_INVALID_ARGUMENT, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

oq_status oq_ipc_close(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

oq_status oq_nccl_get_unique_id(uint8_t id[128]) {
  NcclApi& api = nccl();
  if (!api.ok) return fail(OQ_ERR_NCCL, api.why);
  if (!id) return fail(OQ_ERR_INVALID_ARGUMENT, "null id");
  const int r = api.get_unique_id(id);
  return r ? nccl_fail(r, "ncclGetUniqueId") : OQ_OK;
}

oq_status oq_nccl_comm_init_rank(void** comm, int nranks, const uint8_t id[128], int rank) {
  NcclApi& api = nccl();
  if (!api.ok) return fail(OQ_ERR_NCCL, api.why);
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(OQ_ERR_INVALID_ARGUMENT, "bad communicator arguments");
  // ncclCommInitRank takes the 128-byte unique id by value
  using InitFn = int (*)(void**, int, NcclUid, int);
  NcclUid u;
  std::memcpy(u.b, id, 128);
  const int r = reinterpret_cast<InitFn>(api.init_rank)(comm, nranks, u, rank);
  return r ? nccl_fail(r, "ncclCommInitRank") : OQ_OK;
}

oq_status oq_nccl_comm_destroy(void* comm) {
  NcclApi& api = nccl();
  if (!api.ok) return fail(OQ_ERR_NCCL, api.why);
  const int r = comm ? api.destroy(comm) : 0;
  return r ? nccl_fail(r, "ncclCommDestroy") : OQ_OK;
}

oq_status oq_nccl_comm_info(void* comm, int* rank, int* nranks) {
  NcclApi& api = nccl();
  if (!api.ok) return fail(OQ_ERR_NCCL, api.why);
  if (!comm || !rank || !nranks) return fail(OQ_ERR_INVALID_ARGUMENT, "null communicator");
  int r;
  if ((r = api.user_rank(comm, rank)) != 0) return nccl_fail(r, "ncclCommUserRank");
  if ((r = api.count(comm, nranks)) != 0) return nccl_fail(r, "ncclCommCount");
  return OQ_OK;
}

oq_status oq_scores(const oq_codec* c, const float* q, int nq, const void* records, size_t n,
                    float* out, void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  if (nq < 0 || (n && nq && (!q || !records || !out)))
    return fail(OQ_ERR_INVALID_ARGUMENT, "bad scores arguments");
  cudaError_t e = oqd::launch_scores(c->p, q, nq, static_cast<const uint8_t*>(records), n, out,
                                     as_stream(stream), c->num_sms);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "scores kernel");
}

size_t oq_attention_dense_workspace_bytes(int nq, int n_splits, int vdim) {
  if (nq < 1 || n_splits < 1 || vdim < 1) return 0;
  return oqd::dense_attention_workspace(nq, n_splits, vdim);
}

oq_status oq_attention_decode_dense(const oq_codec* c, const float* q, int nq,
                                    const void* records, size_t n, const float* values,
                                    int vdim, int n_splits, float* out, void* ws,
                                    size_t ws_bytes, void* stream) {
  oq_status s = check_codec(c);
  if (s) return s;
  // attention.hpp:54-56
  if (n == 0) return fail(OQ_ERR_INVALID_ARGUMENT, "empty cache");
  if (n_splits < 1) return fail(OQ_ERR_INVALID_ARGUMENT, "n_splits must be >= 1");
  if (nq < 1 || !q || !records || !values || !out || !ws)
    return fail(OQ_ERR_INVALID_ARGUMENT, "null argument");
  if (vdim < 1 || vdim > 256) return fail(OQ_ERR_UNSUPPORTED, "value width must be in [1, 256]");
  if (ws_bytes < oq_attention_dense_workspace_bytes(nq, n_splits, vdim))
    return fail(OQ_ERR_INVALID_ARGUMENT, "workspace too small");
  cudaError_t e = oqd::launch_dense_attention(c->p, q, nq, static_cast<const uint8_t*>(records), n,
                                              values, vdim, n_splits, static_cast<float*>(ws),
                                              out, as_stream(stream));
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "dense attention kernel");
}

oq_status oq_device_alloc(size_t bytes, void** ptr) {
  if (!ptr) return fail(OQ_ERR_INVALID_ARGUMENT, "null output pointer");
  cudaError_t e = cudaMalloc(ptr, bytes ? bytes : 1);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "cudaMalloc");
}

oq_status oq_device_memset(void* ptr, int value, size_t bytes) {
  cudaError_t e = cudaMemset(ptr, value, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "cudaMemset");
}

oq_status oq_device_free(void* ptr) {
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "cudaFree");
}

oq_status oq_copy_to_device(void* dst, const void* src, size_t bytes) {
  cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "cudaMemcpy H2D");
}

oq_status oq_copy_to_host(void* dst, const void* src, size_t bytes) {
  cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? OQ_OK : cuda_fail(e, "cudaMemcpy D2H");
}

// Kernel timing (bench support): enable/disable, then collect the summed
// milliseconds and launch count of every timed launch named `name`.
void oq_timing_enable(int on) {
  for (auto& m : g_timer.marks) {
    cudaEventDestroy(m.second.first);
    cudaEventDestroy(m.second.second);
  }
  g_timer.marks.clear();
  g_timer.on = on != 0;
}

oq_status oq_timing_collect(const char* name, double* total_ms, int* count) {
  double t = 0.0;
  int n = 0;
  for (auto& m : g_timer.marks) {
    if (m.first != name) continue;
    cudaError_t e = cudaEventSynchronize(m.second.second);
    if (e != cudaSuccess) return cuda_fail(e, "event sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, m.second.first, m.second.second);
    t += ms;
    ++n;
  }
  if (total_ms) *total_ms = t;
  if (count) *count = n;
  return OQ_OK;
}

}  // extern "C"
