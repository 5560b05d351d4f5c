/*
 * octo_oracle.c — CPU restatement of the OCTOPUS codec hot path (TEST
 * INFRASTRUCTURE ONLY; see octo_oracle.h for who may use it and how it is
 * pinned).  All references are to /root/reference/proj/include/octoquant/.
 *
 * Arithmetic is written so that each fp64 rounding step matches the
 * reference's scalar evaluation order (compile with -ffp-contract=off).
 */
#include "octo_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================= */
/* rng.hpp:14-19 mix64 (splitmix64 finalizer).                              */
uint64_t orc_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* rng.hpp:26-28 Stream::child. */
uint64_t orc_stream_child(uint64_t seed, uint64_t idx) {
  return orc_mix64(seed ^ orc_mix64(idx ^ 0x632be59bd9b4e019ull));
}

/* rng.hpp:33 Stream::at. */
uint64_t orc_stream_at(uint64_t seed, uint64_t i) {
  return orc_mix64(seed + i * 0x9e3779b97f4a7c15ull);
}

/* rng.hpp:38 next_unit_pos, :41 next_unit. */
static double unit_pos(uint64_t v) { return (double)((v >> 11) + 1) * 0x1.0p-53; }
static double unit(uint64_t v) { return (double)(v >> 11) * 0x1.0p-53; }

/* rng.hpp:44-51 Box-Muller pair. */
static void gaussian_pair(uint64_t seed, uint64_t* ctr, double* z0, double* z1) {
  const double u1 = unit_pos(orc_stream_at(seed, (*ctr)++));
  const double u2 = unit(orc_stream_at(seed, (*ctr)++));
  const double r = sqrt(-2.0 * log(u1));
  const double th = 6.283185307179586476925286766559 * u2;
  *z0 = r * cos(th);
  *z1 = r * sin(th);
}

/* rng.hpp:59-63 fill_gaussian (odd tail takes z0 of a fresh pair). */
uint64_t orc_fill_gaussian(uint64_t seed, uint64_t ctr, double* out, size_t n) {
  size_t i = 0;
  for (; i + 1 < n; i += 2) gaussian_pair(seed, &ctr, &out[i], &out[i + 1]);
  if (i < n) {
    double z1;
    gaussian_pair(seed, &ctr, &out[i], &z1);
  }
  return ctr;
}

void orc_gaussian_f32(uint64_t seed, size_t n, float* out) {
  uint64_t ctr = 0;
  size_t i = 0;
  for (; i + 1 < n; i += 2) {
    double a, b;
    gaussian_pair(seed, &ctr, &a, &b);
    out[i] = (float)a;
    out[i + 1] = (float)b;
  }
  if (i < n) {
    double a, b;
    gaussian_pair(seed, &ctr, &a, &b);
    out[i] = (float)a;
  }
}

/* ======================================================================= */
/* io.hpp:115-138 f32 -> f16, round-nearest-even. */
uint16_t orc_f32_to_f16(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t ex = (x >> 23) & 0xffu;
  uint32_t man = x & 0x7fffffu;
  if (ex == 0xff) return (uint16_t)(sign | 0x7c00u | (man ? 0x200u : 0));
  const int e = (int)ex - 127 + 15;
  if (e >= 31) return (uint16_t)(sign | 0x7c00u);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    man |= 0x800000u;
    const unsigned sh = (unsigned)(14 - e);
    uint32_t half = man >> sh;
    const uint32_t rem = man & ((1u << sh) - 1u);
    const uint32_t mid = 1u << (sh - 1);
    if (rem > mid || (rem == mid && (half & 1u))) ++half;
    return (uint16_t)(sign | half);
  }
  uint32_t half = ((uint32_t)e << 10) | (man >> 13);
  const uint32_t rem = man & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (half & 1u))) ++half;
  return (uint16_t)(sign | half);
}

/* io.hpp:140-166 f16 -> f32. */
float orc_f16_to_f32(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t ex = (h >> 10) & 0x1fu;
  const uint32_t man = h & 0x3ffu;
  uint32_t x;
  if (ex == 0) {
    if (man == 0) {
      x = sign;
    } else {
      int e = -1;
      uint32_t m = man;
      while (!(m & 0x400u)) {
        m <<= 1;
        ++e;
      }
      x = sign | ((uint32_t)(127 - 15 - e) << 23) | ((m & 0x3ffu) << 13);
    }
  } else if (ex == 31) {
    x = sign | 0x7f800000u | (man << 13);
  } else {
    x = sign | ((ex - 15 + 127) << 23) | (man << 13);
  }
  float f;
  memcpy(&f, &x, 4);
  return f;
}

/* ======================================================================= */
/* rotation.hpp:35-40 signs; :20-31 normalized FWHT. */
void orc_rotation_signs(uint32_t dim, uint64_t seed, double* signs) {
  const uint64_t s = orc_mix64(seed);
  for (uint32_t i = 0; i < dim; ++i) signs[i] = (orc_mix64(s ^ i) >> 63) ? -1.0 : 1.0;
}

void orc_fwht(double* x, size_t d) {
  for (size_t len = 1; len < d; len <<= 1)
    for (size_t i = 0; i < d; i += len << 1)
      for (size_t j = i; j < i + len; ++j) {
        const double a = x[j], b = x[j + len];
        x[j] = a + b;
        x[j + len] = a - b;
      }
  const double scale = 1.0 / sqrt((double)d);
  for (size_t i = 0; i < d; ++i) x[i] *= scale;
}

/* rotation.hpp:46-49 apply: y = H (s .* x). */
static void rot_apply(const double* signs, uint32_t d, const double* x, double* y) {
  for (uint32_t i = 0; i < d; ++i) y[i] = x[i] * signs[i];
  orc_fwht(y, d);
}

/* rotation.hpp:52-56 apply_inverse: y = s .* (H x). */
static void rot_apply_inverse(const double* signs, uint32_t d, const double* x, double* y) {
  for (uint32_t i = 0; i < d; ++i) y[i] = x[i];
  orc_fwht(y, d);
  for (uint32_t i = 0; i < d; ++i) y[i] *= signs[i];
}

/* ======================================================================= */
/* octahedral.hpp:15,18,22-31 oct_encode (sign(0)=+1, eps 1e-12). */
static const double kOctEps = 1e-12;
static double sgn_pos(double v) { return v >= 0.0 ? 1.0 : -1.0; }

void orc_oct_encode(const double n[3], double out[2]) {
  const double l1 = fabs(n[0]) + fabs(n[1]) + fabs(n[2]);
  const double inv = 1.0 / (l1 > kOctEps ? l1 : kOctEps);
  const double px = n[0] * inv, py = n[1] * inv, pz = n[2] * inv;
  if (pz >= 0.0) {
    out[0] = px;
    out[1] = py;
    return;
  }
  out[0] = sgn_pos(px) * (1.0 - fabs(py));
  out[1] = sgn_pos(py) * (1.0 - fabs(px));
}

/* octahedral.hpp:34-47 oct_decode. */
void orc_oct_decode(double xi, double eta, double out[3]) {
  xi = xi < -1.0 ? -1.0 : (xi > 1.0 ? 1.0 : xi);
  eta = eta < -1.0 ? -1.0 : (eta > 1.0 ? 1.0 : eta);
  double x = xi, y = eta, z = 1.0 - fabs(xi) - fabs(eta);
  if (z < 0.0) {
    x = sgn_pos(xi) * (1.0 - fabs(eta));
    y = sgn_pos(eta) * (1.0 - fabs(xi));
  }
  const double norm = sqrt(x * x + y * y + z * z);
  const double inv = 1.0 / (norm > kOctEps ? norm : kOctEps);
  out[0] = x * inv;
  out[1] = y * inv;
  out[2] = z * inv;
}

/* ======================================================================= */
/* lloydmax.hpp:46-49 quantize = std::upper_bound count (ties go up). */
uint32_t orc_quantize(const double* b, uint32_t nb, double x) {
  uint32_t lo = 0, hi = nb; /* first index with b[i] > x */
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (!(x < b[mid])) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

static void rebuild_boundaries(const double* c, size_t K, double* b) {
  /* lloydmax.hpp:39-43 */
  for (size_t i = 0; i + 1 < K; ++i) b[i] = 0.5 * (c[i] + c[i + 1]);
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* lloydmax.hpp:72-80 repair_empty. */
static void repair_empty(double* c, size_t K, const double* edges, const double* cell_dist,
                         size_t empty) {
  size_t donor = 0;
  for (size_t i = 1; i < K; ++i)
    if (cell_dist[i] > cell_dist[donor]) donor = i;
  const double width = edges[donor + 1] - edges[donor];
  c[empty] = c[donor] + 0.25 * width;
  qsort(c, K, sizeof(double), cmp_double);
}

/* first index i with s[i] >= v (std::lower_bound). */
static size_t lower_bound_d(const double* s, size_t n, double v) {
  size_t lo = 0, hi = n;
  while (lo < hi) {
    const size_t mid = lo + (hi - lo) / 2;
    if (s[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

#define LLOYD_ITERS 10000
#define LLOYD_TOL 1e-10

/* lloydmax.hpp:152-236 train_from_samples on pre-sorted samples with
 * prefix sums (sorting is value-deterministic, so it is done once). */
static void train_sorted(const double* s, const double* p1, const double* p2, size_t n,
                         int bits, double* c, double* b) {
  const size_t K = (size_t)1 << bits;
  for (size_t i = 0; i < K; ++i) {
    size_t idx = (size_t)(((double)i + 0.5) / (double)K * (double)n);
    if (idx >= n) idx = n - 1;
    c[i] = s[idx];
  }
  double prev = INFINITY;
  size_t* start = malloc((K + 1) * sizeof(size_t));
  double* cell = malloc(K * sizeof(double));
  double* edges = malloc((K + 1) * sizeof(double));
  for (int it = 0; it < LLOYD_ITERS; ++it) {
    rebuild_boundaries(c, K, b);
    start[0] = 0;
    for (size_t i = 0; i + 1 < K; ++i) start[i + 1] = lower_bound_d(s, n, b[i]);
    start[K] = n;
    edges[0] = s[0];
    for (size_t i = 0; i + 1 < K; ++i) edges[i + 1] = b[i];
    edges[K] = s[n - 1];
    double dist = 0.0;
    size_t empty = K;
    for (size_t i = 0; i < K; ++i) {
      const size_t a = start[i], e = start[i + 1];
      const double cnt = (double)(e - a);
      if (e > a) c[i] = (p1[e] - p1[a]) / cnt;
      else if (empty == K) empty = i;
      const double ci = c[i];
      cell[i] = (p2[e] - p2[a]) - 2.0 * ci * (p1[e] - p1[a]) + ci * ci * cnt;
      dist += cell[i];
    }
    if (empty != K) {
      repair_empty(c, K, edges, cell, empty);
      prev = INFINITY;
      continue;
    }
    dist /= (double)n;
    if (prev - dist < LLOYD_TOL * prev) break;
    prev = dist;
  }
  rebuild_boundaries(c, K, b);
  free(start);
  free(cell);
  free(edges);
}

/* ---- quadrature.hpp ------------------------------------------------------
 * quadrature.hpp:21-40: the 32-point Gauss-Legendre rule (positive half).
 * These are mathematical constants; the literal values must be the ones the
 * reference rounds to, so they are restated digit for digit. */
static const double kGlNodes[16] = {
    4.83076656877383104e-02, 1.44471961582796488e-01, 2.39287362252137065e-01,
    3.31868602282127667e-01, 4.21351276130635333e-01, 5.06899908932229359e-01,
    5.87715757240762304e-01, 6.63044266930215231e-01, 7.32182118740289711e-01,
    7.94483795967942386e-01, 8.49367613732569970e-01, 8.96321155766052202e-01,
    9.34906075937739667e-01, 9.64762255587506390e-01, 9.85611511545268382e-01,
    9.97263861849481570e-01,
};
static const double kGlWeights[16] = {
    9.65400885147278121e-02, 9.56387200792748332e-02, 9.38443990808045664e-02,
    9.11738786957638631e-02, 8.76520930044039082e-02, 8.33119242269468457e-02,
    7.81938957870703111e-02, 7.23457941088484491e-02, 6.58222227763617523e-02,
    5.86840934785357038e-02, 5.09980592623762441e-02, 4.28358980222264263e-02,
    3.42738629130216257e-02, 2.53920653092624266e-02, 1.62743947309059653e-02,
    7.01861000946929839e-03,
};

typedef double (*density_fn)(double x, const void* ctx);
typedef struct { double mass, mean1, mean2; } moments;

/* quadrature.hpp:151-169 MomentTable::panel — one 32-node panel. */
static moments gl_panel(density_fn f, const void* ctx, double a, double b) {
  moments m = {0.0, 0.0, 0.0};
  if (!(b > a)) return m;
  const double mid = 0.5 * (a + b), half = 0.5 * (b - a);
  double m0 = 0.0, m1 = 0.0, m2 = 0.0;
  for (int i = 0; i < 16; ++i) {
    const double off = half * kGlNodes[i];
    const double xl = mid - off, xr = mid + off;
    const double fl = f(xl, ctx), fr = f(xr, ctx);
    const double w = kGlWeights[i];
    m0 += w * (fl + fr);
    m1 += w * (fl * xl + fr * xr);
    m2 += w * (fl * xl * xl + fr * xr * xr);
  }
  m.mass = m0 * half;
  m.mean1 = m1 * half;
  m.mean2 = m2 * half;
  return m;
}

typedef struct {
  density_fn f;
  const void* ctx;
  double lo, hi, h;
  int n;
  double *c0, *c1, *c2;
} moment_table;

/* quadrature.hpp:105-124 MomentTable ctor: long-double prefix sums. */
static void mt_init(moment_table* t, density_fn f, const void* ctx, double lo, double hi,
                    int panels) {
  t->f = f;
  t->ctx = ctx;
  t->lo = lo;
  t->hi = hi;
  t->n = panels;
  t->h = (hi - lo) / panels;
  t->c0 = calloc((size_t)panels + 1, sizeof(double));
  t->c1 = calloc((size_t)panels + 1, sizeof(double));
  t->c2 = calloc((size_t)panels + 1, sizeof(double));
  long double a0 = 0.0L, a1 = 0.0L, a2 = 0.0L;
  for (int p = 0; p < panels; ++p) {
    const moments m = gl_panel(f, ctx, lo + p * t->h, lo + (p + 1) * t->h);
    a0 += m.mass;
    a1 += m.mean1;
    a2 += m.mean2;
    t->c0[p + 1] = (double)a0;
    t->c1[p + 1] = (double)a1;
    t->c2[p + 1] = (double)a2;
  }
}

static void mt_free(moment_table* t) {
  free(t->c0);
  free(t->c1);
  free(t->c2);
}

/* quadrature.hpp:144-149 index. */
static int mt_index(const moment_table* t, double x) {
  int i = (int)((x - t->lo) / t->h);
  if (i < 0) i = 0;
  if (i > t->n - 1) i = t->n - 1;
  return i;
}

/* quadrature.hpp:126-140 cell. */
static moments mt_cell(const moment_table* t, double a, double b) {
  moments m = {0.0, 0.0, 0.0};
  if (!(b > a)) return m;
  a = a > t->lo ? a : t->lo;
  b = b < t->hi ? b : t->hi;
  const int ia = mt_index(t, a), ib = mt_index(t, b);
  if (ia == ib) return gl_panel(t->f, t->ctx, a, b);
  m = gl_panel(t->f, t->ctx, a, t->lo + (ia + 1) * t->h);
  const moments r = gl_panel(t->f, t->ctx, t->lo + ib * t->h, b);
  m.mass += t->c0[ib] - t->c0[ia + 1] + r.mass;
  m.mean1 += t->c1[ib] - t->c1[ia + 1] + r.mean1;
  m.mean2 += t->c2[ib] - t->c2[ia + 1] + r.mean2;
  return m;
}

/* quadrature.hpp:178-218 CdfTable (composite Simpson) + quantile. */
typedef struct {
  double lo, hi, total;
  size_t size;
  double* cum;
} cdf_table;

static void cdf_init(cdf_table* t, density_fn f, const void* ctx, double lo, double hi,
                     int panels) {
  t->lo = lo;
  t->hi = hi;
  t->size = (size_t)panels + 1;
  t->cum = malloc(t->size * sizeof(double));
  const double h = (hi - lo) / panels;
  t->cum[0] = 0.0;
  double prev = f(lo, ctx);
  for (int p = 0; p < panels; ++p) {
    const double a = lo + p * h;
    const double fm = f(a + 0.5 * h, ctx);
    const double fb = f(a + h, ctx);
    t->cum[p + 1] = t->cum[p] + (h / 6.0) * (prev + 4.0 * fm + fb);
    prev = fb;
  }
  t->total = t->cum[panels];
}

static double cdf_quantile(const cdf_table* t, double q) {
  const double target = q * t->total;
  size_t a = 0, b = t->size - 1;
  while (b - a > 1) {
    const size_t m = (a + b) / 2;
    if (t->cum[m] < target) a = m;
    else b = m;
  }
  const double span = t->cum[b] - t->cum[a];
  const double frac = span > 0.0 ? (target - t->cum[a]) / span : 0.5;
  const double h = (t->hi - t->lo) / (double)(t->size - 1);
  return t->lo + ((double)a + frac) * h;
}

/* lloydmax.hpp:84-150 train_from_density. */
static void train_density(density_fn f, const void* ctx, double lo, double hi, int bits,
                          double* c, double* b) {
  const size_t K = (size_t)1 << bits;
  cdf_table cdf;
  cdf_init(&cdf, f, ctx, lo, hi, 1 << 15);
  moment_table tab;
  mt_init(&tab, f, ctx, lo, hi, 128 * (int)K);
  for (size_t i = 0; i < K; ++i) c[i] = cdf_quantile(&cdf, ((double)i + 0.5) / (double)K);
  double prev = INFINITY;
  double* prevc = malloc(K * sizeof(double));
  double* edges = malloc((K + 1) * sizeof(double));
  double* cell = malloc(K * sizeof(double));
  for (int it = 0; it < LLOYD_ITERS; ++it) {
    rebuild_boundaries(c, K, b);
    edges[0] = lo;
    for (size_t i = 0; i + 1 < K; ++i) edges[i + 1] = b[i];
    edges[K] = hi;
    memcpy(prevc, c, K * sizeof(double));
    double total = 0.0, dist = 0.0;
    size_t empty = K;
    for (size_t i = 0; i < K; ++i) {
      const moments m = mt_cell(&tab, edges[i], edges[i + 1]);
      total += m.mass;
      if (m.mass > 0.0) c[i] = m.mean1 / m.mass;
      else if (empty == K) empty = i;
      const double ci = c[i];
      cell[i] = m.mean2 - 2.0 * ci * m.mean1 + ci * ci * m.mass;
      dist += cell[i];
    }
    if (empty != K) {
      repair_empty(c, K, edges, cell, empty);
      prev = INFINITY;
      continue;
    }
    dist /= total;
    if (dist > prev) {
      memcpy(c, prevc, K * sizeof(double));
      break;
    }
    if (prev - dist < LLOYD_TOL * prev) break;
    prev = dist;
  }
  rebuild_boundaries(c, K, b);
  free(prevc);
  free(edges);
  free(cell);
  free(cdf.cum);
  mt_free(&tab);
}

/* marginals.hpp:36-44 triplet_norm_density, with :15-17 log_beta. */
static double triplet_norm_density(double r, const void* ctx) {
  const uint32_t d = *(const uint32_t*)ctx;
  const double a = 1.5, bb = 0.5 * (d - 3.0);
  const double log_norm = lgamma(a) + lgamma(bb) - lgamma(a + bb);
  const double e = 0.5 * (d - 5.0);
  const double base = 1.0 - r * r;
  return 2.0 * r * r * pow(base, e) / exp(log_norm);
}

/* books.hpp:23-24,49-64 the fixed empirical draw for the xi book:
 * 2^21 sphere points from Stream(0xC0DEB00C), each consuming four draws
 * (marginals.hpp:66-79 sample_unit_sphere(3) -> fill_gaussian(3)). */
#define XI_SEED 0xC0DEB00Cull
#define XI_POINTS (1u << 21)

typedef struct {
  double* s;
  double *p1, *p2;
  size_t n;
} xi_samples;

static pthread_mutex_t g_book_mu = PTHREAD_MUTEX_INITIALIZER;
static xi_samples g_xi = {0, 0, 0, 0};

typedef struct {
  uint32_t lo, hi;
  double* out;
} xi_job;

static void* xi_worker(void* arg) {
  xi_job* j = (xi_job*)arg;
  for (uint32_t i = j->lo; i < j->hi; ++i) {
    double n[3], z1;
    uint64_t ctr = 4ull * i;
    gaussian_pair(XI_SEED, &ctr, &n[0], &n[1]);
    gaussian_pair(XI_SEED, &ctr, &n[2], &z1);
    double s = 0.0;
    for (int k = 0; k < 3; ++k) s += n[k] * n[k];
    const double inv = 1.0 / sqrt(s);
    for (int k = 0; k < 3; ++k) n[k] *= inv;
    double fe[2];
    orc_oct_encode(n, fe);
    j->out[2 * (size_t)i] = fe[0];
    j->out[2 * (size_t)i + 1] = fe[1];
  }
  return 0;
}

static const xi_samples* xi_training(void) {
  if (g_xi.s) return &g_xi;
  const size_t n = 2 * (size_t)XI_POINTS;
  double* s = malloc(n * sizeof(double));
  enum { NT = 8 };
  pthread_t th[NT];
  xi_job jobs[NT];
  for (int t = 0; t < NT; ++t) {
    jobs[t].lo = (uint32_t)((uint64_t)XI_POINTS * t / NT);
    jobs[t].hi = (uint32_t)((uint64_t)XI_POINTS * (t + 1) / NT);
    jobs[t].out = s;
    pthread_create(&th[t], 0, xi_worker, &jobs[t]);
  }
  for (int t = 0; t < NT; ++t) pthread_join(th[t], 0);
  qsort(s, n, sizeof(double), cmp_double);
  double* p1 = malloc((n + 1) * sizeof(double));
  double* p2 = malloc((n + 1) * sizeof(double));
  p1[0] = p2[0] = 0.0;
  for (size_t i = 0; i < n; ++i) {
    p1[i + 1] = p1[i] + s[i];
    p2[i + 1] = p2[i] + s[i] * s[i];
  }
  g_xi.p1 = p1;
  g_xi.p2 = p2;
  g_xi.n = n;
  g_xi.s = s;
  return &g_xi;
}

/* Registry caches (books.hpp:28-47): xi by bits, rho by (dim, bits). */
typedef struct {
  int kind;
  uint32_t dim;
  int bits;
  double* c;
  double* b;
} book_entry;
static book_entry g_books[256];
static int g_nbooks = 0;

static const book_entry* get_book(int kind, uint32_t dim, int bits) {
  pthread_mutex_lock(&g_book_mu);
  for (int i = 0; i < g_nbooks; ++i)
    if (g_books[i].kind == kind && g_books[i].dim == dim && g_books[i].bits == bits) {
      pthread_mutex_unlock(&g_book_mu);
      return &g_books[i];
    }
  const size_t K = (size_t)1 << bits;
  double* c = malloc(K * sizeof(double));
  double* b = malloc(K * sizeof(double));
  if (kind == 0) {
    /* books.hpp:69-74 xi_book: samples on [-1, 1]. */
    const xi_samples* xs = xi_training();
    train_sorted(xs->s, xs->p1, xs->p2, xs->n, bits, c, b);
  } else {
    /* books.hpp:86-95 rho_book: density on [0, hi], hi shaved at d=4. */
    const double hi = dim == 4 ? 1.0 - 0x1p-40 : 1.0;
    train_density(triplet_norm_density, &dim, 0.0, hi, bits, c, b);
  }
  book_entry* e = &g_books[g_nbooks++];
  e->kind = kind;
  e->dim = dim;
  e->bits = bits;
  e->c = c;
  e->b = b;
  pthread_mutex_unlock(&g_book_mu);
  return e;
}

int orc_xi_book(int bits, double* c, double* b) {
  if (bits < 1 || bits > 12) return -1;
  const book_entry* e = get_book(0, 0, bits);
  const size_t K = (size_t)1 << bits;
  memcpy(c, e->c, K * sizeof(double));
  memcpy(b, e->b, (K - 1) * sizeof(double));
  return 0;
}

int orc_rho_book(uint32_t dim, int bits, double* c, double* b) {
  if (bits < 1 || bits > 12 || dim < 4) return -1;
  const book_entry* e = get_book(1, dim, bits);
  const size_t K = (size_t)1 << bits;
  memcpy(c, e->c, K * sizeof(double));
  memcpy(b, e->b, (K - 1) * sizeof(double));
  return 0;
}

/* ======================================================================= */
/* codec.hpp */
struct orc_encoder {
  orc_config cfg;
  uint32_t nt, K, KR;
  const double *xc, *xb, *rc, *rb;
  double* dirs; /* K*K*3, codec.hpp:100-107 build_dir_table */
  double* signs;
  double* qsigns;
};

orc_encoder* orc_encoder_new(const orc_config* cfg) {
  /* codec.hpp:65-72 validate */
  const uint32_t d = cfg->dim;
  if (d < 4 || (d & (d - 1))) return 0;
  if (cfg->b_dir < 1 || cfg->b_dir > 8 || cfg->b_nrm < 1 || cfg->b_nrm > 8) return 0;
  if (cfg->qjl && cfg->qjl_seed == cfg->rotation_seed) return 0;
  orc_encoder* e = calloc(1, sizeof(orc_encoder));
  e->cfg = *cfg;
  e->nt = (d + 2) / 3;
  const book_entry* xb = get_book(0, 0, cfg->b_dir);
  const book_entry* rb = get_book(1, d, cfg->b_nrm);
  e->K = 1u << cfg->b_dir;
  e->KR = 1u << cfg->b_nrm;
  e->xc = xb->c;
  e->xb = xb->b;
  e->rc = rb->c;
  e->rb = rb->b;
  e->dirs = malloc((size_t)e->K * e->K * 3 * sizeof(double));
  for (uint32_t a = 0; a < e->K; ++a)
    for (uint32_t b = 0; b < e->K; ++b) orc_oct_decode(e->xc[a], e->xc[b], &e->dirs[3 * (a * e->K + b)]);
  e->signs = malloc(d * sizeof(double));
  orc_rotation_signs(d, cfg->rotation_seed, e->signs);
  e->qsigns = malloc(d * sizeof(double));
  orc_rotation_signs(d, cfg->qjl_seed, e->qsigns);
  return e;
}

void orc_encoder_free(orc_encoder* e) {
  if (!e) return;
  free(e->dirs);
  free(e->signs);
  free(e->qsigns);
  free(e);
}

size_t orc_record_bytes(const orc_config* cfg) {
  /* codec.hpp:427-430 */
  const size_t nt = (cfg->dim + 2) / 3;
  size_t r = 4 + (2 * nt * cfg->b_dir + 7) / 8 + (nt * cfg->b_nrm + 7) / 8;
  if (cfg->qjl) r += 2 + (cfg->dim + 7) / 8;
  return r;
}

/* codec.hpp:143-195 joint_round_triplet. */
static void joint_round(const orc_encoder* e, const double t[3], uint32_t* ixi, uint32_t* ieta,
                        uint32_t* irho) {
  const uint32_t K = e->K;
  double fe[2];
  orc_oct_encode(t, fe);
  const uint32_t sx = orc_quantize(e->xb, K - 1, fe[0]);
  const uint32_t sy = orc_quantize(e->xb, K - 1, fe[1]);
  const int mode = e->cfg.rounding;
  if (mode == 0) {
    double r = sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
    r = r < 0.0 ? 0.0 : (r > 1.0 ? 1.0 : r);
    *ixi = sx;
    *ieta = sy;
    *irho = orc_quantize(e->rb, e->KR - 1, r);
    return;
  }
  uint32_t ax0 = sx, ax1 = sx, ay0 = sy, ay1 = sy;
  if (mode == 1) {
    ax1 = sx + 1 < K - 1 ? sx + 1 : K - 1;
    ay1 = sy + 1 < K - 1 ? sy + 1 : K - 1;
  } else if (mode == 2) {
    ax0 = sx > 0 ? sx - 1 : 0;
    ay0 = sy > 0 ? sy - 1 : 0;
    ax1 = sx + 1 < K - 1 ? sx + 1 : K - 1;
    ay1 = sy + 1 < K - 1 ? sy + 1 : K - 1;
  } else {
    ax0 = ay0 = 0;
    ax1 = ay1 = K - 1;
  }
  double best = -INFINITY;
  uint32_t bx = ax0, by = ay0;
  for (uint32_t a = ax0; a <= ax1; ++a)
    for (uint32_t b = ay0; b <= ay1; ++b) {
      const double* n = &e->dirs[3 * (a * K + b)];
      const double s = t[0] * n[0] + t[1] * n[1] + t[2] * n[2];
      if (s > best) {
        best = s;
        bx = a;
        by = b;
      }
    }
  *ixi = bx;
  *ieta = by;
  const double cl = best < 0.0 ? 0.0 : (best > 1.0 ? 1.0 : best);
  *irho = orc_quantize(e->rb, e->KR - 1, cl);
}

/* io.hpp:66-85 BitWriter semantics: LSB-first fields, zero byte padding. */
static void put_bits(uint8_t* buf, size_t* pos, uint32_t v, unsigned bits) {
  for (unsigned i = 0; i < bits; ++i) {
    if ((v >> i) & 1u) buf[*pos >> 3] |= (uint8_t)(1u << (*pos & 7));
    ++*pos;
  }
}

static uint32_t get_bits(const uint8_t* buf, size_t* pos, unsigned bits) {
  uint32_t v = 0;
  for (unsigned i = 0; i < bits; ++i) {
    if ((buf[*pos >> 3] >> (*pos & 7)) & 1u) v |= 1u << i;
    ++*pos;
  }
  return v;
}

/* codec.hpp:252-266 reconstruct_rotated (truncated to d). */
static void reconstruct_rotated(const orc_encoder* e, const uint16_t* dir, const uint16_t* nrm,
                                double* out) {
  const uint32_t d = e->cfg.dim;
  for (uint32_t i = 0; i < d; ++i) out[i] = 0.0;
  for (uint32_t t = 0; t < e->nt; ++t) {
    const double* n = &e->dirs[3 * (dir[2 * t] * e->K + dir[2 * t + 1])];
    const double r = e->rc[nrm[t]];
    for (uint32_t j = 0; j < 3 && 3 * t + j < d; ++j) out[3 * t + j] = r * n[j];
  }
}

/* codec.hpp:214-249 Encoder::encode, serialized as one pack_keys record
 * (codec.hpp:381-393). */
void orc_encode_record(const orc_encoder* e, const double* k, uint8_t* rec) {
  const uint32_t d = e->cfg.dim, nt = e->nt;
  double g2 = 0.0;
  for (uint32_t i = 0; i < d; ++i) g2 += k[i] * k[i];
  const double gamma = sqrt(g2);
  const double inv = 1.0 / (gamma > 1e-12 ? gamma : 1e-12);
  double u[256], ur[256], padded[258];
  for (uint32_t i = 0; i < d; ++i) u[i] = k[i] * inv;
  rot_apply(e->signs, d, u, ur);
  for (uint32_t i = 0; i < 3 * nt; ++i) padded[i] = i < d ? ur[i] : 0.0;
  uint16_t dir[2 * 86], nrm[86];
  for (uint32_t t = 0; t < nt; ++t) {
    uint32_t a, b, r;
    joint_round(e, &padded[3 * t], &a, &b, &r);
    dir[2 * t] = (uint16_t)a;
    dir[2 * t + 1] = (uint16_t)b;
    nrm[t] = (uint16_t)r;
  }
  const float gf = (float)gamma;
  memset(rec, 0, orc_record_bytes(&e->cfg));
  memcpy(rec, &gf, 4);
  size_t off = 4;
  const size_t db = (2 * (size_t)nt * e->cfg.b_dir + 7) / 8;
  const size_t nb = ((size_t)nt * e->cfg.b_nrm + 7) / 8;
  size_t pos = 0;
  for (uint32_t i = 0; i < 2 * nt; ++i) put_bits(rec + off, &pos, dir[i], e->cfg.b_dir);
  off += db;
  pos = 0;
  for (uint32_t i = 0; i < nt; ++i) put_bits(rec + off, &pos, nrm[i], e->cfg.b_nrm);
  off += nb;
  if (e->cfg.qjl) {
    /* codec.hpp:243-247 + qjl.hpp:23-36 */
    double uh[256], r[256], w[256];
    reconstruct_rotated(e, dir, nrm, uh);
    for (uint32_t i = 0; i < d; ++i) r[i] = ur[i] - uh[i];
    rot_apply(e->qsigns, d, r, w);
    double n2 = 0.0;
    for (uint32_t i = 0; i < d; ++i) n2 += r[i] * r[i];
    const uint16_t gr = orc_f32_to_f16((float)sqrt(n2));
    memcpy(rec + off, &gr, 2);
    off += 2;
    for (uint32_t i = 0; i < d; ++i)
      if (w[i] >= 0.0) rec[off + (i >> 3)] |= (uint8_t)(1u << (i & 7));
  }
}

typedef struct {
  const orc_encoder* e;
  const float* x;
  uint8_t* recs;
  size_t lo, hi, rb;
} enc_job;

static void* enc_worker(void* arg) {
  enc_job* j = (enc_job*)arg;
  const uint32_t d = j->e->cfg.dim;
  double k[256];
  for (size_t v = j->lo; v < j->hi; ++v) {
    for (uint32_t i = 0; i < d; ++i) k[i] = (double)j->x[v * d + i];
    orc_encode_record(j->e, k, j->recs + v * j->rb);
  }
  return 0;
}

void orc_encode_f32(const orc_encoder* e, const float* x, size_t n, uint8_t* recs, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  enc_job jobs[256];
  const size_t rb = orc_record_bytes(&e->cfg);
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (enc_job){e, x, recs, n * t / threads, n * (t + 1) / threads, rb};
    pthread_create(&th[t], 0, enc_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], 0);
}

int orc_record_codes(const orc_config* cfg, const uint8_t* rec, float* gamma, uint16_t* dir,
                     uint16_t* nrm, uint16_t* gamma_r, uint8_t* signs) {
  const size_t nt = (cfg->dim + 2) / 3;
  const size_t db = (2 * nt * cfg->b_dir + 7) / 8;
  const size_t nb = (nt * cfg->b_nrm + 7) / 8;
  memcpy(gamma, rec, 4);
  size_t pos = 0;
  for (size_t i = 0; i < 2 * nt; ++i) dir[i] = (uint16_t)get_bits(rec + 4, &pos, cfg->b_dir);
  /* codec.hpp:447 padding_clear */
  for (; pos < db * 8; ++pos)
    if ((rec[4 + (pos >> 3)] >> (pos & 7)) & 1u) return -1;
  pos = 0;
  for (size_t i = 0; i < nt; ++i) nrm[i] = (uint16_t)get_bits(rec + 4 + db, &pos, cfg->b_nrm);
  for (; pos < nb * 8; ++pos)
    if ((rec[4 + db + (pos >> 3)] >> (pos & 7)) & 1u) return -1;
  if (cfg->qjl) {
    memcpy(gamma_r, rec + 4 + db + nb, 2);
    memcpy(signs, rec + 4 + db + nb + 2, (cfg->dim + 7) / 8);
  }
  return 0;
}

/* codec.hpp:319-330 check_codes. */
static int check_codes(const orc_encoder* e, const uint16_t* dir, const uint16_t* nrm) {
  for (uint32_t t = 0; t < e->nt; ++t) {
    if (dir[2 * t] >= e->K || dir[2 * t + 1] >= e->K) return -1;
    if (nrm[t] >= e->KR) return -1;
  }
  return 0;
}

/* codec.hpp:268-275 Encoder::decode. */
int orc_decode_records(const orc_encoder* e, const uint8_t* recs, size_t n, double* out) {
  const uint32_t d = e->cfg.dim;
  const size_t rb = orc_record_bytes(&e->cfg);
  for (size_t v = 0; v < n; ++v) {
    float g;
    uint16_t dir[2 * 86], nrm[86], gr;
    uint8_t sg[32];
    if (orc_record_codes(&e->cfg, recs + v * rb, &g, dir, nrm, &gr, sg)) return -1;
    if (check_codes(e, dir, nrm)) return -1;
    double ur[256];
    reconstruct_rotated(e, dir, nrm, ur);
    double* u = out + v * d;
    rot_apply_inverse(e->signs, d, ur, u);
    const double gamma = g;
    for (uint32_t i = 0; i < d; ++i) u[i] *= gamma;
  }
  return 0;
}

/* codec.hpp:282-292 prepare; :295-316 score; qjl.hpp:39-48 estimate. */
typedef struct {
  double rot[256], sketch[256];
} prepared;

static void prepare(const orc_encoder* e, const double* q, prepared* p) {
  rot_apply(e->signs, e->cfg.dim, q, p->rot);
  if (e->cfg.qjl) rot_apply(e->qsigns, e->cfg.dim, p->rot, p->sketch);
}

static double score_codes(const orc_encoder* e, const prepared* p, float gamma,
                          const uint16_t* dir, const uint16_t* nrm, uint16_t gr,
                          const uint8_t* sg) {
  const uint32_t d = e->cfg.dim;
  double acc = 0.0;
  for (uint32_t t = 0; t < e->nt; ++t) {
    const double* n = &e->dirs[3 * (dir[2 * t] * e->K + dir[2 * t + 1])];
    double dot = 0.0;
    for (uint32_t j = 0; j < 3 && 3 * t + j < d; ++j) dot += p->rot[3 * t + j] * n[j];
    acc += e->rc[nrm[t]] * dot;
  }
  double est = acc;
  if (e->cfg.qjl) {
    double a = 0.0;
    for (uint32_t i = 0; i < d; ++i) {
      const int pos = (sg[i >> 3] >> (i & 7)) & 1u;
      a += pos ? p->sketch[i] : -p->sketch[i];
    }
    const double g_r = orc_f16_to_f32(gr);
    est += sqrt(1.5707963267948966 / (double)d) * g_r * a;
  }
  return (double)gamma * est;
}

double orc_score(const orc_encoder* e, const double* q, const uint8_t* rec) {
  prepared p;
  prepare(e, q, &p);
  float g;
  uint16_t dir[2 * 86], nrm[86], gr = 0;
  uint8_t sg[32];
  if (orc_record_codes(&e->cfg, rec, &g, dir, nrm, &gr, sg) || check_codes(e, dir, nrm))
    return NAN;
  return score_codes(e, &p, g, dir, nrm, gr, sg);
}

/* attention.hpp:20-45 SoftmaxState push/merge. */
static void sm_push(double* m, double* l, double* acc, double s, const double* v, size_t w) {
  const double mn = s > *m ? s : *m;
  const double scale = exp(*m - mn);
  const double wt = exp(s - mn);
  *l = *l * scale + wt;
  for (size_t j = 0; j < w; ++j) acc[j] = acc[j] * scale + wt * v[j];
  *m = mn;
}

static void sm_merge(double* m, double* l, double* acc, double om, double ol, const double* oacc,
                     size_t w) {
  if (ol == 0.0) return;
  const double mn = *m > om ? *m : om;
  const double sa = exp(*m - mn);
  const double sb = exp(om - mn);
  *l = *l * sa + ol * sb;
  for (size_t j = 0; j < w; ++j) acc[j] = acc[j] * sa + oacc[j] * sb;
  *m = mn;
}

void orc_attention_partial(const orc_encoder* ek, const double* q, const uint8_t* krecs,
                           size_t begin, size_t end, const double* values, size_t vdim,
                           double* m, double* l, double* acc) {
  prepared p;
  prepare(ek, q, &p);
  const double inv_sqrt_d = 1.0 / sqrt((double)ek->cfg.dim);
  const size_t rb = orc_record_bytes(&ek->cfg);
  *m = -INFINITY;
  *l = 0.0;
  for (size_t j = 0; j < vdim; ++j) acc[j] = 0.0;
  for (size_t t = begin; t < end; ++t) {
    float g;
    uint16_t dir[2 * 86], nrm[86], gr = 0;
    uint8_t sg[32];
    orc_record_codes(&ek->cfg, krecs + t * rb, &g, dir, nrm, &gr, sg);
    const double s = score_codes(ek, &p, g, dir, nrm, gr, sg) * inv_sqrt_d;
    sm_push(m, l, acc, s, values + t * vdim, vdim);
  }
}

/* attention.hpp:50-73 attention_decode. */
int orc_attention(const orc_encoder* ek, const double* q, const uint8_t* krecs, size_t n,
                  const double* values, size_t vdim, int n_splits, double* out) {
  if (n == 0 || n_splits < 1) return -1;
  const size_t chunk = (n + (size_t)n_splits - 1) / (size_t)n_splits;
  double M = -INFINITY, L = 0.0;
  double* acc = calloc(vdim, sizeof(double));
  double* part = calloc(vdim, sizeof(double));
  for (size_t begin = 0; begin < n; begin += chunk) {
    const size_t end = begin + chunk < n ? begin + chunk : n;
    double pm, pl;
    orc_attention_partial(ek, q, krecs, begin, end, values, vdim, &pm, &pl, part);
    sm_merge(&M, &L, acc, pm, pl, part, vdim);
  }
  for (size_t j = 0; j < vdim; ++j) out[j] = acc[j] / L;
  free(acc);
  free(part);
  return 0;
}

/* codec.hpp:369-375 header. */
void orc_wire_header(const orc_config* cfg, uint64_t count, uint8_t hdr[20]) {
  memcpy(hdr, "OCTO", 4);
  hdr[4] = 1;
  hdr[5] = cfg->qjl ? 1 : 0;
  hdr[6] = cfg->b_dir;
  hdr[7] = cfg->b_nrm;
  memcpy(hdr + 8, &cfg->dim, 4);
  memcpy(hdr + 12, &count, 8);
}

/* codec.hpp:410-465 unpack_keys validation. */
int orc_unpack_check(const uint8_t* p, size_t n, orc_config* cfg, uint64_t* count) {
  if (n < 20 || memcmp(p, "OCTO", 4) != 0 || p[4] != 1) return -1;
  if (p[5] & ~1u) return -1;
  memset(cfg, 0, sizeof(*cfg));
  cfg->qjl = p[5] & 1u;
  cfg->b_dir = p[6];
  cfg->b_nrm = p[7];
  if (cfg->b_dir < 1 || cfg->b_dir > 8 || cfg->b_nrm < 1 || cfg->b_nrm > 8) return -1;
  memcpy(&cfg->dim, p + 8, 4);
  if (cfg->dim < 4 || (cfg->dim & (cfg->dim - 1))) return -1;
  memcpy(count, p + 12, 8);
  const size_t rb = orc_record_bytes(cfg);
  if (n - 20 != *count * rb) return -1;
  for (uint64_t i = 0; i < *count; ++i) {
    float g;
    uint16_t dir[2 * 86], nrm[86], gr;
    uint8_t sg[32];
    const uint8_t* rec = p + 20 + i * rb;
    if (orc_record_codes(cfg, rec, &g, dir, nrm, &gr, sg)) return -1;
    if (cfg->qjl && cfg->dim % 8 != 0) {
      const uint8_t mask = (uint8_t)(0xffu << (cfg->dim % 8));
      if (sg[(cfg->dim + 7) / 8 - 1] & mask) return -1;
    }
  }
  return 0;
}
