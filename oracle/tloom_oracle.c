/*
 * tloom_oracle.c -- TEST INFRASTRUCTURE ONLY (see tloom_oracle.h).
 *
 * A fixed-order CPU restatement of the reference's training path.  Every
 * summation below reproduces the reference's per-element order exactly
 * (sequential fp32 accumulators starting at 0.0f, each product rounded before
 * it is added -- no FMA), so results are bit-identical to the reference
 * library on the same inputs.  This is pinned by tests/test_oracle.py against
 * oracle/_ref (the reference compiled from its own sources) and against the
 * committed golden vectors in tests/golden/.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, no -march).
 */
#include "tloom_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (the engine the reference pins in network.cpp:57 and     */
/* synth.cpp:119).  Standard MT19937-64 parameters.                          */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* net::init_params (network.cpp:56-79): Glorot uniform from the top 24 bits of
 * each draw, tensors filled row-major k1 -> k2 -> fc, biases zero. */
void orc_init_params(uint64_t seed, float* p) {
  mt64 g;
  mt64_seed(&g, seed);
  memset(p, 0, sizeof(float) * ORC_NPARAM);
  const struct { int off, n, fan_in, fan_out; } t[3] = {
      {ORC_K1, 150, 25, 576}, {ORC_K2, 1800, 150, 64}, {ORC_FC, 1920, 192, 1}};
  for (int k = 0; k < 3; ++k) {
    const float limit = sqrtf(6.0f / (float)(t[k].fan_in + t[k].fan_out));
    for (int i = 0; i < t[k].n; ++i) {
      const float u = (float)(mt64_next(&g) >> 40) * 0x1p-24f;
      p[t[k].off + i] = (u * 2.0f - 1.0f) * limit;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* synth::make_digits (synth.cpp:117-153).  The 5x7 font is data.            */
/* ------------------------------------------------------------------------ */
/* 5x7 font as row bitmasks (bit 4 = leftmost column); same glyphs as synth.cpp:14-94. */
static const uint8_t kGlyphRows[10][7] = {
    {0x0E, 0x11, 0x13, 0x15, 0x19, 0x11, 0x0E}, {0x04, 0x0C, 0x04, 0x04, 0x04, 0x04, 0x0E},
    {0x0E, 0x11, 0x01, 0x02, 0x04, 0x08, 0x1F}, {0x0E, 0x11, 0x01, 0x06, 0x01, 0x11, 0x0E},
    {0x02, 0x06, 0x0A, 0x12, 0x1F, 0x02, 0x02}, {0x1F, 0x10, 0x1E, 0x01, 0x01, 0x11, 0x0E},
    {0x06, 0x08, 0x10, 0x1E, 0x11, 0x11, 0x0E}, {0x1F, 0x01, 0x02, 0x02, 0x04, 0x04, 0x04},
    {0x0E, 0x11, 0x11, 0x0E, 0x11, 0x11, 0x0E}, {0x0E, 0x11, 0x11, 0x0F, 0x01, 0x02, 0x0C},
};

static double glyph_cell(int d, int gy, int gx) { /* synth.cpp:96-100 */
  if (gx < 0 || gx >= 5 || gy < 0 || gy >= 7) return 0.0;
  return ((kGlyphRows[d][gy] >> (4 - gx)) & 1) ? 1.0 : 0.0;
}

static double glyph_sample(int d, double gx, double gy) { /* synth.cpp:102-113 */
  const double fx = floor(gx), fy = floor(gy);
  const int ix = (int)fx, iy = (int)fy;
  const double wx = gx - fx, wy = gy - fy;
  return glyph_cell(d, iy, ix) * (1 - wx) * (1 - wy) + glyph_cell(d, iy, ix + 1) * wx * (1 - wy) +
         glyph_cell(d, iy + 1, ix) * (1 - wx) * wy + glyph_cell(d, iy + 1, ix + 1) * wx * wy;
}

void orc_make_digits(int64_t n, uint64_t seed, uint8_t* pixels, int32_t* labels) {
  mt64 g;
  mt64_seed(&g, seed);
#define U01() ((double)(mt64_next(&g) >> 40) * 0x1p-24)
  for (int64_t img = 0; img < n; ++img) {
    const int digit = (int)(img % 10);
    const double sx = 3.3 + (3.7 - 3.3) * U01();
    const double sy = 3.3 + (3.7 - 3.3) * U01();
    const double tx = -0.8 + (0.8 - -0.8) * U01();
    const double ty = -0.8 + (0.8 - -0.8) * U01();
    labels[img] = digit;
    uint8_t* out = pixels + img * 784;
    for (int y = 0; y < 28; ++y)
      for (int x = 0; x < 28; ++x) {
        const double gx = (x - 13.5 - tx) / sx + (5 - 1) / 2.0;
        const double gy = (y - 13.5 - ty) / sy + (7 - 1) / 2.0;
        double v = glyph_sample(digit, gx, gy) + 0.02 * U01();
        v = fmin(fmax(v, 0.0), 1.0);
        out[y * 28 + x] = (uint8_t)lround(v * 255.0);
      }
  }
#undef U01
}

void orc_make_set(int64_t n, uint64_t seed, float* images, int32_t* labels) {
  uint8_t* px = (uint8_t*)malloc((size_t)(n > 0 ? n : 1) * 784);
  orc_make_digits(n, seed, px, labels);
  for (int64_t i = 0; i < n * 784; ++i) images[i] = (float)px[i] / 255.0f; /* synth.cpp:155-161 */
  free(px);
}

/* ------------------------------------------------------------------------ */
/* expf.  The reference calls std::exp(float) -> glibc 2.39 expf (IFUNC).    */
/* orc_expf_port restates that algorithm (ARM optimized-routines, N=32) in   */
/* its FMA placement; the CUDA exact mode uses the same restatement.         */
/* ------------------------------------------------------------------------ */
float orc_expf(float x) { return expf(x); }

static const uint64_t kExpTab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL,
};

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint64_t d2u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static inline double u2d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }

float orc_expf_port(float x) {
  const double xd = (double)x;
  const uint32_t abstop = (f2u(x) >> 20) & 0x7ff;
  if (abstop >= (f2u(88.0f) >> 20)) {
    if (f2u(x) == f2u(-INFINITY)) return 0.0f;
    if (abstop >= (f2u(INFINITY) >> 20)) return x + x;
    if (x > 0x1.62e42ep6f) return INFINITY;
    if (x < -0x1.9fe368p6f) return 0.0f;
  }
  const double kInvLn2N = 0x1.71547652b82fep+5, kShift = 0x1.8p+52;
  double kd = fma(kInvLn2N, xd, kShift);
  const uint64_t ki = d2u(kd);
  kd -= kShift;
  const double r = fma(kInvLn2N, xd, -kd);
  const uint64_t t = kExpTab[ki % 32] + (ki << 47);
  const double s = u2d(t);
  const double z = fma(0x1.c6af84b912394p-20, r, 0x1.ebfce50fac4f3p-13);
  const double r2 = r * r;
  double y = fma(0x1.62e42ff0c52d6p-6, r, 1.0);
  y = fma(z, r2, y);
  y = y * s;
  return (float)y;
}

float orc_sigmoid(float x) { return 1.0f / (1.0f + expf(-x)); }

/* ---- tiny static-chunk thread helper (mirrors runtime::static_chunk) ---- */
typedef void (*range_fn)(int64_t lo, int64_t hi, void* ctx);
typedef struct {
  range_fn fn;
  void* ctx;
  int64_t lo, hi;
} range_job;

static void* range_thunk(void* a) {
  range_job* j = (range_job*)a;
  if (j->lo < j->hi) j->fn(j->lo, j->hi, j->ctx);
  return NULL;
}

static void parallel_for(int64_t n, int threads, range_fn fn, void* ctx) {
  if (threads <= 1 || n < 2) {
    if (n > 0) fn(0, n, ctx);
    return;
  }
  if (threads > 256) threads = 256;
  pthread_t th[256];
  range_job jobs[256];
  const int64_t block = (n + threads - 1) / threads;
  for (int w = 0; w < threads; ++w) {
    int64_t lo = (int64_t)w * block;
    if (lo > n) lo = n;
    int64_t hi = lo + block;
    if (hi > n) hi = n;
    jobs[w] = (range_job){fn, ctx, lo, hi};
  }
  for (int w = 1; w < threads; ++w) pthread_create(&th[w], NULL, range_thunk, &jobs[w]);
  range_thunk(&jobs[0]);
  for (int w = 1; w < threads; ++w) pthread_join(th[w], NULL);
}

typedef struct {
  uint32_t lo;
  int64_t bad;
  const float* got;
  uint32_t first_bad;
} expf_job;

static void expf_port_range(int64_t lo, int64_t hi, void* c) {
  expf_job* j = (expf_job*)c;
  int64_t bad = 0;
  for (int64_t i = lo; i < hi; ++i) {
    const float x = u2f(j->lo + (uint32_t)i);
    const float want = expf(x);
    const float got = j->got ? j->got[i] : orc_expf_port(x);
    if (f2u(want) != f2u(got) && !(want != want && got != got)) {
      if (!bad) __atomic_store_n(&j->first_bad, j->lo + (uint32_t)i, __ATOMIC_RELAXED);
      ++bad;
    }
  }
  __atomic_add_fetch(&j->bad, bad, __ATOMIC_RELAXED);
}

int64_t orc_expf_port_mismatches(uint32_t lo_bits, uint32_t hi_bits, int threads) {
  expf_job j = {lo_bits, 0, NULL, 0};
  parallel_for((int64_t)hi_bits - (int64_t)lo_bits + 1, threads, expf_port_range, &j);
  return j.bad;
}

int64_t orc_expf_compare(uint32_t start_bits, int64_t count, const float* got, int threads,
                         uint32_t* first_bad_bits) {
  expf_job j = {start_bits, 0, got, 0};
  parallel_for(count, threads, expf_port_range, &j);
  if (first_bad_bits) *first_bad_bits = j.first_bad;
  return j.bad;
}

/* ------------------------------------------------------------------------ */
/* Network, fixed Zhang shapes (network.cpp:17-23).  Orders follow           */
/* SURVEY.md §8(a) "numerics contract", derived from nn.cpp / network.cpp.   */
/* ------------------------------------------------------------------------ */

/* net::forward (network.cpp:81-95) composed of mconv (nn.cpp:110-125, tap
 * order row-major, `in*k`), sigmoid (:127-129) and avgpool (:135-146). */
void orc_forward(const float* I, const float* p, float* act) {
  const float* k1 = p + ORC_K1;
  const float* b1 = p + ORC_B1;
  const float* k2 = p + ORC_K2;
  const float* b2 = p + ORC_B2;
  const float* fc = p + ORC_FC;
  const float* b = p + ORC_B;
  float* c1 = act + ORC_C1;
  float* s1 = act + ORC_S1;
  float* c2 = act + ORC_C2;
  float* s2 = act + ORC_S2;
  float* out = act + ORC_OUT;
  for (int i = 0; i < 6; ++i)
    for (int y = 0; y < 24; ++y)
      for (int x = 0; x < 24; ++x) {
        float acc = 0.0f;
        for (int ky = 0; ky < 5; ++ky)
          for (int kx = 0; kx < 5; ++kx) acc += I[(y + ky) * 28 + x + kx] * k1[i * 25 + ky * 5 + kx];
        c1[(i * 24 + y) * 24 + x] = orc_sigmoid(acc + b1[i]);
      }
  for (int c = 0; c < 6; ++c)
    for (int y = 0; y < 12; ++y)
      for (int x = 0; x < 12; ++x) {
        const float* q = c1 + (c * 24 + 2 * y) * 24 + 2 * x;
        s1[(c * 12 + y) * 12 + x] = (q[0] + q[1] + q[24] + q[25]) * 0.25f;
      }
  for (int i = 0; i < 12; ++i)
    for (int y = 0; y < 8; ++y)
      for (int x = 0; x < 8; ++x) {
        float acc = 0.0f;
        for (int c = 0; c < 6; ++c)
          for (int ky = 0; ky < 5; ++ky)
            for (int kx = 0; kx < 5; ++kx)
              acc += s1[(c * 12 + y + ky) * 12 + x + kx] * k2[((i * 6 + c) * 5 + ky) * 5 + kx];
        c2[(i * 8 + y) * 8 + x] = orc_sigmoid(acc + b2[i]);
      }
  for (int c = 0; c < 12; ++c)
    for (int y = 0; y < 4; ++y)
      for (int x = 0; x < 4; ++x) {
        const float* q = c2 + (c * 8 + 2 * y) * 8 + 2 * x;
        s2[(c * 4 + y) * 4 + x] = (q[0] + q[1] + q[8] + q[9]) * 0.25f;
      }
  for (int i = 0; i < 10; ++i) {
    float acc = 0.0f;
    for (int j = 0; j < 192; ++j) acc += s2[j] * fc[i * 192 + j];
    out[i] = orc_sigmoid(acc + b[i]);
  }
}

/* net::loss (network.cpp:97-109). */
float orc_loss(const float* yhat, const float* y) {
  float acc = 0.0f;
  for (int i = 0; i < 10; ++i) {
    const float d = y[i] - yhat[i];
    acc += d * d;
  }
  return 0.5f * acc;
}

/* net::backward (network.cpp:145-169) via mconv_layer_backward (:116-141):
 * backsigmoid (nn.cpp:131-133), backweights = conv(in, d) (:160), backbias =
 * sum_all (:162, tensor.cpp:310-314), backin clipped nested sums (:164-217),
 * backavgpool (:148-158). */
void orc_backward(const float* I, const float* act, const float* p, const float* y, float* g) {
  const float* k2 = p + ORC_K2;
  const float* fc = p + ORC_FC;
  const float* c1 = act + ORC_C1;
  const float* s1 = act + ORC_S1;
  const float* c2 = act + ORC_C2;
  const float* s2 = act + ORC_S2;
  const float* out = act + ORC_OUT;
  float dz[10], ds2[192], dz2[768], ds1[864];
  float* dz1 = (float*)malloc(sizeof(float) * 3456);

  for (int i = 0; i < 10; ++i) dz[i] = (out[i] - y[i]) * out[i] * (1.0f - out[i]);
  for (int i = 0; i < 10; ++i) {
    for (int j = 0; j < 192; ++j) g[ORC_FC + i * 192 + j] = 0.0f + s2[j] * dz[i];
    g[ORC_B + i] = 0.0f + dz[i];
  }
  for (int j = 0; j < 192; ++j) {
    float acc = 0.0f;
    for (int i = 0; i < 10; ++i) acc = acc + (0.0f + fc[i * 192 + j] * dz[i]);
    ds2[j] = acc;
  }
  for (int c = 0; c < 12; ++c)
    for (int yy = 0; yy < 8; ++yy)
      for (int x = 0; x < 8; ++x) {
        const int e = (c * 8 + yy) * 8 + x;
        const float d = ds2[(c * 4 + yy / 2) * 4 + x / 2] * 0.25f;
        dz2[e] = d * c2[e] * (1.0f - c2[e]);
      }
  for (int i = 0; i < 12; ++i) {
    for (int c = 0; c < 6; ++c)
      for (int u = 0; u < 5; ++u)
        for (int v = 0; v < 5; ++v) {
          float acc = 0.0f;
          for (int yy = 0; yy < 8; ++yy)
            for (int x = 0; x < 8; ++x)
              acc += s1[(c * 12 + u + yy) * 12 + v + x] * dz2[(i * 8 + yy) * 8 + x];
          g[ORC_K2 + ((i * 6 + c) * 5 + u) * 5 + v] = acc;
        }
    float acc = 0.0f;
    for (int e = 0; e < 64; ++e) acc += dz2[i * 64 + e];
    g[ORC_B2 + i] = acc;
  }
  for (int e = 0; e < 864; ++e) ds1[e] = 0.0f;
  for (int i = 0; i < 12; ++i)
    for (int c = 0; c < 6; ++c)
      for (int pp = 0; pp < 12; ++pp)
        for (int qq = 0; qq < 12; ++qq) {
          const int off1 = pp < 8 ? 0 : pp - 7, off2 = qq < 8 ? 0 : qq - 7;
          int cnt1 = pp + 1 < 8 ? pp + 1 : 8;
          if (5 - off1 < cnt1) cnt1 = 5 - off1;
          int cnt2 = qq + 1 < 8 ? qq + 1 : 8;
          if (5 - off2 < cnt2) cnt2 = 5 - off2;
          float outer = 0.0f;
          for (int u1 = 0; u1 < cnt1; ++u1) {
            float row = 0.0f;
            for (int u2 = 0; u2 < cnt2; ++u2)
              row += k2[((i * 6 + c) * 5 + off1 + u1) * 5 + off2 + u2] *
                     dz2[(i * 8 + pp - off1 - u1) * 8 + qq - off2 - u2];
            outer += row;
          }
          const int e = (c * 12 + pp) * 12 + qq;
          ds1[e] = ds1[e] + (0.0f + outer);
        }
  for (int c = 0; c < 6; ++c)
    for (int yy = 0; yy < 24; ++yy)
      for (int x = 0; x < 24; ++x) {
        const int e = (c * 24 + yy) * 24 + x;
        const float d = ds1[(c * 12 + yy / 2) * 12 + x / 2] * 0.25f;
        dz1[e] = d * c1[e] * (1.0f - c1[e]);
      }
  for (int i = 0; i < 6; ++i) {
    for (int u = 0; u < 5; ++u)
      for (int v = 0; v < 5; ++v) {
        float acc = 0.0f;
        for (int yy = 0; yy < 24; ++yy)
          for (int x = 0; x < 24; ++x) acc += I[(u + yy) * 28 + v + x] * dz1[(i * 24 + yy) * 24 + x];
        g[ORC_K1 + (i * 5 + u) * 5 + v] = acc;
      }
    float acc = 0.0f;
    for (int e = 0; e < 576; ++e) acc += dz1[i * 576 + e];
    g[ORC_B1 + i] = acc;
  }
  free(dz1);
}

void orc_example_cell(const float* image, const float* params, int32_t label, float* cell) {
  float act[ORC_NACT], y[10] = {0};
  y[label] = 1.0f; /* mnist::one_hot (mnist.cpp:161-167) */
  orc_forward(image, params, act);
  orc_backward(image, act, params, y, cell);
  cell[ORC_NPARAM] = orc_loss(act + ORC_OUT, y);
}

typedef struct {
  const float* images;
  const int32_t* labels;
  const float* params;
  int64_t start;
  float* cells;
} cell_job;

static void cells_range(int64_t lo, int64_t hi, void* c) {
  cell_job* j = (cell_job*)c;
  for (int64_t i = lo; i < hi; ++i)
    orc_example_cell(j->images + (j->start + i) * 784, j->params, j->labels[j->start + i],
                     j->cells + i * (ORC_NPARAM + 1));
}

void orc_train_group(const float* images, const int32_t* labels, int64_t start, int64_t m,
                     float* params, float rate, double* loss_sum, int threads) {
  float* cells = (float*)malloc(sizeof(float) * (size_t)m * (ORC_NPARAM + 1));
  cell_job j = {images, labels, params, start, cells};
  parallel_for(m, threads, cells_range, &j);
  float acc[ORC_NPARAM];
  for (int k = 0; k < ORC_NPARAM; ++k) acc[k] = 0.0f;
  for (int64_t i = 0; i < m; ++i) { /* network.cpp:238-243 */
    const float* row = cells + i * (ORC_NPARAM + 1);
    for (int k = 0; k < ORC_NPARAM; ++k) acc[k] += row[k];
    *loss_sum += row[ORC_NPARAM];
  }
  for (int k = 0; k < ORC_NPARAM; ++k) /* sgd_step (network.cpp:171-180) */
    params[k] = params[k] - rate * (acc[k] / (float)m);
  free(cells);
}

int orc_train(const float* images, const int32_t* labels, int64_t n, float* params, float rate,
              int epochs, int64_t batch, double* epoch_loss, int threads) {
  if (n == 0) return -1;
  if (epochs < 0) return -2;
  if (!(rate > 0.0f)) return -3;
  if (batch < 1) return -4;
  for (int e = 0; e < epochs; ++e) {
    double loss_sum = 0.0;
    for (int64_t s = 0; s < n; s += batch) {
      const int64_t m = (s + batch < n ? s + batch : n) - s;
      orc_train_group(images, labels, s, m, params, rate, &loss_sum, threads);
    }
    epoch_loss[e] = loss_sum / (double)n;
  }
  return 0;
}

int orc_predict(const float* yhat) { /* network.cpp:253-261 */
  int best = 0;
  for (int i = 1; i < 10; ++i)
    if (yhat[i] > yhat[best]) best = i;
  return best;
}

typedef struct {
  const float* params;
  const float* images;
  int32_t* pred;
} eval_job;

static void eval_range(int64_t lo, int64_t hi, void* c) {
  eval_job* j = (eval_job*)c;
  float act[ORC_NACT];
  for (int64_t i = lo; i < hi; ++i) {
    orc_forward(j->images + i * 784, j->params, act);
    j->pred[i] = orc_predict(act + ORC_OUT);
  }
}

int64_t orc_evaluate(const float* params, const float* images, const int32_t* labels, int64_t n,
                     int32_t* pred, int threads) {
  eval_job j = {params, images, pred};
  parallel_for(n, threads, eval_range, &j);
  int64_t correct = 0;
  for (int64_t i = 0; i < n; ++i) correct += pred[i] == labels[i];
  return correct;
}

/* ------------------------------------------------------------------------ */
/* Generic rank-polymorphic ops (nn.cpp:37-217), row-major, rank <= 8.       */
/* ------------------------------------------------------------------------ */
static int64_t count_of(const int64_t* s, int r) {
  int64_t c = 1;
  for (int a = 0; a < r; ++a) c *= s[a];
  return c;
}

static void strides_of(const int64_t* s, int r, int64_t* st) {
  int64_t acc = 1;
  for (int a = r - 1; a >= 0; --a) {
    st[a] = acc;
    acc *= s[a];
  }
}

static void unflat(const int64_t* s, int r, int64_t flat, int64_t* iv) {
  for (int a = r - 1; a >= 0; --a) {
    iv[a] = s[a] > 0 ? flat % s[a] : 0;
    if (s[a] > 0) flat /= s[a];
  }
}

/* conv (nn.cpp:96-108): out[iv] = sum over row-major taps ov of in[iv+ov]*k[ov]. */
void orc_conv(const float* in, const int64_t* is, int r, const float* k, const int64_t* ks,
              float* out) {
  int64_t os[8], ist[8], iv[8], ov[8];
  for (int a = 0; a < r; ++a) os[a] = is[a] - ks[a] + 1;
  strides_of(is, r, ist);
  const int64_t n = count_of(os, r), nk = count_of(ks, r);
  for (int64_t o = 0; o < n; ++o) {
    unflat(os, r, o, iv);
    float acc = 0.0f;
    for (int64_t t = 0; t < nk; ++t) {
      unflat(ks, r, t, ov);
      int64_t off = 0;
      for (int a = 0; a < r; ++a) off += (iv[a] + ov[a]) * ist[a];
      acc += in[off] * k[t];
    }
    out[o] = acc;
  }
}

/* mconv (nn.cpp:110-125): slice i = conv(in, k[i]) + b[i]. */
void orc_mconv(const float* in, const int64_t* is, int r, const float* k, const int64_t* ks,
               const float* b, float* out) {
  const int64_t nk = ks[0], slice = count_of(ks + 1, r);
  int64_t os[8];
  for (int a = 0; a < r; ++a) os[a] = is[a] - ks[a + 1] + 1;
  const int64_t per = count_of(os, r);
  for (int64_t i = 0; i < nk; ++i) {
    orc_conv(in, is, r, k + i * slice, ks + 1, out + i * per);
    for (int64_t o = 0; o < per; ++o) out[i * per + o] = out[i * per + o] + b[i];
  }
}

/* avgpool (nn.cpp:135-146). */
void orc_avgpool(const float* in, const int64_t* s, int r, float* out) {
  int64_t os[8], st[8] = {0}, iv[8];
  for (int a = 0; a < r; ++a) os[a] = a >= r - 2 ? s[a] / 2 : s[a];
  strides_of(s, r, st);
  const int64_t n = count_of(os, r), row = st[r - 2];
  for (int64_t o = 0; o < n; ++o) {
    unflat(os, r, o, iv);
    int64_t base = 0;
    for (int a = 0; a < r; ++a) base += iv[a] * st[a] * (a >= r - 2 ? 2 : 1);
    out[o] = (in[base] + in[base + 1] + in[base + row] + in[base + row + 1]) * 0.25f;
  }
}

/* backavgpool (nn.cpp:148-158); `s` is the shape of d. */
void orc_backavgpool(const float* d, const int64_t* s, int r, float* out) {
  int64_t os[8], st[8], iv[8];
  for (int a = 0; a < r; ++a) os[a] = a >= r - 2 ? s[a] * 2 : s[a];
  strides_of(s, r, st);
  const int64_t n = count_of(os, r);
  for (int64_t o = 0; o < n; ++o) {
    unflat(os, r, o, iv);
    int64_t base = 0;
    for (int a = 0; a < r; ++a) base += (a >= r - 2 ? iv[a] / 2 : iv[a]) * st[a];
    out[o] = d[base] * 0.25f;
  }
}

typedef struct {
  const float* d;
  const float* k;
  int64_t dst[8], kst[8], cnt[8];
  int r;
} box_t;

static float box_sum(const box_t* b, int axis, int64_t doff, int64_t koff) { /* nn.cpp:169-189 */
  float acc = 0.0f;
  if (axis == b->r - 1) {
    for (int64_t u = 0; u < b->cnt[axis]; ++u) acc += b->k[koff + u] * b->d[doff - u];
    return acc;
  }
  for (int64_t u = 0; u < b->cnt[axis]; ++u)
    acc += box_sum(b, axis + 1, doff - u * b->dst[axis], koff + u * b->kst[axis]);
  return acc;
}

/* backin (nn.cpp:193-217): clipped correlation, nested per-axis sums. */
void orc_backin(const float* d, const int64_t* ds, const float* k, const int64_t* ks, int r,
                float* out) {
  if (r == 0) {
    out[0] = d[0] * k[0];
    return;
  }
  box_t b;
  b.d = d;
  b.k = k;
  b.r = r;
  int64_t os[8], iv[8];
  for (int a = 0; a < r; ++a) os[a] = ds[a] + ks[a] - 1;
  strides_of(ds, r, b.dst);
  strides_of(ks, r, b.kst);
  const int64_t n = count_of(os, r);
  for (int64_t o = 0; o < n; ++o) {
    unflat(os, r, o, iv);
    int64_t dbase = 0, kbase = 0;
    for (int a = 0; a < r; ++a) {
      const int64_t i = iv[a];
      const int64_t off = i < ds[a] ? 0 : i - ds[a] + 1;
      int64_t c = ds[a] < i + 1 ? ds[a] : i + 1;
      if (ks[a] - off < c) c = ks[a] - off;
      b.cnt[a] = c;
      dbase += (i - off) * b.dst[a];
      kbase += off * b.kst[a];
    }
    out[o] = box_sum(&b, 0, dbase, kbase);
  }
}

float orc_sum_all(const float* x, int64_t n) {
  float acc = 0.0f;
  for (int64_t i = 0; i < n; ++i) acc += x[i];
  return acc;
}
