// host_data.cpp -- host-side pieces of the reference API that are not per-step device work:
// net::init_params (network.cpp:56-79), the synthetic digit corpus (synth.cpp:117-161) and the
// mnist::make_set invariants (mnist.cpp:126-154).  They produce the exact bytes the reference
// produces (tests/test_oracle.py / tests/test_capi.py pin them against the golden hashes), so the
// GPU path trains on identical inputs and initial weights.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

#include "tlb_capi_internal.h"
#include "tloom_b200.h"

namespace {

// 5x7 font, one bitmask per row (bit 4 = leftmost column): the glyph table of synth.cpp:14-94.
constexpr uint8_t kFont[10][7] = {
    {0x0E, 0x11, 0x13, 0x15, 0x19, 0x11, 0x0E}, {0x04, 0x0C, 0x04, 0x04, 0x04, 0x04, 0x0E},
    {0x0E, 0x11, 0x01, 0x02, 0x04, 0x08, 0x1F}, {0x0E, 0x11, 0x01, 0x06, 0x01, 0x11, 0x0E},
    {0x02, 0x06, 0x0A, 0x12, 0x1F, 0x02, 0x02}, {0x1F, 0x10, 0x1E, 0x01, 0x01, 0x11, 0x0E},
    {0x06, 0x08, 0x10, 0x1E, 0x11, 0x11, 0x0E}, {0x1F, 0x01, 0x02, 0x02, 0x04, 0x04, 0x04},
    {0x0E, 0x11, 0x11, 0x0E, 0x11, 0x11, 0x0E}, {0x0E, 0x11, 0x11, 0x0F, 0x01, 0x02, 0x0C},
};

double font_cell(int digit, int gy, int gx) {
  if (gx < 0 || gx > 4 || gy < 0 || gy > 6) return 0.0;
  return (kFont[digit][gy] >> (4 - gx)) & 1u ? 1.0 : 0.0;
}

// Bilinear sample, zero outside the glyph (synth.cpp:102-113); term order kept for bit parity.
double font_sample(int digit, double gx, double gy) {
  const double fx = std::floor(gx), fy = std::floor(gy);
  const int ix = static_cast<int>(fx), iy = static_cast<int>(fy);
  const double wx = gx - fx, wy = gy - fy;
  return font_cell(digit, iy, ix) * (1 - wx) * (1 - wy) + font_cell(digit, iy, ix + 1) * wx * (1 - wy) +
         font_cell(digit, iy + 1, ix) * (1 - wx) * wy + font_cell(digit, iy + 1, ix + 1) * wx * wy;
}

}  // namespace

extern "C" int tlb_init_params(uint64_t seed, float* p) {
  if (!p) return tlb::fail(TLB_ERR_ARG, "tlb_init_params: null output");
  std::mt19937_64 rng(seed);
  std::fill(p, p + TLB_NPARAM, 0.0f);
  struct Fill {
    int off, count, fan_in, fan_out;
  };
  // k1 [6,5,5] fan (25, 576); k2 [12,6,5,5] fan (150, 64); fc [10,12,1,4,4] fan (192, 1).
  const Fill fills[3] = {{0, 150, 25, 576}, {156, 1800, 150, 64}, {1968, 1920, 192, 1}};
  for (const Fill& f : fills) {
    const float limit = std::sqrt(6.0f / static_cast<float>(f.fan_in + f.fan_out));
    for (int i = 0; i < f.count; ++i) {
      const float u = static_cast<float>(rng() >> 40) * 0x1p-24f;
      p[f.off + i] = (u * 2.0f - 1.0f) * limit;
    }
  }
  return TLB_OK;
}

extern "C" int tlb_synth_make_digits(int64_t n, uint64_t seed, uint8_t* pixels, int32_t* labels) {
  if (n < 0) return tlb::fail(TLB_ERR_ERROR, "make_digits: negative count");
  if (n > 0 && (!pixels || !labels)) return tlb::fail(TLB_ERR_ARG, "tlb_synth_make_digits: null output");
  std::mt19937_64 rng(seed);
  auto u01 = [&rng] { return static_cast<double>(rng() >> 40) * 0x1p-24; };
  for (int64_t img = 0; img < n; ++img) {
    const int digit = static_cast<int>(img % 10);
    const double sx = 3.3 + (3.7 - 3.3) * u01();
    const double sy = 3.3 + (3.7 - 3.3) * u01();
    const double tx = -0.8 + (0.8 - -0.8) * u01();
    const double ty = -0.8 + (0.8 - -0.8) * u01();
    labels[img] = digit;
    uint8_t* out = pixels + img * 784;
    for (int y = 0; y < 28; ++y) {
      for (int x = 0; x < 28; ++x) {
        const double gx = (x - 13.5 - tx) / sx + 2.0;
        const double gy = (y - 13.5 - ty) / sy + 3.0;
        double v = font_sample(digit, gx, gy) + 0.02 * u01();
        v = std::min(std::max(v, 0.0), 1.0);
        out[y * 28 + x] = static_cast<uint8_t>(std::lround(v * 255.0));
      }
    }
  }
  return TLB_OK;
}

extern "C" int tlb_synth_make_set(int64_t n, uint64_t seed, float* images, int32_t* labels) {
  if (n < 0) return tlb::fail(TLB_ERR_ERROR, "make_digits: negative count");
  std::string px(static_cast<size_t>(n) * 784, '\0');
  const int rc = tlb_synth_make_digits(n, seed, reinterpret_cast<uint8_t*>(px.data()), labels);
  if (rc) return rc;
  for (int64_t i = 0; i < n * 784; ++i)
    images[i] = static_cast<float>(static_cast<uint8_t>(px[static_cast<size_t>(i)])) / 255.0f;
  return TLB_OK;
}

extern "C" int tlb_validate_set(const float* images, const int32_t* labels, int64_t n) {
  if (n < 0) return tlb::fail(TLB_ERR_ARG, "tlb_validate_set: negative count");
  for (int64_t i = 0; i < n * 784; ++i) {
    if (!(images[i] >= 0.0f && images[i] <= 1.0f))
      return tlb::fail(TLB_ERR_VALUE, "dataset: pixel " + std::to_string(images[i]) + " at flat index " +
                                          std::to_string(i) + " out of range [0,1]");
  }
  for (int64_t i = 0; i < n; ++i) {
    if (labels[i] < 0 || labels[i] > 9)
      return tlb::fail(TLB_ERR_VALUE, "dataset: label " + std::to_string(labels[i]) + " at index " +
                                          std::to_string(i) + " out of range 0..9");
  }
  return TLB_OK;
}

// ---- widened CNN (BASELINE configs[4]) host data ------------------------------------------------------
// init_params (network.cpp:56-79) with the widened shapes: k1 [32,5,5] fan (25, 60*60), k2 [64,32,5,5]
// fan (32*25, 26*26), fc [10,64,1,13,13] fan (64*13*13, 1); fill order k1, k2, fc from one mt19937_64
// stream; biases zero.  Offsets follow write_flat order (k1, b1, k2, b2, fc, b).
extern "C" int tlb_wide_init_params(uint64_t seed, float* p) {
  if (!p) return tlb::fail(TLB_ERR_ARG, "tlb_wide_init_params: null output");
  std::mt19937_64 rng(seed);
  std::fill(p, p + TLB_WIDE_NPARAM, 0.0f);
  struct Fill {
    int off, count, fan_in, fan_out;
  };
  const Fill fills[3] = {{0, 800, 25, 3600}, {832, 51200, 800, 676}, {52096, 108160, 10816, 1}};
  for (const Fill& f : fills) {
    const float limit = std::sqrt(6.0f / static_cast<float>(f.fan_in + f.fan_out));
    for (int i = 0; i < f.count; ++i) {
      const float u = static_cast<float>(rng() >> 40) * 0x1p-24f;
      p[f.off + i] = (u * 2.0f - 1.0f) * limit;
    }
  }
  return TLB_OK;
}

extern "C" int tlb_wide_make_set(int64_t n, uint64_t seed, float* images, int32_t* labels) {
  if (n < 0) return tlb::fail(TLB_ERR_ERROR, "make_digits: negative count");
  if (n > 0 && (!images || !labels)) return tlb::fail(TLB_ERR_ARG, "tlb_wide_make_set: null output");
  std::vector<uint8_t> px((size_t)n * 784);
  std::vector<int32_t> lab((size_t)n);
  const int rc = tlb_synth_make_digits(n, seed, px.data(), lab.data());
  if (rc != TLB_OK) return rc;
  std::fill(images, images + (size_t)n * TLB_WIDE_IMG, 0.0f);
  for (int64_t i = 0; i < n; ++i) {
    labels[i] = lab[(size_t)i];
    for (int y = 0; y < 28; ++y)
      for (int x = 0; x < 28; ++x)
        images[(size_t)i * TLB_WIDE_IMG + (y + 18) * 64 + x + 18] = static_cast<float>(px[(size_t)i * 784 + y * 28 + x]) / 255.0f;
  }
  return TLB_OK;
}
