// batch_train.cu -- fast-mode persistent train kernel for large SGD groups (BASELINE configs[3]: batch
// 1k .. 256k per GPU; net::train, proj/src/network.cpp:209-251).
//
// The one-image-per-CTA kernels (zhang_kernels.cu) keep one image's activations resident and run every
// stage on that image: at batch >= 1k each stage's barrier is paid per image and every weight-gradient
// output is read-modified-written in shared memory per image.  Here a CTA trains NI images per ROUND:
//   * every stage's lanes span the NI images (one barrier per stage per round, not per image);
//   * the weight-gradient lanes own their outputs and loop over the round's images in registers, so the
//     CTA's gradient accumulator G (shared memory) is updated once per round per output;
//   * the NI images of a round are contiguous in HBM and arrive with ONE TMA bulk copy into a
//     double-buffered ring (the next round -- possibly the next step's first -- is in flight meanwhile).
// Per step (one SGD group): each CTA trains its rounds of the group (a contiguous chunk, or interleaved
// rounds while a host call's chunks are in flight; SM-pair shares with two CTAs per SM: seek_round), writes
// its partial gradient row, grid barrier, CTA b reduces parameters static_chunk(3898, grid, b) over the
// partial rows in CTA order (fixed tree: deterministic run to run) and applies sgd_step
// (network.cpp:171-180) or, in DP shard mode, writes the shard's gradient sum; grid barrier.
//
// Stages of a round (cnt <= NI images; lane counts per image):
//   S1 conv1+sigmoid+pool, and g1 = c1(1-c1)                         144 lanes x 600 FFMA
//   S2 conv2+sigmoid+pool, and g2 = c2(1-c2) into padded dz2 rows     192 lanes x 600 FFMA (row x channel half)
//   S3 FC+sigmoid, dz = ((o-y)o)(1-o)                                  80 lanes (8 per class)
//   S4 d_s2 = fc^T dz, dz2 = (d_s2/4) g2                               192 lanes
//   S5 backin (36 row pairs x 4 kernel-group lanes, valid taps only: 720-840 FFMA each), whose epilogue
//      writes dz1 = (d_s1/4) g1 in place of g1; g_k2 + g_b2 (720 + 24 lanes over the round's images,
//      320 FFMA per image); g_fc (480 lanes, 4 columns each) + g_b (10 lanes)
//   S6 g_k1 (30 outputs x 8 row-chunk lanes over the round's images), g_b1
// Arithmetic is the fast mode's (FFMA, ex2/rcp MUFU logistic; fixed summation trees), within the
// north-star 1e-4 tolerance; EXACT mode never runs here.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "tlb_common.cuh"
#include "tlb_launch.h"
#include "train_common.cuh"

#ifndef TLB_GK2_FULL
#define TLB_GK2_FULL 1  // batched g_k2: one lane per output row over all 8 tap rows (0: two row-half lanes)
#endif

namespace tlb {
namespace bt {

// Padded weight copies (built per step from P): conv1 rows [6][5][8] in 44-float channel slots, conv2 rows
// [12][6][5][8] in 244-float kernel slots: every 5-tap row is an aligned float4 + a scalar, and the
// distinct channels / kernels a warp touches fall in distinct bank groups (11 and 61 float4s, odd mod 8).
constexpr int kW1Stride = 44, kW1Floats = 6 * kW1Stride;
constexpr int kW2Stride = 244, kW2Floats = 12 * kW2Stride;
// Per-image region: g1 (c1(1-c1), then dz1 in place) [6][24][24] in 580-float planes | s1 [6][12][12] |
// dz2 zero-padded by 4 rows top and bottom [12][16][8] in 132-float kernel slots (g2 = c2(1-c2) first) |
// s2 [192] | out [10] at 0, dz [10] at 16.
constexpr int kG1Plane = 580, kG1Floats = 6 * kG1Plane;
constexpr int kD2K = 132, kD2Floats = 12 * kD2K;
constexpr int kOffS1 = kG1Floats, kOffD2 = kOffS1 + 864, kOffS2 = kOffD2 + kD2Floats, kOffOd = kOffS2 + 192;
constexpr int kImgRegion = kOffOd + 32;
static_assert(kOffS1 % 4 == 0 && kOffD2 % 4 == 0 && kOffS2 % 4 == 0 && kImgRegion % 4 == 0, "float4 regions");

template <int NI>
struct Layout {
  static constexpr int kP = 0;
  static constexpr int kW1 = kP + kPStride;
  static constexpr int kW2 = kW1 + kW1Floats;
  static constexpr int kG = kW2 + kW2Floats;
  static constexpr int kRing = kG + kPStride;          // [2][NI][784] TMA ring
  static constexpr int kLab = kRing + 2 * NI * kImg;   // [2][NI] labels (ints)
  static constexpr int kImgs = kLab + 16;
  static constexpr int kFloats = kImgs + NI * kImgRegion;
  // + 2 mbarriers, 2 int64 round indices and the [2][NI][784] pixel-byte ring (byte ingestion)
  static constexpr size_t kBytes = (size_t)kFloats * sizeof(float) + 2 * sizeof(uint64_t) + 2 * sizeof(int64_t) +
                                   2 * NI * kImg + 4 * sizeof(int);
  static_assert(kRing % 4 == 0 && kImgs % 4 == 0, "16-byte aligned regions");
  static_assert(2 * NI <= 16, "label slots");
};

extern __shared__ __align__(128) float bt_smem[];

#ifndef TLB_PAIR_SHARE_DEFAULT
#define TLB_PAIR_SHARE_DEFAULT 0.54f
#endif
constexpr float kPairShare = TLB_PAIR_SHARE_DEFAULT;

// logistic(acc + b) with nb = -b log2(e): one FFMA, ex2.approx.ftz, add, rcp.approx.ftz (fast mode).
__device__ __forceinline__ float logistic(float acc, float nb) {
  constexpr float kNegLog2e = -1.4426950408889634f;
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(__fmaf_rn(acc, kNegLog2e, nb)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return r;
}
__device__ __forceinline__ float neg_log2e_times(float b) { return b * -1.4426950408889634f; }

__device__ __forceinline__ void load5(const float* wrow, float (&w)[5]) {
  const float4 a = *reinterpret_cast<const float4*>(wrow);
  w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
  w[4] = wrow[4];
}
template <int N>
__device__ __forceinline__ void load_row(const float* src, float (&v)[N]) {
  static_assert(N % 4 == 0, "float4 rows");
#pragma unroll
  for (int q = 0; q < N / 4; ++q) {
    const float4 x = reinterpret_cast<const float4*>(src)[q];
    v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
  }
}

// S1: lane (image k, pooled row py, 12-column half xs, channel i), channel fastest: conv rows 2py, 2py+1
// x 12 columns over the 25 taps (nn.cpp:28-33 order per output), sigmoid, g1 = c1(1-c1), 2x2 pool.
__device__ __forceinline__ void conv1_item(const float* P, const float* W1, const float* imgs, float* regs, int it) {
  const int k = it / 144, r = it - k * 144;
  const int pos = r / 6, i = r - pos * 6, py = pos >> 1, xs = pos & 1;
  const int y0 = 2 * py, x0 = 12 * xs;
  const float* img = imgs + k * kImg;
  const float* w = W1 + i * kW1Stride;
  float a[2][12];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int o = 0; o < 12; ++o) a[q][o] = 0.0f;
#pragma unroll
  for (int rr = 0; rr < 6; ++rr) {  // image row y0 + rr feeds conv row q with ky = rr - q
    float in[16];
    load_row<16>(img + (y0 + rr) * 28 + x0, in);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int ky = rr - q;
      if (ky < 0 || ky > 4) continue;
      float wv[5];
      load5(w + ky * 8, wv);
#pragma unroll
      for (int kx = 0; kx < 5; ++kx)
#pragma unroll
        for (int o = 0; o < 12; ++o) a[q][o] = __fmaf_rn(in[o + kx], wv[kx], a[q][o]);
    }
  }
  const float nb = neg_log2e_times(P[kB1 + i]);
  float* reg = regs + k * kImgRegion;
  float* g1 = reg + i * kG1Plane + y0 * 24 + x0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int o = 0; o < 12; ++o) a[q][o] = logistic(a[q][o], nb);
#pragma unroll
    for (int o4 = 0; o4 < 3; ++o4) {
      float4 g;
      g.x = a[q][4 * o4] * (1.0f - a[q][4 * o4]);
      g.y = a[q][4 * o4 + 1] * (1.0f - a[q][4 * o4 + 1]);
      g.z = a[q][4 * o4 + 2] * (1.0f - a[q][4 * o4 + 2]);
      g.w = a[q][4 * o4 + 3] * (1.0f - a[q][4 * o4 + 3]);
      *reinterpret_cast<float4*>(g1 + q * 24 + 4 * o4) = g;
    }
  }
  float* s1 = reg + kOffS1 + (i * 12 + py) * 12 + 6 * xs;
#pragma unroll
  for (int px = 0; px < 6; px += 2) {  // avgpool (nn.cpp:144): ((p00 + p01) + p10) + p11, then * 0.25f
    float pv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = 2 * (px + h);
      pv[h] = (((a[0][c] + a[0][c + 1]) + a[1][c]) + a[1][c + 1]) * 0.25f;
    }
    *reinterpret_cast<float2*>(s1 + px) = make_float2(pv[0], pv[1]);
  }
}

// S2: lane (image k, pooled row py, kernel i, conv row r of the pooling window, channel half ch), ch fastest:
// the partial sum of conv row y = 2py + r (8 columns) over channels 3ch..3ch+2 (the 150 taps in
// (c, ky, kx) order within each half), joined by a shuffle; lane ch then owns columns 4ch..4ch+3: sigmoid,
// g2 into the padded dz2 row, and -- with the partner row from lane ^ 2 -- the 2x2 pool.
__device__ __forceinline__ void conv2_item(const float* P, const float* W2, float* regs, int it) {
  const int ch = it & 1, r = (it >> 1) & 1, rest = it >> 2;
  const int i = rest % 12, kp = rest / 12, py = kp & 3, k = kp >> 2;
  const int y = 2 * py + r;
  float* reg = regs + k * kImgRegion;
  const float* s1 = reg + kOffS1;
  float acc[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) acc[o] = 0.0f;
#pragma unroll 1
  for (int c = 3 * ch; c < 3 * ch + 3; ++c) {
    const float* wc = W2 + i * kW2Stride + c * 40;
    const float* srow = s1 + (c * 12 + y) * 12;
#pragma unroll
    for (int ky = 0; ky < 5; ++ky) {
      float in[12], wv[5];
      load_row<12>(srow + ky * 12, in);
      load5(wc + ky * 8, wv);
#pragma unroll
      for (int kx = 0; kx < 5; ++kx)
#pragma unroll
        for (int o = 0; o < 8; ++o) acc[o] = __fmaf_rn(in[o + kx], wv[kx], acc[o]);
    }
  }
#pragma unroll
  for (int o = 0; o < 8; ++o) acc[o] += __shfl_xor_sync(0xffffffffu, acc[o], 1);
  const float nb = neg_log2e_times(P[kB2 + i]);
  float t[4], u[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) t[j] = logistic(ch ? acc[4 + j] : acc[j], nb);
  *reinterpret_cast<float4*>(reg + kOffD2 + i * kD2K + (4 + y) * 8 + 4 * ch) =
      make_float4(t[0] * (1.0f - t[0]), t[1] * (1.0f - t[1]), t[2] * (1.0f - t[2]), t[3] * (1.0f - t[3]));
#pragma unroll
  for (int j = 0; j < 4; ++j) u[j] = __shfl_xor_sync(0xffffffffu, t[j], 2);  // conv row y ^ 1
  if (r == 0)  // avgpool (nn.cpp:144): ((p00 + p01) + p10) + p11, then * 0.25f
    *reinterpret_cast<float2*>(reg + kOffS2 + (i * 4 + py) * 4 + 2 * ch) =
        make_float2((((t[0] + t[1]) + u[0]) + u[1]) * 0.25f, (((t[2] + t[3]) + u[2]) + u[3]) * 0.25f);
}

// S3: eight lanes per (image, class): 24-term partials of the 192-tap FC dot, a 3-level xor tree, sigmoid;
// dz = ((o - y) o)(1 - o) with y = one_hot(label) (network.cpp:146-152).  Whole warps (see fc_item in
// infer_kernels.cu); lanes past the last task recompute task 0 and store nothing.
__device__ __forceinline__ void fc_item(const float* P, float* regs, const int* lab, int it, bool valid) {
  const int task = valid ? it >> 3 : 0, part = it & 7, k = task / 10, i = task - k * 10;
  float* reg = regs + k * kImgRegion;
  const float4* s2 = reinterpret_cast<const float4*>(reg + kOffS2 + 24 * part);
  const float4* w = reinterpret_cast<const float4*>(P + kFC + i * 192 + 24 * part);
  float acc = 0.0f;
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const float4 x = s2[q], y = w[q];
    acc = __fmaf_rn(x.x, y.x, acc);
    acc = __fmaf_rn(x.y, y.y, acc);
    acc = __fmaf_rn(x.z, y.z, acc);
    acc = __fmaf_rn(x.w, y.w, acc);
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  if (valid && part == 0) {
    const float o = logistic(acc, neg_log2e_times(P[kB + i]));
    const float y = i == lab[k] ? 1.0f : 0.0f;
    reg[kOffOd + i] = o;
    reg[kOffOd + 16 + i] = ((o - y) * o) * (1.0f - o);
  }
}

// S5 backin lane (4 lanes per task, kernels 3ig..3ig+2 each, joined by shuffles): the d_s1 rows pA = pp and
// pB = pp + 6 of channel c (pp < 6) -- 12 columns each -- over exactly the valid kernel rows of the reference's
// BackinBox (nn.cpp:169-189): u <= pA for row pA, u >= pB - 7 for row pB (6-7 rows per lane for every pp;
// the column bounds are compile-time).  Tasks run pp-major, so a warp holds at most two pp values.  Epilogue:
// dz1 = (d_s1 * 0.25) g1 for conv1 rows 2p, 2p+1 of both rows, columns 6ig..6ig+5 (in place of g1).
template <bool WP>  // WP: weight rows read from P (5 floats per row) instead of the padded W2 copy (8)
__device__ __forceinline__ void backin_acc(const float* d2i, const float* wrow, int p, int u0, int u1, float (&acc)[12]) {
#pragma unroll 1
  for (int u = u0; u <= u1; ++u) {
    float d[8], w[5];
    load_row<8>(d2i + (4 + p - u) * 8, d);
    if constexpr (WP) {
#pragma unroll
      for (int v = 0; v < 5; ++v) w[v] = wrow[u * 5 + v];
    } else {
      load5(wrow + u * 8, w);
    }
#pragma unroll
    for (int q = 0; q < 12; ++q)
#pragma unroll
      for (int v = 0; v < 5; ++v)
        if (q - v >= 0 && q - v < 8) acc[q] = __fmaf_rn(w[v], d[q - v], acc[q]);
  }
}

__device__ __forceinline__ void backin_dz1(float* g1c, int p, int ig, const float (&acc)[12]) {
  float ds[3];
#pragma unroll
  for (int h = 0; h < 3; ++h)
    ds[h] = 0.25f * (ig == 0 ? acc[h] : ig == 1 ? acc[3 + h] : ig == 2 ? acc[6 + h] : acc[9 + h]);
  float* g1 = g1c + (2 * p) * 24 + 6 * ig;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
#pragma unroll
    for (int h = 0; h < 3; ++h) {
      float2* q2 = reinterpret_cast<float2*>(g1 + a * 24 + 2 * h);
      const float2 g = *q2;
      *q2 = make_float2(ds[h] * g.x, ds[h] * g.y);
    }
  }
}

template <bool WP = false>  // WP: W2 is P (unpadded k2), see backin_acc
__device__ __forceinline__ void backin_item(const float* W2, float* regs, int bi, int cnt, bool valid) {
  const int ig = bi & 3, task = valid ? bi >> 2 : 0;
  const int c = task % 6, kp = task / 6, k = kp % cnt, pp = kp / cnt;
  float* reg = regs + k * kImgRegion;
  float accA[12], accB[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) accA[q] = accB[q] = 0.0f;
  const int pA = pp, pB = pp + 6;
#pragma unroll 1
  for (int ii = 0; ii < 3; ++ii) {
    const int i = 3 * ig + ii;
    const float* wrow = WP ? W2 + kK2 + (i * 6 + c) * 25 : W2 + i * kW2Stride + c * 40;
    const float* d2i = reg + kOffD2 + i * kD2K;
    if constexpr (WP) {  // each weight row loaded once for both d_s1 rows (valid u: A <= pA, B >= pB - 7)
#pragma unroll 1
      for (int u = 0; u < 5; ++u) {
        float w[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) w[v] = wrow[u * 5 + v];
        if (u <= pA) {
          float d[8];
          load_row<8>(d2i + (4 + pA - u) * 8, d);
#pragma unroll
          for (int q = 0; q < 12; ++q)
#pragma unroll
            for (int v = 0; v < 5; ++v)
              if (q - v >= 0 && q - v < 8) accA[q] = __fmaf_rn(w[v], d[q - v], accA[q]);
        }
        if (u >= pB - 7) {
          float d[8];
          load_row<8>(d2i + (4 + pB - u) * 8, d);
#pragma unroll
          for (int q = 0; q < 12; ++q)
#pragma unroll
            for (int v = 0; v < 5; ++v)
              if (q - v >= 0 && q - v < 8) accB[q] = __fmaf_rn(w[v], d[q - v], accB[q]);
        }
      }
    } else {
      backin_acc<WP>(d2i, wrow, pA, 0, min(4, pA), accA);
      backin_acc<WP>(d2i, wrow, pB, max(0, pB - 7), 4, accB);
    }
  }
#pragma unroll
  for (int q = 0; q < 12; ++q) {
    accA[q] += __shfl_xor_sync(0xffffffffu, accA[q], 1);
    accB[q] += __shfl_xor_sync(0xffffffffu, accB[q], 1);
    accA[q] += __shfl_xor_sync(0xffffffffu, accA[q], 2);
    accB[q] += __shfl_xor_sync(0xffffffffu, accB[q], 2);
  }
  if (!valid) return;
  float* g1c = reg + c * kG1Plane;
  backin_dz1(g1c, pA, ig, accA);
  backin_dz1(g1c, pB, ig, accB);
}

// S5 weight-gradient lane of conv2 (or of its bias): G[k2(i,c,u,0..4)] += sum over the round's images, rows
// y in half yh (4 rows), x < 8 of s1[c][u+y][v+x] * dz2[i][y][x] (nn.cpp:96-108 via backweights); the two
// row halves join by a shuffle.  Items 720..743: g_b2 (kernel i, half yh).  Kernel i varies fastest after yh:
// the lanes of a (c, u) read the same s1 rows (broadcast).
__device__ __forceinline__ void gk2_item(float* G, const float* regs, int it, int cnt) {
  const int yh = it & 1, task = it >> 1;
  float acc[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
  if (task < 360) {
    const int i = task % 12, cu = task / 12, c = cu / 5, u = cu - c * 5;
#pragma unroll 1
    for (int k = 0; k < cnt; ++k) {
      const float* reg = regs + k * kImgRegion;
      const float* s1 = reg + kOffS1 + (c * 12 + u + 4 * yh) * 12;
      const float* d2 = reg + kOffD2 + i * kD2K + (4 + 4 * yh) * 8;
#pragma unroll 2
      for (int y = 0; y < 4; ++y) {
        float in[12], d[8];
        load_row<12>(s1 + y * 12, in);
        load_row<8>(d2 + y * 8, d);
#pragma unroll
        for (int v = 0; v < 5; ++v)
#pragma unroll
          for (int x = 0; x < 8; ++x) acc[v] = __fmaf_rn(in[v + x], d[x], acc[v]);
      }
    }
  } else if (task < 372) {
    const int i = task - 360;
    for (int k = 0; k < cnt; ++k) {
      const float4* d = reinterpret_cast<const float4*>(regs + k * kImgRegion + kOffD2 + i * kD2K + (4 + 4 * yh) * 8);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 v = d[q];
        acc[0] += (v.x + v.y) + (v.z + v.w);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < 5; ++v) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], 1);
  if (yh == 0) {
    if (task < 360) {
      const int i = task % 12, cu = task / 12, c = cu / 5, u = cu - c * 5;
      float* g = G + kK2 + ((i * 6 + c) * 5 + u) * 5;
#pragma unroll
      for (int v = 0; v < 5; ++v) g[v] += acc[v];
    } else if (task < 372) {
      G[kB2 + task - 360] += acc[0];
    }
  }
}

// S5 g_k2 lane over all 8 rows (TLB_GK2_FULL): task (kernel i, channel c, row u), i fastest (the twelve
// kernel lanes of a (c, u) read the same s1 rows: broadcast) -- 5 outputs over the 64 taps per image, no
// row-half shuffle; tasks 360..371: g_b2[i].  372 lanes (half the items of gk2_item, twice the work each).
__device__ __forceinline__ void gk2_item_full(float* G, const float* regs, int task, int cnt) {
  float acc[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
  if (task < 360) {
    const int i = task % 12, cu = task / 12, c = cu / 5, u = cu - c * 5;
#pragma unroll 1
    for (int k = 0; k < cnt; ++k) {
      const float* reg = regs + k * kImgRegion;
      const float* s1 = reg + kOffS1 + (c * 12 + u) * 12;
      const float* d2 = reg + kOffD2 + i * kD2K + 4 * 8;
#pragma unroll 2
      for (int y = 0; y < 8; ++y) {
        float in[12], d[8];
        load_row<12>(s1 + y * 12, in);
        load_row<8>(d2 + y * 8, d);
#pragma unroll
        for (int v = 0; v < 5; ++v)
#pragma unroll
          for (int x = 0; x < 8; ++x) acc[v] = __fmaf_rn(in[v + x], d[x], acc[v]);
      }
    }
    float* g = G + kK2 + ((i * 6 + c) * 5 + u) * 5;
#pragma unroll
    for (int v = 0; v < 5; ++v) g[v] += acc[v];
  } else if (task < 372) {
    const int i = task - 360;
    for (int k = 0; k < cnt; ++k) {
      const float4* d = reinterpret_cast<const float4*>(regs + k * kImgRegion + kOffD2 + i * kD2K + 4 * 8);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float4 v = d[q];
        acc[0] += (v.x + v.y) + (v.z + v.w);
      }
    }
    G[kB2 + i] += acc[0];
  }
}

// S6: g_k1 lane (kernel i, row u, row chunk yc of 3 rows), yc fastest: 5 partials over the round's images;
// or a g_b1 lane (kernel i, row chunk yc).  The 8 row-chunk lanes join by a 3-level xor tree.
__device__ __forceinline__ void gk1_item(float* G, const float* imgs, const float* regs, int it, int cnt) {
  const int yc = it & 7;
  float acc[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
  const bool bias = it >= 240;
  const int task = bias ? (it - 240) >> 3 : it >> 3;
  const int i = bias ? task : task / 5, u = bias ? 0 : task - (task / 5) * 5;
  if (!bias) {
#pragma unroll 1
    for (int k = 0; k < cnt; ++k) {
      const float* img = imgs + k * kImg + u * 28;
      const float* dz1 = regs + k * kImgRegion + i * kG1Plane;
#pragma unroll 1
      for (int yy = 0; yy < 3; ++yy) {
        const int y = 3 * yc + yy;
        float in[28], d[24];
        load_row<28>(img + y * 28, in);
        load_row<24>(dz1 + y * 24, d);
#pragma unroll
        for (int v = 0; v < 5; ++v)
#pragma unroll
          for (int x = 0; x < 24; ++x) acc[v] = __fmaf_rn(in[v + x], d[x], acc[v]);
      }
    }
  } else {
    for (int k = 0; k < cnt; ++k) {
      const float4* dz1 = reinterpret_cast<const float4*>(regs + k * kImgRegion + i * kG1Plane + 3 * yc * 24);
#pragma unroll
      for (int q = 0; q < 18; ++q) {
        const float4 v = dz1[q];
        acc[0] += (v.x + v.y) + (v.z + v.w);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], 4);
    acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], 2);
    acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], 1);
  }
  if (yc == 0) {
    if (bias) {
      G[kB1 + i] += acc[0];
    } else {
      float* g = G + kK1 + i * 25 + u * 5;
#pragma unroll
      for (int v = 0; v < 5; ++v) g[v] += acc[v];
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Packed-pair forward items (PAIR = true): conv1 and conv2 run on packed FP32 pairs (__ffma2_rn -> SASS
// FFMA2, sm_100: the FP32 rate of FFMA at half the issued instructions), one operand a broadcast scalar --
//   conv1 : pixel (broadcast) x (k1[c], k1[c+3])        -> (c1[c], c1[c+3])
//   conv2 : s1 (broadcast) x (k2[i][c], k2[i+6][c])     -> (out[i], out[i+6])
// with the same lane counts as the scalar items; activations keep their canonical layouts, so the backward
// items are the scalar ones.  Fast-mode arithmetic (summation trees differ; within the 1e-4 tolerance).
// ------------------------------------------------------------------------------------------------
constexpr int kW1PFloats = 152, kW2PFloats = 6 * 364;
static_assert(kW1PFloats <= kW1Floats && kW2PFloats <= kW2Floats, "pair weights fit the padded slots");
__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 ld2(const float* p) { return *reinterpret_cast<const float2*>(p); }

// Pair weights from P (once per step, all threads): W1p[ip][t] = (k1[ip][t], k1[ip+3][t]) (ip < 3);
// W2p[ip][c][ky][kx] = (k2[ip][c][ky][kx], k2[ip+6][c][ky][kx]) (ip < 6; kx = 5 is a zero pad pair).
__device__ __forceinline__ void build_pair_weights(const float* P, float* W1p, float* W2p, int t, int T) {
  for (int q = t; q < 75 + 6 * 180; q += T) {
    if (q < 75) {
      const int ip = q / 25, tp = q - ip * 25;
      *reinterpret_cast<float2*>(W1p + 2 * q) = make_float2(P[kK1 + ip * 25 + tp], P[kK1 + (ip + 3) * 25 + tp]);
    } else {
      const int q2 = q - 75, ip = q2 / 180, r = q2 - ip * 180, c = r / 30, r2 = r - c * 30, ky = r2 / 6, kx = r2 - ky * 6;
      const float2 v = kx < 5 ? make_float2(P[kK2 + (ip * 6 + c) * 25 + ky * 5 + kx], P[kK2 + ((ip + 6) * 6 + c) * 25 + ky * 5 + kx])
                              : make_float2(0.0f, 0.0f);
      *reinterpret_cast<float2*>(W2p + ip * 364 + c * 60 + ky * 12 + 2 * kx) = v;
    }
  }
}

// S1 pair lane (image k, pooled row py, 6-column strip xs, channel pair ip), ip fastest (the three pair lanes
// of a (py, xs) read the same image rows): conv rows 2py, 2py+1 x 6 columns x channels (ip, ip+3) = 12 FFMA2
// accumulators over the 25 taps (300 FFMA2), logistic, g1 = c1(1-c1), 2x2 pool -> s1 (canonical layouts).
__device__ __forceinline__ void conv1_item_p(const float* P, const float* W1p, const float* imgs, float* regs, int it) {
  const int k = it / 144, r = it - k * 144;
  const int ip = r % 3, pos = r / 3, xs = pos & 3, py = pos >> 2;
  const int y0 = 2 * py, x0 = 6 * xs;
  const float* img = imgs + k * kImg;
  float2 a[2][6];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int o = 0; o < 6; ++o) a[q][o] = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int rr = 0; rr < 6; ++rr) {  // image row y0 + rr feeds conv row q with ky = rr - q
    float in[10];
#pragma unroll
    for (int h = 0; h < 5; ++h) {
      const float2 v = ld2(img + (y0 + rr) * 28 + x0 + 2 * h);
      in[2 * h] = v.x;
      in[2 * h + 1] = v.y;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int ky = rr - q;
      if (ky < 0 || ky > 4) continue;
#pragma unroll
      for (int kx = 0; kx < 5; ++kx) {
        const float2 w = ld2(W1p + 2 * (ip * 25 + ky * 5 + kx));
#pragma unroll
        for (int o = 0; o < 6; ++o) a[q][o] = __ffma2_rn(bc2(in[o + kx]), w, a[q][o]);
      }
    }
  }
  const float nb[2] = {neg_log2e_times(P[kB1 + ip]), neg_log2e_times(P[kB1 + ip + 3])};
  float* reg = regs + k * kImgRegion;
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // channel ip + 3h
    const int i = ip + 3 * h;
    float t[2][6];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int o = 0; o < 6; ++o) t[q][o] = logistic(h ? a[q][o].y : a[q][o].x, nb[h]);
      float* g1 = reg + i * kG1Plane + (y0 + q) * 24 + x0;
#pragma unroll
      for (int o2 = 0; o2 < 3; ++o2)
        *reinterpret_cast<float2*>(g1 + 2 * o2) =
            make_float2(t[q][2 * o2] * (1.0f - t[q][2 * o2]), t[q][2 * o2 + 1] * (1.0f - t[q][2 * o2 + 1]));
    }
    float* s1 = reg + kOffS1 + (i * 12 + py) * 12 + 3 * xs;
#pragma unroll
    for (int px = 0; px < 3; ++px)  // avgpool (nn.cpp:144): ((p00 + p01) + p10) + p11, then * 0.25f
      s1[px] = (((t[0][2 * px] + t[0][2 * px + 1]) + t[1][2 * px]) + t[1][2 * px + 1]) * 0.25f;
  }
}

// S2 pair lane (image k, pooled row py, kernel pair ip, conv row r of the pooling window, channel half h), h
// fastest: conv row y = 2py + r x 8 columns x kernels (ip, ip+6) over channels 3h..3h+2 -- the s1 value is
// the broadcast operand, (k2[ip][c], k2[ip+6][c]) the weight pair (600 FFMA2) -- the halves joined by a
// shuffle (lane ^ 1); lane h finishes kernel ip + 6h: logistic, g2 into the padded dz2 row, and the 2x2
// pool with the partner row (lane ^ 2).  W2p: [ip][c][ky][6] float2 in 364-float kernel-pair rows.
constexpr int kW2PRow = 364;
__device__ __forceinline__ void conv2_item_kp(const float* P, const float* W2p, float* regs, int it) {
  const int h = it & 1, r = (it >> 1) & 1, rest = it >> 2;
  const int ip = rest % 6, kp = rest / 6, py = kp & 3, k = kp >> 2;
  const int y = 2 * py + r;
  float* reg = regs + k * kImgRegion;
  const float* s1 = reg + kOffS1;
  float2 acc[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) acc[o] = make_float2(0.0f, 0.0f);
#pragma unroll 1
  for (int c = 3 * h; c < 3 * h + 3; ++c) {
    const float* wc = W2p + ip * kW2PRow + c * 60;
#pragma unroll
    for (int ky = 0; ky < 5; ++ky) {
      float in[12];
      load_row<12>(s1 + (c * 12 + y + ky) * 12, in);
      const float4* wr = reinterpret_cast<const float4*>(wc + ky * 12);
      const float4 w01 = wr[0], w23 = wr[1], w4 = wr[2];
      const float2 wv[5] = {make_float2(w01.x, w01.y), make_float2(w01.z, w01.w), make_float2(w23.x, w23.y),
                            make_float2(w23.z, w23.w), make_float2(w4.x, w4.y)};
#pragma unroll
      for (int kx = 0; kx < 5; ++kx)
#pragma unroll
        for (int o = 0; o < 8; ++o) acc[o] = __ffma2_rn(bc2(in[o + kx]), wv[kx], acc[o]);
    }
  }
  float t[8], u[8];
  const int i = ip + 6 * h;
  const float nb = neg_log2e_times(P[kB2 + i]);
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    const float ox = acc[o].x + __shfl_xor_sync(0xffffffffu, acc[o].x, 1);
    const float oy = acc[o].y + __shfl_xor_sync(0xffffffffu, acc[o].y, 1);
    t[o] = logistic(h ? oy : ox, nb);
  }
  float* g2 = reg + kOffD2 + i * kD2K + (4 + y) * 8;
  reinterpret_cast<float4*>(g2)[0] =
      make_float4(t[0] * (1.0f - t[0]), t[1] * (1.0f - t[1]), t[2] * (1.0f - t[2]), t[3] * (1.0f - t[3]));
  reinterpret_cast<float4*>(g2)[1] =
      make_float4(t[4] * (1.0f - t[4]), t[5] * (1.0f - t[5]), t[6] * (1.0f - t[6]), t[7] * (1.0f - t[7]));
#pragma unroll
  for (int o = 0; o < 8; ++o) u[o] = __shfl_xor_sync(0xffffffffu, t[o], 2);  // conv row y ^ 1
  if (r == 0) {  // avgpool (nn.cpp:144): ((p00 + p01) + p10) + p11, then * 0.25f
    float pv[4];
#pragma unroll
    for (int px = 0; px < 4; ++px) pv[px] = (((t[2 * px] + t[2 * px + 1]) + u[2 * px]) + u[2 * px + 1]) * 0.25f;
    *reinterpret_cast<float4*>(reg + kOffS2 + (i * 4 + py) * 4) = make_float4(pv[0], pv[1], pv[2], pv[3]);
  }
}

// Rounds of one CTA: (step, first local example, end of the CTA's range -- the group's size when
// interleaved, the contiguous chunk's end otherwise --, the CTA's position index j in the group).
struct Round {
  int64_t step, e, hi, j;
};

// Which rounds of a group a CTA trains (round r = local examples [r NI, r NI + NI)).
// Interleaved (TLB_BT_INTERLEAVE, default): round r belongs to CTA r % grid, so any prefix of the group
// feeds every CTA's first rounds -- a host call's ingestion chunks (tlb_train on host buffers) are
// consumed as they land instead of the whole first group having to arrive before the last CTA can start.
// With two CTAs per SM the warp schedulers favour the CTA that arrived first (measured: it finishes its
// rounds 13% sooner on 144-148 of 148 SMs, profiles/r2/trace_batch_*_trb2.json), so the partner would idle
// through the tail of every step.  Paired mapping: round r belongs to SM pair p = r % (grid / 2) at
// position j = r / (grid / 2); slot 0 (the first-arrived CTA) takes the positions where floor(j share)
// steps (`share` of them), slot 1 the others.  Partial rows and loss slots are indexed by the work id
// 2p + slot, so which examples are summed into which row -- and the result -- does not depend on where
// the hardware placed the CTAs.  TLB_BT_INTERLEAVE=0: contiguous static chunks (the earlier mapping).
#ifndef TLB_BT_INTERLEAVE
#define TLB_BT_INTERLEAVE 1
#endif
struct WorkMap {
  int wid;      // work id: partial row, rounds
  int paired;   // 1: SM-pair mapping
  float share;  // slot 0's share of the pair's examples
  int share_q;  // share in 1/1024
};

// Slot of a pair's position j: slot 0 takes the positions where floor(j share) steps (share in 1/1024).
// (An exact per-pair count -- round(n share) of the pair's n positions, spread by division -- measured
// slower: profiles/r2/bt_ilv*_ilv4.jsonl.)
__device__ __forceinline__ int pair_slot(int64_t j, int q) {
  return (((j + 1) * q) >> 10) != ((j * q) >> 10) ? 0 : 1;
}

template <int NI>
__device__ __forceinline__ void work_chunk(int64_t m, const WorkMap& w, int64_t& lo, int64_t& hi) {
  if (!w.paired) {
    static_chunk(m, gridDim.x, w.wid, lo, hi);
    return;
  }
  int64_t plo, phi;
  static_chunk(m, gridDim.x / 2, w.wid >> 1, plo, phi);
  const int64_t len = phi - plo;
  int64_t s0 = (int64_t)__fmul_rn(w.share, (float)len);
  s0 = min(len, (s0 + NI / 2) / NI * NI);
  if (w.wid & 1) lo = plo + s0, hi = phi;
  else lo = plo, hi = plo + s0;
}

// The CTA's first round at position >= j of a group of m examples (r.step is the caller's).  ILV: the
// interleaved mapping (launches whose groups give every CTA >= 4 rounds); otherwise contiguous chunks
// (with fewer rounds a contiguous chunk can end in a partial round -- 1k images on 148 CTAs: 4 + 3 images
// each -- where whole interleaved rounds put 8 images on some CTAs: -5% at 1k, profiles/r2/bt_ilv*_ilv1.jsonl).
template <int NI, bool ILV>
__device__ __forceinline__ bool seek_round(const WorkMap& w, int64_t m, int64_t j, Round& r) {
  if constexpr (!ILV) {
    int64_t lo, hi;
    work_chunk<NI>(m, w, lo, hi);
    if (lo + j * NI >= hi) return false;
    r.e = lo + j * NI;
    r.hi = hi;
    r.j = j;
    return true;
  }
  const int64_t R = (m + NI - 1) / NI;
  if (!w.paired) {
    const int64_t rr = w.wid + j * (int64_t)gridDim.x;
    if (rr >= R) return false;
    r.e = rr * NI;
    r.hi = m;
    r.j = j;
    return true;
  }
  const int P = (int)gridDim.x >> 1, p = w.wid >> 1, sl = w.wid & 1;
  for (;; ++j) {
    const int64_t rr = p + j * (int64_t)P;
    if (rr >= R) return false;
    if (pair_slot(j, w.share_q) == sl) {
      r.e = rr * NI;
      r.hi = m;
      r.j = j;
      return true;
    }
  }
}
// The CTA's next round of the same group (false: none left).
template <int NI, bool ILV>
__device__ __forceinline__ bool step_round(const WorkMap& w, Round& r) {
  if constexpr (ILV) return seek_round<NI, true>(w, r.hi, r.j + 1, r);
  if (r.e + NI >= r.hi) return false;
  r.e += NI;
  ++r.j;
  return true;
}

template <int NI, bool ILV>
__device__ __forceinline__ bool first_round(const TrainArgs& a, const WorkMap& w, int64_t from, Round& r) {
  for (int64_t st = from; st < a.step_end; ++st) {
    if (seek_round<NI, ILV>(w, local_size(a, st), 0, r)) {
      r.step = st;
      return true;
    }
  }
  return false;
}
template <int NI, bool ILV>
__device__ __forceinline__ bool next_round(const TrainArgs& a, const WorkMap& w, Round& r) {
  if (step_round<NI, ILV>(w, r)) return true;
  return first_round<NI, ILV>(a, w, r.step + 1, r);
}

// Paired mapping (MINB == 2): every CTA publishes (SM id, arrival slot on its SM); after a grid barrier each
// CTA ranks its SM among the SMs present.  Any SM without exactly two CTAs (or an odd grid) keeps the
// default mapping on every CTA -- all CTAs read the same table, so they agree.  `scratch` holds >= 544 ints.
__device__ WorkMap pair_map(const TrainArgs& a, int* scratch, unsigned int& target) {
  constexpr int kMaxSm = 512;
  static_assert((kMaxSm + kPairMaxGrid) * 4 <= kBatchWorkExtraBytes, "slot counters + table fit");
  const int t = threadIdx.x, T = blockDim.x, nb = gridDim.x;
  unsigned int* slots = reinterpret_cast<unsigned int*>(a.work + (int64_t)nb * kPStride);  // zeroed at launch
  unsigned int* table = slots + kMaxSm;
  if (t == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const unsigned int slot = smid < kMaxSm ? atomicAdd(slots + smid, 1u) : 2u;
    __stcg(table + blockIdx.x, smid < kMaxSm && slot < 2 ? (smid << 1 | slot) : 0xffffffffu);
  }
  grid_sync(a.barrier, target);
  int* hist = scratch;           // [kMaxSm] CTAs per SM id
  int* flags = scratch + kMaxSm;  // [0] bad, [1] my SM's rank x 2
  for (int q = t; q < kMaxSm; q += T) hist[q] = 0;
  if (t < 2) flags[t] = 0;
  __syncthreads();
  for (int q = t; q < nb; q += T) {
    const unsigned int v = __ldcg(table + q);
    if (v == 0xffffffffu) flags[0] = 1;
    else atomicAdd(hist + (v >> 1), 1);
  }
  __syncthreads();
  const unsigned int mine = __ldcg(table + blockIdx.x);
  int below = 0;
  for (int q = t; q < kMaxSm; q += T) {
    if (hist[q] != 0 && hist[q] != 2) flags[0] = 1;
    if (mine != 0xffffffffu && q < (int)(mine >> 1)) below += hist[q];
  }
  if (below) atomicAdd(flags + 1, below);
  __syncthreads();
  WorkMap w{(int)blockIdx.x, 0, 0.5f, 512};
  if (!flags[0] && (nb & 1) == 0)
    w = WorkMap{flags[1] + (int)(mine & 1), 1, a.pair_share, (int)__float2int_rn(a.pair_share * 1024.0f)};
  __syncthreads();  // scratch is reused by the caller
  return w;
}

// Issuer: the round's labels (cp.async, completed at the round's start) and ONE bulk copy of its images.
// Byte-ingestion state of the two ring buffers (shared memory): first example index, byte flag, count.
struct RoundBytes {
  int64_t* idx;
  int* bst;
  int* cnt;
};

template <int NI>
__device__ __forceinline__ void issue_round(const TrainArgs& a, float* ring, uint8_t* pxring, const RoundBytes& rb,
                                            int* lab, uint64_t* bar, int buf, const Round& r) {
  const int cnt = (int)min((int64_t)NI, r.hi - r.e);
  const int64_t first = example_index(a, r.step, r.e);
  for (int q = 0; q < cnt; ++q) wait_ready_at(a, r.step, first + q);
  for (int q = 0; q < cnt; ++q) cp_async4(lab + buf * NI + q, a.labels + first + q);
  fence_proxy_async_smem();
  rb.bst[buf] = step_bytes(a, r.step) ? 1 : 0;
  if (rb.bst[buf]) {  // byte ingestion: the round's bytes, converted during the previous round's S3
    rb.idx[buf] = first;
    rb.cnt[buf] = cnt;
    mbar_arrive_expect_tx(&bar[buf], (uint32_t)(cnt * kImg));
    tma_load_1d(pxring + buf * NI * kImg, a.pixels + first * kImg, (uint32_t)(cnt * kImg), &bar[buf]);
    return;
  }
  if (a.pixels) asm volatile("fence.proxy.async.global;" ::: "memory");  // fp32 written back in epoch 1
  mbar_arrive_expect_tx(&bar[buf], (uint32_t)(cnt * kImg * sizeof(float)));
  tma_load_1d(ring + buf * NI * kImg, a.images + first * kImg, (uint32_t)(cnt * kImg * sizeof(float)), &bar[buf]);
}

template <int NI, int T, int MINB, bool PAIR, bool ILV>
__global__ void __launch_bounds__(T, MINB) train_batch_kernel(TrainArgs a) {
  static_assert(T % 32 == 0, "stage loops run whole warps");
  using L = Layout<NI>;
  float* const P = bt_smem + L::kP;
  float* const W1 = bt_smem + L::kW1;
  float* const W2 = bt_smem + L::kW2;
  float* const G = bt_smem + L::kG;
  float* const ring = bt_smem + L::kRing;
  int* const lab = reinterpret_cast<int*>(bt_smem + L::kLab);
  float* const regs = bt_smem + L::kImgs;
  uint64_t* const bar = reinterpret_cast<uint64_t*>(bt_smem + L::kFloats);
  int64_t* const ridx = reinterpret_cast<int64_t*>(bar + 2);
  uint8_t* const pxring = reinterpret_cast<uint8_t*>(ridx + 2);
  int* const rbst = reinterpret_cast<int*>(pxring + 2 * NI * kImg);
  const RoundBytes rb{ridx, rbst, rbst + 2};
  const int t = threadIdx.x, nb = gridDim.x;
  unsigned int target = 0;

  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  WorkMap wm{(int)blockIdx.x, 0, 0.5f, 512};
  if (MINB == 2 && a.pair_share > 0.0f) wm = pair_map(a, reinterpret_cast<int*>(regs), target);
  for (int q = t; q < NI * kImgRegion; q += T) regs[q] = 0.0f;  // dz2 pad rows stay zero
  __syncthreads();
  const bool issuer = t == T - 32;  // lane 0 of the last warp (idle in S2/S6 of a full round)
  Round pf;
  bool pf_valid = first_round<NI, ILV>(a, wm, a.step_begin, pf);
  if (issuer && pf_valid) issue_round<NI>(a, ring, pxring, rb, lab, bar, 0, pf);
  if (pf_valid && step_bytes(a, pf.step)) {  // the first round's bytes: converted by every thread
    __syncthreads();
    mbar_wait(&bar[0], 0);
    convert_pixels(pxring, ring, (a.images_wb ? a.images_wb + ridx[0] * kImg : nullptr), rb.cnt[0], t, T);
    __syncthreads();
  }
  uint32_t consumed = 0;

  // profiling (tlb_ctx_set_trace): per step and CTA, globaltimer stamps [8]: 0 step start (weights
  // staged), 1 rounds done, 2 after grid barrier 1, 3 reduction done, 4 after grid barrier 2, 5 rounds;
  // step 0's row also holds 6 the SM id and 7 the kernel entry time
  unsigned long long* const trace = (a.trace && t == 0) ? a.trace + (int64_t)blockIdx.x * 8 : nullptr;
  const auto stamp = [&](int64_t st, int k) {
    if (trace) trace[(st - a.step_begin) * nb * 8 + k] = globaltimer_ns();
  };
  if (trace) {  // 6: SM id, 7: kernel entry (step 0's row)
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    trace[6] = smid;
    trace[7] = globaltimer_ns();
  }
  int64_t ks = umod(a.step_begin, a.steps_per_epoch), ep = udiv(a.step_begin, a.steps_per_epoch);
  for (int64_t st = a.step_begin; st < a.step_end; ++st, ks = ks + 1 == a.steps_per_epoch ? (++ep, 0) : ks + 1) {
    int64_t l_lo, l_hi;
    local_range_k(a, ks, l_lo, l_hi);
    const int64_t m = l_hi - l_lo;
    // ---- the step's weights -> shared (+ padded conv copies), zero the CTA gradient ----
    {
      const float4* src = reinterpret_cast<const float4*>(a.params);
      float4* dst = reinterpret_cast<float4*>(P);
      for (int q = t; q < kPStride / 4; q += T) dst[q] = __ldcg(src + q);
      for (int q = t; q < kPStride; q += T) G[q] = 0.0f;
    }
    __syncthreads();
    if constexpr (PAIR) {
      build_pair_weights(P, W1, W2, t, T);
    } else {
      for (int q = t; q < kW1Floats + kW2Floats; q += T) {
        if (q < kW1Floats) {
          const int i = q / kW1Stride, rr = q - i * kW1Stride, ky = rr >> 3, kx = rr & 7;
          W1[q] = (ky < 5 && kx < 5) ? P[kK1 + i * 25 + ky * 5 + kx] : 0.0f;
        } else {
          const int q2 = q - kW1Floats, i = q2 / kW2Stride, rr = q2 - i * kW2Stride, c = rr / 40, r2 = rr - c * 40;
          const int ky = r2 >> 3, kx = r2 & 7;
          W2[q2] = (c < 6 && kx < 5) ? P[kK2 + (i * 6 + c) * 25 + ky * 5 + kx] : 0.0f;
        }
      }
    }
    __syncthreads();

    double cta_loss = 0.0;  // thread 0: this CTA's example losses in example order (fp64)
    stamp(st, 0);
    Round cur{st, 0, 0, 0};
    int64_t nrounds = 0;  // this CTA's rounds of the step (trace)
    for (bool have = seek_round<NI, ILV>(wm, m, 0, cur); have; have = step_round<NI, ILV>(wm, cur), ++nrounds) {
      const int cnt = (int)min((int64_t)NI, cur.hi - cur.e);
      const int buf = consumed & 1;
      mbar_wait(&bar[buf], (consumed >> 1) & 1);
      if (issuer) {
        cp_async_wait_all();  // this round's labels (published by S1's barrier)
        rbst[buf ^ 1] = 0;    // (issue_round sets it for a next round that arrives as bytes)
        if (pf_valid) {
          Round nx = pf;
          if (next_round<NI, ILV>(a, wm, nx)) {
            issue_round<NI>(a, ring, pxring, rb, lab, bar, buf ^ 1, nx);  // buf^1 was last read by the previous round's S6
            pf = nx;
          } else {
            pf_valid = false;
          }
        }
      }
      const float* imgs = ring + buf * NI * kImg;
      const int* rl = lab + buf * NI;
      // S1
      for (int it = t; it < cnt * 144; it += T) {
        if constexpr (PAIR) conv1_item_p(P, W1, imgs, regs, it);
        else conv1_item(P, W1, imgs, regs, it);
      }
      __syncthreads();
      // S2 (cnt * 192 lanes: whole warps)
      for (int it = t; it < cnt * (PAIR ? 96 : 192); it += T) {  // pair items: 96 lanes per image
        if constexpr (PAIR) conv2_item_kp(P, W2, regs, it);
        else conv2_item(P, W2, regs, it);
      }
      __syncthreads();
      // S3
      {
        const int nfc = (cnt * 80 + 31) / 32 * 32;
        for (int it = t; it < nfc; it += T) fc_item(P, regs, rl, it, it < cnt * 80);
        // byte ingestion: the idle threads convert the NEXT round's bytes (landed during S1/S2)
        const int nb = buf ^ 1;
        if (t >= nfc && rbst[nb]) {
          mbar_wait(&bar[nb], ((consumed + 1) >> 1) & 1);
          convert_pixels(pxring + nb * NI * kImg, ring + nb * NI * kImg, (a.images_wb ? a.images_wb + ridx[nb] * kImg : nullptr), rb.cnt[nb],
                         t - nfc, T - nfc);
        }
      }
      __syncthreads();
      // S4: d_s2 = fc^T dz -> dz2 = (d_s2 / 4) g2 in place; thread 0 adds the round's losses
      if (t == 0) {
        for (int k = 0; k < cnt; ++k) {  // net::loss (network.cpp:97-109)
          const float* od = regs + k * kImgRegion + kOffOd;
          float l = 0.0f;
#pragma unroll
          for (int i = 0; i < 10; ++i) {
            const float d = (i == rl[k] ? 1.0f : 0.0f) - od[i];
            l = __fmaf_rn(d, d, l);
          }
          cta_loss += (double)(0.5f * l);
        }
      }
      for (int it = t; it < cnt * 96; it += T) {  // two pooled columns (j, j + 1) per lane
        const int k = it / 96, j = 2 * (it - k * 96);
        float* reg = regs + k * kImgRegion;
        const float* dz = reg + kOffOd + 16;
        float ds0 = 0.0f, ds1 = 0.0f;
#pragma unroll
        for (int i = 0; i < 10; ++i) {
          const float2 w = *reinterpret_cast<const float2*>(P + kFC + i * 192 + j);
          ds0 = __fmaf_rn(w.x, dz[i], ds0);
          ds1 = __fmaf_rn(w.y, dz[i], ds1);
        }
        ds0 *= 0.25f;  // backavgpool (nn.cpp:148-158)
        ds1 *= 0.25f;
        const int i2 = j >> 4, py = (j >> 2) & 3, px = j & 3;
        float* d2 = reg + kOffD2 + i2 * kD2K + (4 + 2 * py) * 8 + 2 * px;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          float4* q4 = reinterpret_cast<float4*>(d2 + rr * 8);
          const float4 g = *q4;
          *q4 = make_float4(ds0 * g.x, ds0 * g.y, ds1 * g.z, ds1 * g.w);
        }
      }
      __syncthreads();
      // S5: backin (heaviest items first; 4-lane groups, whole warps) | g_k2 + g_b2 (lane pairs, whole
      // warps) | g_fc + g_b (one lane per output, light items that fill the tail)
      {
        const int nbi = (cnt * 144 + 31) / 32 * 32, n2 = nbi + (TLB_GK2_FULL ? 384 : 768), nfc = n2 + 490;
        for (int it = t; it < nfc; it += T) {
          if (it < nbi) {
            if constexpr (PAIR) backin_item<true>(P, regs, it, cnt, it < cnt * 144);
            else backin_item(W2, regs, it, cnt, it < cnt * 144);
          } else if (it < n2) {
            if constexpr (TLB_GK2_FULL) gk2_item_full(G, regs, it - nbi, cnt);
            else gk2_item(G, regs, it - nbi, cnt);
          } else if (it < n2 + 480) {  // g_fc, four columns per lane (float4 s2 / G)
            const int o4 = it - n2, i = o4 / 48, j4 = o4 - i * 48;
            float4 g = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            for (int k = 0; k < cnt; ++k) {
              const float* reg = regs + k * kImgRegion;
              const float4 sv = reinterpret_cast<const float4*>(reg + kOffS2)[j4];
              const float d = reg[kOffOd + 16 + i];
              g.x = __fmaf_rn(sv.x, d, g.x);
              g.y = __fmaf_rn(sv.y, d, g.y);
              g.z = __fmaf_rn(sv.z, d, g.z);
              g.w = __fmaf_rn(sv.w, d, g.w);
            }
            float4* gp = reinterpret_cast<float4*>(G + kFC) + o4;
            float4 gv = *gp;
            gv.x += g.x; gv.y += g.y; gv.z += g.z; gv.w += g.w;
            *gp = gv;
          } else {
            const int i = it - n2 - 480;
            float g = 0.0f;
            for (int k = 0; k < cnt; ++k) g += regs[k * kImgRegion + kOffOd + 16 + i];
            G[kB + i] += g;
          }
        }
      }
      __syncthreads();
      // S6: g_k1 (240 lanes) + g_b1 (48 lanes)
      for (int it = t; it < 288; it += T) gk1_item(G, imgs, regs, it, cnt);
      __syncthreads();
      ++consumed;
    }

    // ---- CTA partial -> work row; grid barrier; ordered reduction + sgd_step; grid barrier ----
    stamp(st, 1);
    if (trace) trace[(st - a.step_begin) * nb * 8 + 5] = (unsigned long long)nrounds;
    {  // every row is written (zero if the CTA had no round: small groups)
      float4* dst = reinterpret_cast<float4*>(a.work + (int64_t)wm.wid * kPStride);
      const float4* src = reinterpret_cast<const float4*>(G);
      for (int q = t; q < kPStride / 4; q += T) __stcg(dst + q, src[q]);
      if (t == 0) a.loss_part[wm.wid] = cta_loss;
    }
    grid_sync(a.barrier, target);
    stamp(st, 2);
    const int64_t nrows = nb;  // every CTA's row (written above)
    {
      int64_t j0, j1;
      static_chunk(kNParam, nb, blockIdx.x, j0, j1);
      float* red = G;  // the CTA gradient is in its work row; G is zeroed again at the next step
      for (int64_t jb = j0; jb < j1; jb += T) {
        const int W = (int)min((int64_t)T, j1 - jb);
        const int rstep = T / W, c = t % W, r0 = t / W;
        float acc = 0.0f;
        if (r0 < rstep) {
          if constexpr (MINB == 1) {
            // one CTA per SM (groups < 8k): up to 16 rows in flight per thread (one L2 round trip for the
            // usual ~7 rows), summed by a fixed tree (absent rows add +0.0f: exact); 1 k: +1-2.5%
            // (profiles/r2/bt_ilv*_red1.jsonl).  (With two CTAs per SM it showed intermittent -2.5% runs at
            // 16 k / 64 k: red2; the four-wide loop stays there.)
            for (int64_t r = r0; r < nrows; r += 16 * rstep) {
              float v[16];
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const int64_t rr = r + u * rstep;
                v[u] = rr < nrows ? __ldcg(a.work + rr * kPStride + jb + c) : 0.0f;
              }
#pragma unroll
              for (int w = 1; w < 16; w <<= 1)
#pragma unroll
                for (int u = 0; u < 16; u += 2 * w) v[u] += v[u + w];
              acc += v[0];
            }
          } else {
            int64_t r = r0;
            for (; r + 3 * rstep < nrows; r += 4 * rstep) {  // four loads in flight, fixed order
              const float v0 = __ldcg(a.work + r * kPStride + jb + c);
              const float v1 = __ldcg(a.work + (r + rstep) * kPStride + jb + c);
              const float v2 = __ldcg(a.work + (r + 2 * rstep) * kPStride + jb + c);
              const float v3 = __ldcg(a.work + (r + 3 * rstep) * kPStride + jb + c);
              acc = ((acc + v0) + v1) + (v2 + v3);
            }
            for (; r < nrows; r += rstep) acc += __ldcg(a.work + r * kPStride + jb + c);
          }
        }
        red[t] = acc;
        __syncthreads();
        if (t < W) {
          float s = 0.0f;
          for (int q = 0; q < rstep; ++q) s += red[t + q * W];
          const int j = (int)jb + t;
          if (a.grad_out) a.grad_out[j] = s;
          else __stcg(a.params + j, fsub(P[j], fmul(a.rate, __fdiv_rn(s, (float)m))));
        }
        __syncthreads();
      }
    }
    if (blockIdx.x == nb - 1) {  // fp64 loss of the group (network.cpp:239-242): CTA partials in CTA order
      double* dl = reinterpret_cast<double*>(G);  // G is free until the next step zeroes it
      double l = (!a.grad_out && ks != 0) ? a.epoch_loss[ep] : 0.0;
      for (int64_t r0 = 0; r0 < nrows; r0 += 1024) {
        const int n = (int)min((int64_t)1024, nrows - r0);
        for (int q = t; q < n; q += T) dl[q] = __ldcg(a.loss_part + r0 + q);
        __syncthreads();
        if (t == 0)
          for (int q = 0; q < n; ++q) l = __dadd_rn(l, dl[q]);
        __syncthreads();
      }
      if (t == 0) {
        if (a.grad_out) a.loss_out[0] = l;
        else a.epoch_loss[ep] = (ks == a.steps_per_epoch - 1) ? __ddiv_rn(l, (double)a.n) : l;
      }
    }
    stamp(st, 3);
    grid_sync(a.barrier, target);
    stamp(st, 4);
  }
}

template <int NI, int T, int MINB, bool PAIR, bool ILV = false>
cudaError_t prep(int* occ) {
  auto kern = train_batch_kernel<NI, T, MINB, PAIR, ILV>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Layout<NI>::kBytes);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, T, Layout<NI>::kBytes);
}

// Slot 0's share of an SM pair's examples (TLB_PAIR_SHARE overrides; 0 = per-CTA static chunks).
inline float pair_share() {
  static const float v = [] {
    const char* e = std::getenv("TLB_PAIR_SHARE");
    return e ? std::strtof(e, nullptr) : kPairShare;
  }();
  return v;
}

template <int NI, int T, int MINB, bool PAIR>
cudaError_t launch_cfg(const TrainArgs& a, int sm_count, int64_t m_max, cudaStream_t st, int* grid_out) {
  int occ = 0;
  int occ_ilv = 0;
  cudaError_t e = prep<NI, T, MINB, PAIR>(&occ);
  if (e == cudaSuccess) e = prep<NI, T, MINB, PAIR, true>(&occ_ilv);
  occ = std::min(occ, occ_ilv);
  if (e != cudaSuccess) return e;
  const int64_t cap = (int64_t)std::max(occ, 1) * sm_count;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cap, (m_max + NI - 1) / NI));
  if (grid_out) {  // sizing query only
    *grid_out = grid;
    return cudaSuccess;
  }
  e = cudaMemsetAsync(a.barrier, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return e;
  TrainArgs la = a;
  la.pair_share = (MINB == 2 && grid % 2 == 0 && grid <= kPairMaxGrid) ? pair_share() : 0.0f;
  if (la.pair_share > 0.0f) {  // the paired mapping's per-SM slot counters (after the grid's partial rows)
    e = cudaMemsetAsync(a.work + (int64_t)grid * kPStride, 0, 512 * sizeof(unsigned int), st);
    if (e != cudaSuccess) return e;
  }
  void* args[] = {&la};
  // Interleaved rounds only while a host call's ingestion chunks are landing (a.ready: tlb_train on host
  // buffers) and every CTA gets >= 4 rounds of a full group (see seek_round): with the data resident the
  // contiguous chunks are ~2% faster (profiles/r2/bt_ilv*_ilv5.jsonl), with chunks in flight interleaving
  // lets every CTA start on the first chunk (16k e2e 17-20 -> 23 M img/s).
  const bool ilv = TLB_BT_INTERLEAVE && a.ready != nullptr && m_max >= 4LL * NI * grid;
  const void* kern = ilv ? (const void*)train_batch_kernel<NI, T, MINB, PAIR, true>
                         : (const void*)train_batch_kernel<NI, T, MINB, PAIR, false>;
  return cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(T), args,
                                     Layout<NI>::kBytes, st);
}

// TLB_BATCH_CFG = "[p]NIxTHREADSxMINB" picks a measured alternative (A/B); default below:
// the packed-pair forward with 4 images per 640-thread CTA (one per SM) for groups of < 8k images per GPU
// (1k: 17.0 -> 20.6 M img/s), 2 images per 320-thread CTA (two per SM, SM-pair work mapping) from 8k
// (16k: 23.3 -> 25.0, 256k: 24.2 -> 25.9 M img/s; profiles/r2/pair_time_p3.jsonl, pair_time_p5.jsonl;
// with the SM-pair mapping the two are within +-2% at 2k-4k either way: profiles/r2/thr_*.jsonl, sweep_r2z).
template <typename F>
cudaError_t dispatch(F&& f, int64_t m_max) {
  static const char* cfg = std::getenv("TLB_BATCH_CFG");
  const auto is = [](const char* want) { return cfg && !std::strcmp(cfg, want); };
  if (is("p2x384x2")) return f.template operator()<2, 384, 2, true>();
  if (is("p2x256x2")) return f.template operator()<2, 256, 2, true>();
  if (is("p2x288x2")) return f.template operator()<2, 288, 2, true>();
  if (is("2x384x2")) return f.template operator()<2, 384, 2>();
  if (is("2x512x1")) return f.template operator()<2, 512, 1>();
  if (is("4x512x1")) return f.template operator()<4, 512, 1>();
  if (is("p4x512x1")) return f.template operator()<4, 512, 1, true>();
  if (is("p4x640x1") || (!cfg && m_max < 8192)) return f.template operator()<4, 640, 1, true>();
  return f.template operator()<2, 320, 2, true>();
}

struct GridQuery {
  int sm;
  int64_t m;
  int* g;
  template <int NI, int T, int MINB, bool PAIR = false>
  cudaError_t operator()() { return launch_cfg<NI, T, MINB, PAIR>(TrainArgs{}, sm, m, nullptr, g); }
};
struct Launcher {
  const TrainArgs& a;
  int sm;
  int64_t m;
  cudaStream_t st;
  template <int NI, int T, int MINB, bool PAIR = false>
  cudaError_t operator()() { return launch_cfg<NI, T, MINB, PAIR>(a, sm, m, st, nullptr); }
};

}  // namespace bt

// Grid of the batched train kernel for groups of up to m_max local examples (the work-row count).
int batch_train_grid(int sm_count, int64_t m_max) {
  int grid = 0;
  bt::GridQuery q{sm_count, m_max, &grid};
  if (bt::dispatch(q, m_max) != cudaSuccess) return 0;
  return grid;
}

cudaError_t launch_train_batch(const TrainArgs& a, int sm_count, int64_t m_max, cudaStream_t st) {
  bt::Launcher l{a, sm_count, m_max, st};
  return bt::dispatch(l, m_max);
}

}  // namespace tlb
