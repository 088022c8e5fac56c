// zhang_step.cuh -- one CTA (512 threads, or 256 with two CTAs per SM) runs the whole Zhang-CNN
// training cell of one image out of shared memory.
//
// Reference path (proj/src/network.cpp:81-169, kernels proj/src/nn.cpp:96-217):
//   c1 = sigmoid(mconv(I,k1,b1)); s1 = avgpool(c1); c2 = sigmoid(mconv(s1,k2,b2)); s2 = avgpool(c2);
//   out = sigmoid(mconv(s2,fc,b)); loss = 1/2 sum (y-out)^2; hand backprop FC -> C2 -> C1.
//
// Every stage maps the reference's per-output computation onto CTA threads.  With EXACT=true each
// output is produced in exactly the reference's summation order with separately rounded products (no
// FMA), the glibc expf restatement and IEEE reciprocal, so results are bitwise identical to the
// reference (SURVEY.md §8(a) numerics contract).  Where an output's order is a chain over kernels
// (backin's acc = acc + b_i), the per-kernel terms are formed by separate lanes and handed to one lane by
// warp shuffles, which adds them in kernel order; backin forms only the valid (unclipped) taps, in the
// reference's order (backin_rows_exact).  With EXACT=false the stages use FFMA, split long sums across
// lanes (deterministic fixed trees; within the 1e-4 tolerance) and the MUFU sigmoid; the schedule of
// the fast backward (scatter-form backin, row-form g_k2 split across the C2/C1 phases) and of every
// variant kept for the stage bench (csrc/stage_bench.cu) is chosen by the TLB_* switches below, each
// settled by a same-box A/B (profiles/README.md).
//
// Batch 100 runs one 512-thread CTA per SM (16 warps, latency-bound step); launches with more than one
// image per SM run 256-thread CTAs, two per SM, whose barrier stalls overlap (the stages loop over their
// lanes).  Shared memory: a common prefix + an aliased fast/EXACT tail (+ the clustered kernel's DSMEM
// receive buffer), see carve_smem: 104 KB fast, 94 KB EXACT, 146 KB clustered.
#pragma once

#include "tlb_common.cuh"

// EXACT C1 weight gradient: register-blocked v-groups (1, default) or one lane per output (0).
#ifndef TLB_C1BACK_GROUP2
#define TLB_C1BACK_GROUP2 1
#endif
#ifndef TLB_C1BACK_EXACT_BLOCKED
#define TLB_C1BACK_EXACT_BLOCKED 1
#endif

namespace tlb {

constexpr int kThreads = 512;
// backin_rows kernel-loop unroll (A/B: 3 = the three kernels' loads can overlap, +0.7% vs 1)
// Fast forward on packed FP32 pairs (fma.rn.f32x2 -> FFMA2; see "Packed-pair fast forward" below).
// 0 = the scalar fast forward stages.
#ifndef TLB_PAIR
#define TLB_PAIR 1
#endif
#ifndef TLB_GK2K
#define TLB_GK2K 1  // fast g_k2 on kernel pairs (FFMA2): TLB_GK2K_SPLIT lanes beside backin, the rest beside g_k1
#endif
#ifndef TLB_GK2K_SPLIT
#define TLB_GK2K_SPLIT 96
#endif

#ifndef TLB_C2K
#define TLB_C2K 8  // pair conv2: columns per lane (8: 96 lanes, 4: 192 lanes)
#endif
#ifndef TLB_CONV1_ROWS2
#define TLB_CONV1_ROWS2 1  // fast conv1: 1 = two rows x 8 columns per lane, 2 = two rows x 4, 0 = row strips
#endif
#ifndef TLB_V15_C1_LANES
#define TLB_V15_C1_LANES 0
#endif
#ifndef TLB_EXACT_GK2_SPLIT
#define TLB_EXACT_GK2_SPLIT 224  // EXACT V15: ordered g_k2 chains beside backin (the rest beside C1)
#endif
#ifndef TLB_GK2R_SPLIT
#define TLB_GK2R_SPLIT 96  // row-form g_k2 lanes beside backin, the rest beside the C1 gradient (A/B: 64-160 best)
#endif
#ifndef TLB_BACKIN_KUNROLL
#define TLB_BACKIN_KUNROLL 3
#endif
constexpr int kBackinKUnroll = TLB_BACKIN_KUNROLL;
#ifndef TLB_GK2R_YUNROLL
#define TLB_GK2R_YUNROLL 2
#endif
constexpr int kGk2rYUnroll = TLB_GK2R_YUNROLL;  // gk2_rows tap-row loop unroll (A/B switch)
#ifndef TLB_C1G2_UNROLL
#define TLB_C1G2_UNROLL 1
#endif
constexpr int kC1g2Unroll = TLB_C1G2_UNROLL;  // conv1_back_fast_group2 tap-row loop unroll (A/B switch)

struct Smem {
  float* P;    // parameters [3904]
  float* Kp;   // k2 re-laid out with each (i,c,ky) row of 5 padded to 8: [12][6][5][8]
  float* img;  // two image buffers of kImg floats (double-buffered TMA ring)
  float* sh;   // image shifted by v (0..4): sh[v][y][x] = I[y][x+v], x < 24: [5][28][24]
  float* c1;   // c1, then dz1 in place        } c1|s1|c2|s2 contiguous (5,280 floats): reused as
  float* s1;   //                               } the staging buffer of the batch reduction
  float* c2;
  float* s2;
  float* out;
  float* dz;
  float* dzp;  // dz2 zero-padded by 4 on every side: [12][16][16] (strided, see dzp_at); border stays 0
  float* fcp;  // EXACT FC products [10][192]
  float* red;  // fast C1 weight-gradient row partials [144][26]
  float* G;    // fast per-CTA gradient accumulator [3904]
  float* term; // backin per-kernel terms b_i(c, p, q): [12][6][12][12]
  int* lab;    // labels of the two image buffers (train kernels; aliases out[12..13], unused by the FC)
  uint64_t* tab;
  uint64_t* bar;
  int64_t* jidx;  // dataset index of the job in each image buffer (byte ingestion write-back)
  uint8_t* px;    // [2][784] pixel bytes of the two image buffers (byte ingestion)
  int* bst;       // [2] 1 = the job in this buffer arrives as bytes (set by the issuer)
  unsigned long long* tr;  // optional per-stage clock64 trace (CTA 0 only), nullptr otherwise
};

// Profiling hook: stamp the SM clock after a stage (thread 0 of a traced CTA).  BAR.SYNC on sm_100
// blocks lazily (at the next barrier-protected access), so a shared load feeds the clock read to
// make the stamp land after the barrier really released.
__device__ __forceinline__ void mark(const Smem& s, int slot) {
  if (s.tr && threadIdx.x == 0) {
    const unsigned int v = *reinterpret_cast<volatile const unsigned int*>(s.P);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) : "r"(v) : "memory");
    s.tr[slot] = t;
  }
}

constexpr int kKp = 12 * 6 * 5 * 8;
// Bank-conflict-free strides (in float4 units the plane/kernel strides are odd mod 8):
constexpr int kShPlane = 28 * 24 + 4;   // shifted-image plane (v) stride
constexpr int kSh = 5 * kShPlane + 4;   // (+4 keeps the next buffer 16-B aligned)
constexpr int kDzpRow = 24;             // padded dz2 row: 16 used columns (6 float4: neighbouring
                                        // backin tiles land in different bank groups)
constexpr int kDzpK = 16 * kDzpRow + 4; // padded dz2 kernel (i) stride
constexpr int kDzp = 12 * kDzpK;
constexpr int kRed = 144 * 26;          // fast C1 weight-gradient row partials
constexpr int kTerm = 12 * 864;         // backin per-kernel terms

__device__ __forceinline__ int dzp_at(int i, int R, int col) { return i * kDzpK + R * kDzpRow + col; }
// Fast mode (TLB_GK2K): a second copy of dz2 as kernel pairs (dz2[ip], dz2[ip+6]) [6][8][8] float2 for the
// packed-pair g_k2, in the Kp slot (from float 1800); rows padded to 20 floats and pair planes to
// 164 (both 4 mod 32 banks in 16-byte units: a warp's row loads of different rows / pairs do not collide).
constexpr int kDzkOff = 1800, kDzkRow = 20, kDzkPlane = 8 * kDzkRow + 4;
static_assert(kDzkOff + 6 * kDzkPlane <= kKp, "dz2 pairs fit the Kp slot");
__device__ __forceinline__ int dzk_at(int ip, int y, int x) { return kDzkOff + ip * kDzkPlane + y * kDzkRow + 2 * x; }
// c1 / dz1 channel planes padded 576 -> 580 floats: the six channel rows of one y start in six different
// bank groups (580 mod 32 = 4), so the C1 weight-gradient lanes read them conflict-free.
constexpr int kC1Plane = 580;
constexpr int kC1Floats = 6 * kC1Plane;
__device__ __forceinline__ int c1_at(int i, int y, int x) { return i * kC1Plane + y * 24 + x; }
__device__ __forceinline__ int sh_at(int v, int y) { return v * kShPlane + y * 24; }
// Shared-memory layout: a prefix every kernel uses, then a mode tail -- fast kernels: the C1 row partials
// and the per-CTA gradient accumulator; EXACT kernels: the shifted image copies and the FC products (the
// two tails alias: no kernel uses both) -- then the clustered kernel's DSMEM receive buffer (`term`).
// Kernels allocate only what they touch, so both the fast and the EXACT flat kernels fit two CTAs per SM.
constexpr int kPrefixFloats = kPStride + kKp + 2 * kImg + kC1Floats + 864 + 768 + 192 + 16 + 16 + kDzp;
// + 2 x 784 B pixel-byte staging and 2 int64 job indices (byte ingestion, see TrainArgs::pixels)
constexpr size_t kPrefixBytes =
    ((sizeof(float) * kPrefixFloats + 34 * sizeof(uint64_t) + 2 * sizeof(int64_t) + 2 * kImg + 2 * sizeof(int)) + 15) /
    16 * 16;
constexpr int kFastTailFloats = kRed + kPStride;
constexpr int kExactTailFloats = kSh + 1920;
constexpr int kTailFloats = kFastTailFloats > kExactTailFloats ? kFastTailFloats : kExactTailFloats;
constexpr size_t kSmemFastBytes = kPrefixBytes + sizeof(float) * kFastTailFloats;
constexpr size_t kSmemExactBytes = kPrefixBytes + sizeof(float) * kExactTailFloats;
constexpr size_t kSmemBytes = kPrefixBytes + sizeof(float) * (kTailFloats + kTerm);  // clustered kernel
template <bool EXACT>
constexpr size_t smem_bytes_for() { return EXACT ? kSmemExactBytes : kSmemFastBytes; }

// The CTA's dynamic shared memory (one declaration for every kernel and stage).
extern __shared__ __align__(128) float tlb_smem[];

__device__ __forceinline__ Smem carve_smem(float* base) {
  Smem s;
  float* p = base;
  s.P = p; p += kPStride;
  s.Kp = p; p += kKp;
  s.img = p; p += 2 * kImg;
  s.c1 = p; p += kC1Floats;
  s.s1 = p; p += 864;
  s.c2 = p; p += 768;
  s.s2 = p; p += 192;
  s.out = p;
  s.lab = reinterpret_cast<int*>(p + 12);
  p += 16;
  s.dz = p; p += 16;
  s.dzp = p; p += kDzp;
  s.tab = reinterpret_cast<uint64_t*>(p);
  s.bar = s.tab + 32;
  s.jidx = reinterpret_cast<int64_t*>(s.bar + 2);
  s.px = reinterpret_cast<uint8_t*>(s.jidx + 2);  // 16-byte aligned (the prefix floats are a 16-B multiple)
  s.bst = reinterpret_cast<int*>(s.px + 2 * kImg);
  float* const tail = base + kPrefixBytes / sizeof(float);
  s.red = tail;                   // fast tail
  s.G = tail + kRed;
  s.sh = tail;                    // EXACT tail (aliases the fast tail)
  s.fcp = tail + kSh;
  s.term = tail + kTailFloats;    // clustered-kernel tail
  s.tr = nullptr;
  return s;
}

__device__ __forceinline__ Smem smem_view() { return carve_smem(tlb_smem); }


// One-time per-CTA setup: exp2 table, zero padding of dz2, image mbarriers.
__device__ __forceinline__ void smem_setup(const Smem& s) {
  if (threadIdx.x < 32) s.tab[threadIdx.x] = exp_tab_entry(threadIdx.x);
  for (int i = threadIdx.x; i < kDzp; i += blockDim.x) s.dzp[i] = 0.0f;
  if (threadIdx.x == 0) {
    mbar_init(&s.bar[0], 1);
    mbar_init(&s.bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
}

// Issue the TMA bulk copy of one 28x28 fp32 image (3,136 B) into buffer `buf` (thread 0 only).
__device__ __forceinline__ void issue_image(const Smem& s, int buf, const float* src) {
  fence_proxy_async_smem();  // order earlier generic reads of this buffer before the async write
  mbar_arrive_expect_tx(&s.bar[buf], kImg * sizeof(float));
  tma_load_1d(s.img + buf * kImg, src, kImg * sizeof(float), &s.bar[buf]);
}

// Parameters (3,898 floats, padded) global -> shared, then (EXACT / scalar conv2) the padded k2 copy.
// __ldcg: other CTAs rewrote them in the previous step's SGD phase, so bypass L1.  Ends with __syncthreads.
template <bool EXACT = true>
__device__ __forceinline__ void load_params(const Smem& s, const float* params) {
  const float4* src = reinterpret_cast<const float4*>(params);
  float4* dst = reinterpret_cast<float4*>(s.P);
  constexpr int kBatch = 2;  // every load in flight before the first shared store
  for (int base = threadIdx.x; base < kPStride / 4; base += kBatch * blockDim.x) {
    float4 v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (base + u * (int)blockDim.x < kPStride / 4) v[u] = __ldcg(src + base + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (base + u * (int)blockDim.x < kPStride / 4) dst[base + u * blockDim.x] = v[u];
  }
  __syncthreads();
  if constexpr (EXACT || !TLB_PAIR) {  // (the pair conv2 reads its weight pairs straight from P)
    for (int idx = threadIdx.x; idx < kKp; idx += blockDim.x) {
      const int row = idx >> 3, k = idx & 7;
      s.Kp[idx] = k < 5 ? s.P[kK2 + row * 5 + k] : 0.0f;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float target_of(int i, int label, const float* y) {
  return y ? y[i] : (i == label ? 1.0f : 0.0f);  // mnist::one_hot (mnist.cpp:161-167)
}

// ---------------------------------------------------------------------------------------------
// Forward stages (net::forward, network.cpp:81-95)
// ---------------------------------------------------------------------------------------------

// sh[v][y][x] = I[y][x+v] (x < 24): the EXACT C1 weight gradient reads each shifted row with two
// aligned 128-bit loads instead of 24 scalar ones.
__device__ __forceinline__ void build_shifted(const Smem& s, const float* img, int t0, int nt) {
  for (int q = t0; q < 5 * 28 * 6; q += nt) {  // 5 planes x 28 rows x 6 float4
    const int v = q / 168, rem = q - v * 168, y = rem / 6, x4 = 4 * (rem - y * 6);
    const float* srow = img + y * 28 + x4 + v;
    *reinterpret_cast<float4*>(s.sh + sh_at(v, y) + x4) = make_float4(srow[0], srow[1], srow[2], srow[3]);
  }
}

// C1: mconv(I,k1,b1) -> sigmoid -> avgpool.  Item = (channel i, conv row y, 8-wide strip xs); the
// two rows of a pooling window sit on adjacent lanes and meet through a shuffle.  Per output: taps
// (ky,kx) row-major (nn.cpp:28-33), then + b1[i] (nn.cpp:123); pool ((p00+p01)+p10)+p11, *0.25f.
// Warps 13.5..15 meanwhile build the v-shifted image copies used by the C1 weight gradient.
// Fast conv1 variant (TLB_CONV1_ROWS2): lane = (channel i, pooled row py, 8-column strip xs) computes
// both conv rows 2py, 2py+1 (16 outputs): the six image rows it loads and the 25 weights serve both
// rows, and the 2x2 pooling windows are lane-local (no shuffle).  216 lanes.
template <int W>  // output columns per lane: 8 (216 lanes) or 4 (432 lanes)
__device__ __forceinline__ void stage_conv1_rows2(const Smem& s, const float* img) {
  constexpr int kStrips = 24 / W, kItems = 6 * 12 * kStrips;
  for (int it = threadIdx.x; it < (kItems + 31) / 32 * 32; it += blockDim.x) {
    if (it >= kItems) continue;
    const int i = it / (12 * kStrips), rem = it - i * 12 * kStrips, py = rem / kStrips, xs = rem - py * kStrips;
    const int y0 = 2 * py, x0 = W * xs;
    const float* k = s.P + kK1 + i * 25;
    float a[2][W];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int o = 0; o < W; ++o) a[r][o] = 0.0f;
#pragma unroll
    for (int rr = 0; rr < 6; ++rr) {  // image row y0 + rr feeds conv row r with ky = rr - r
      const float4* src = reinterpret_cast<const float4*>(img + (y0 + rr) * 28 + x0);
      float in[W + 4];
#pragma unroll
      for (int q = 0; q < (W + 4) / 4; ++q) {
        const float4 v = src[q];
        in[4 * q] = v.x; in[4 * q + 1] = v.y; in[4 * q + 2] = v.z; in[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int ky = rr - r;
        if (ky < 0 || ky > 4) continue;
#pragma unroll
        for (int kx = 0; kx < 5; ++kx) {
          const float w = k[ky * 5 + kx];
#pragma unroll
          for (int o = 0; o < W; ++o) a[r][o] = __fmaf_rn(in[o + kx], w, a[r][o]);
        }
      }
    }
    const float b = s.P[kB1 + i];
    float t[2][W];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int o = 0; o < W; ++o) t[r][o] = sigmoid_m<false>(fadd(a[r][o], b), s.tab);
      float4* d = reinterpret_cast<float4*>(s.c1 + c1_at(i, y0 + r, x0));
#pragma unroll
      for (int q = 0; q < W / 4; ++q) d[q] = make_float4(t[r][4 * q], t[r][4 * q + 1], t[r][4 * q + 2], t[r][4 * q + 3]);
    }
    float pv[W / 2];
#pragma unroll
    for (int px = 0; px < W / 2; ++px)  // avgpool (nn.cpp:144): ((p00 + p01) + p10) + p11, then * 0.25f
      pv[px] = fmul(fadd(fadd(fadd(t[0][2 * px], t[0][2 * px + 1]), t[1][2 * px]), t[1][2 * px + 1]), 0.25f);
    float* sp = s.s1 + (i * 12 + py) * 12 + (W / 2) * xs;
    if constexpr (W == 8) *reinterpret_cast<float4*>(sp) = make_float4(pv[0], pv[1], pv[2], pv[3]);
    else *reinterpret_cast<float2*>(sp) = make_float2(pv[0], pv[1]);
  }
}

// ---------------------------------------------------------------------------------------------
// Packed-pair fast forward (TLB_PAIR): the two forward contractions run on packed FP32 pairs (__ffma2_rn,
// SASS FFMA2: the FP32 rate of FFMA at half the issued instructions -- measured peak 74.1 vs 72.4 TFLOP/s,
// profiles/r2/ffma2_peak_r2k.json), one operand a broadcast scalar:
//   conv1 : pixel (broadcast) x (k1[c], k1[c+3])            -> (c1[c], c1[c+3])
//   conv2 : s1 (broadcast) x (k2[i][c], k2[i+6][c])         -> (out[i], out[i+6])
// The conv2 weight pair is two scalar loads from P (k2[i] and k2[i+6], 900 floats apart): a float2 copy
// rebuilt after every exchange cost more than the extra loads (profiles/r2/b_*_c2d1.json); every
// activation keeps its canonical layout, so the backward stages are the scalar ones.  (Pair
// layouts for the backward contractions were measured slower at one image per SM: their weight-pair and
// dz2-pair loads cost more shared-memory wavefronts than the halved FFMA issue saves; profiles/README.md.)
// Fast-mode arithmetic (FFMA, fixed summation trees; within the north-star 1e-4); EXACT keeps the scalar
// ordered stages.
__device__ __forceinline__ float2 bcast2(float v) { return make_float2(v, v); }

// conv1 pair lane = (channel pair ip, pooled row py, 4-column strip xs), 216 lanes: the two conv rows x 4
// columns x 2 channels (8 FFMA2 accumulators) over the 25 taps -- 200 FFMA2 for 400 multiply-adds -- with
// the pixel as the broadcast operand and the (k1[ip], k1[ip+3]) weight pair in registers; logistic, c1
// pairs, 2x2 pool in registers -> s1 pairs.
__device__ __forceinline__ void stage_conv1_pair(const Smem& s, const float* img) {
  const int it = threadIdx.x;
  if (it >= 216) return;
  const int ip = it / 72, rem = it - ip * 72, py = rem / 6, xs = rem - py * 6;
  const int y0 = 2 * py, x0 = 4 * xs;
  float2 w[25];
#pragma unroll
  for (int t = 0; t < 25; ++t) w[t] = make_float2(s.P[kK1 + ip * 25 + t], s.P[kK1 + (ip + 3) * 25 + t]);
  float2 a[2][4];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int o = 0; o < 4; ++o) a[r][o] = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int rr = 0; rr < 6; ++rr) {  // image row y0 + rr feeds conv row r with ky = rr - r
    const float4* src = reinterpret_cast<const float4*>(img + (y0 + rr) * 28 + x0);
    const float4 v0 = src[0], v1 = src[1];
    const float in[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int ky = rr - r;
      if (ky < 0 || ky > 4) continue;
#pragma unroll
      for (int kx = 0; kx < 5; ++kx)
#pragma unroll
        for (int o = 0; o < 4; ++o) a[r][o] = __ffma2_rn(bcast2(in[o + kx]), w[ky * 5 + kx], a[r][o]);
    }
  }
  const float bx = s.P[kB1 + ip], by = s.P[kB1 + ip + 3];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
#pragma unroll
    for (int o = 0; o < 4; ++o)
      a[r][o] = make_float2(sigmoid_m<false>(fadd(a[r][o].x, bx), s.tab), sigmoid_m<false>(fadd(a[r][o].y, by), s.tab));
    *reinterpret_cast<float4*>(s.c1 + c1_at(ip, y0 + r, x0)) = make_float4(a[r][0].x, a[r][1].x, a[r][2].x, a[r][3].x);
    *reinterpret_cast<float4*>(s.c1 + c1_at(ip + 3, y0 + r, x0)) = make_float4(a[r][0].y, a[r][1].y, a[r][2].y, a[r][3].y);
  }
  float2 pv[2];
#pragma unroll
  for (int px = 0; px < 2; ++px) {  // avgpool (nn.cpp:144): ((p00 + p01) + p10) + p11, then * 0.25f
    const float2 p00 = a[0][2 * px], p01 = a[0][2 * px + 1], p10 = a[1][2 * px], p11 = a[1][2 * px + 1];
    pv[px] = make_float2(fmul(fadd(fadd(fadd(p00.x, p01.x), p10.x), p11.x), 0.25f),
                         fmul(fadd(fadd(fadd(p00.y, p01.y), p10.y), p11.y), 0.25f));
  }
  // s1 stays in the canonical [6][12][12] layout (conv2 and g_k2 broadcast it against kernel pairs)
  *reinterpret_cast<float2*>(s.s1 + (ip * 12 + py) * 12 + 2 * xs) = make_float2(pv[0].x, pv[1].x);
  *reinterpret_cast<float2*>(s.s1 + ((ip + 3) * 12 + py) * 12 + 2 * xs) = make_float2(pv[0].y, pv[1].y);
}

// conv2 on kernel pairs (i, i+6): lane = (channel half h, column block xh, pool row r, kernel pair ip,
// pooled row py), h fastest.  The s1 row value is the broadcast operand, (k2[i][c], k2[i+6][c]) the weight
// pair; COLS columns of conv row y = 2py + r over the lane's 3 channels (15 x 5 x COLS FFMA2), the two
// channel halves joined by a shuffle (lane ^ 1), lane h finishes kernel ip + 6h: sigmoid, c2, and the 2x2
// pool with the partner row (lane ^ (2 * 8 / COLS)).  COLS = 8: 96 lanes; COLS = 4: 192 lanes.
template <int COLS>
__device__ __forceinline__ void stage_conv2_kpair(const Smem& s) {
  constexpr int XB = 8 / COLS, kLanes = 96 * XB;
  const int it = threadIdx.x;
  if (it >= kLanes) return;
  const int h = it & 1, xh = (it >> 1) % XB, r = (it / (2 * XB)) & 1, rest = it / (4 * XB);
  const int ip = rest % 6, py = rest / 6, y = 2 * py + r, x0 = COLS * xh;
  const float* k2a = s.P + kK2 + ip * 150;  // k2[ip] (and k2[ip + 6], 900 floats later)
  float2 acc[COLS];
#pragma unroll
  for (int o = 0; o < COLS; ++o) acc[o] = make_float2(0.0f, 0.0f);
#pragma unroll 1
  for (int c = 3 * h; c < 3 * h + 3; ++c) {
#pragma unroll
    for (int ky = 0; ky < 5; ++ky) {
      const float4* src = reinterpret_cast<const float4*>(s.s1 + (c * 12 + y + ky) * 12 + x0);
      float in[COLS + 4];
#pragma unroll
      for (int q = 0; q < (COLS + 4) / 4; ++q) {
        const float4 v = src[q];
        in[4 * q] = v.x; in[4 * q + 1] = v.y; in[4 * q + 2] = v.z; in[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int kx = 0; kx < 5; ++kx) {
        const float2 w = make_float2(k2a[c * 25 + ky * 5 + kx], k2a[900 + c * 25 + ky * 5 + kx]);
#pragma unroll
        for (int o = 0; o < COLS; ++o) acc[o] = __ffma2_rn(bcast2(in[o + kx]), w, acc[o]);
      }
    }
  }
  float t[COLS], u[COLS];
  const int i = ip + 6 * h;
  const float b = s.P[kB2 + i];
#pragma unroll
  for (int o = 0; o < COLS; ++o) {
    const float ox = acc[o].x + __shfl_xor_sync(0xffffffffu, acc[o].x, 1);
    const float oy = acc[o].y + __shfl_xor_sync(0xffffffffu, acc[o].y, 1);
    t[o] = sigmoid_m<false>(fadd(h ? oy : ox, b), s.tab);
  }
#pragma unroll
  for (int o = 0; o < COLS; ++o) u[o] = __shfl_xor_sync(0xffffffffu, t[o], 2 * XB);  // conv row y ^ 1
  float* c2 = s.c2 + (i * 8 + y) * 8 + x0;
#pragma unroll
  for (int q = 0; q < COLS / 4; ++q)
    reinterpret_cast<float4*>(c2)[q] = make_float4(t[4 * q], t[4 * q + 1], t[4 * q + 2], t[4 * q + 3]);
  if (r == 0) {  // avgpool (nn.cpp:144): ((p00 + p01) + p10) + p11, then * 0.25f
    float pv[COLS / 2];
#pragma unroll
    for (int px = 0; px < COLS / 2; ++px)
      pv[px] = fmul(fadd(fadd(fadd(t[2 * px], t[2 * px + 1]), u[2 * px]), u[2 * px + 1]), 0.25f);
    float* s2 = s.s2 + (i * 4 + py) * 4 + (COLS / 2) * xh;
    if constexpr (COLS == 8) *reinterpret_cast<float4*>(s2) = make_float4(pv[0], pv[1], pv[2], pv[3]);
    else *reinterpret_cast<float2*>(s2) = make_float2(pv[0], pv[1]);
  }
}

template <bool EXACT>
__device__ __forceinline__ void stage_conv1(const Smem& s, const float* img) {
  if constexpr (!EXACT && TLB_PAIR) {
    stage_conv1_pair(s, img);
    return;
  }
  if constexpr (!EXACT && TLB_CONV1_ROWS2) {
    stage_conv1_rows2<TLB_CONV1_ROWS2 == 2 ? 4 : 8>(s, img);
    return;
  }
  // 448 item lanes (14 full warps; items >= 432 are padding lanes, valid = false); with fewer threads
  // than items the lanes loop (whole warps per round, so the pool shuffle stays warp-uniform).
  for (int it = threadIdx.x; it < 448; it += blockDim.x) {
    const bool valid = it < 432;
    const int pair = (valid ? it : 0) >> 1, r = it & 1;
    const int i = pair / 36, rem = pair - i * 36, py = rem / 3, xs = rem - py * 3;
    const int y = 2 * py + r, x0 = 8 * xs;
    const float* k = s.P + kK1 + i * 25;
    float a[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) a[o] = 0.0f;
#pragma unroll
    for (int ky = 0; ky < 5; ++ky) {
      const float4* src = reinterpret_cast<const float4*>(img + (y + ky) * 28 + x0);
      const float4 v0 = src[0], v1 = src[1], v2 = src[2];
      const float in[12] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w, v2.x, v2.y, v2.z, v2.w};
#pragma unroll
      for (int kx = 0; kx < 5; ++kx) {
        const float w = k[ky * 5 + kx];
#pragma unroll
        for (int o = 0; o < 8; ++o) a[o] = mac<EXACT>(a[o], in[o + kx], w);
      }
    }
    const float b = s.P[kB1 + i];
    float t[8], u[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) t[o] = sigmoid_m<EXACT>(fadd(a[o], b), s.tab);
#pragma unroll
    for (int o = 0; o < 8; ++o) u[o] = __shfl_xor_sync(0xffffffffu, t[o], 1);
    if (valid) {
      float4* d = reinterpret_cast<float4*>(s.c1 + c1_at(i, y, x0));
      d[0] = make_float4(t[0], t[1], t[2], t[3]);
      d[1] = make_float4(t[4], t[5], t[6], t[7]);
      float pv[2];
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2) {
        const int px = 2 * r + k2;
        const float t00 = r ? u[2 * px] : t[2 * px], t01 = r ? u[2 * px + 1] : t[2 * px + 1];
        const float t10 = r ? t[2 * px] : u[2 * px], t11 = r ? t[2 * px + 1] : u[2 * px + 1];
        pv[k2] = fmul(fadd(fadd(fadd(t00, t01), t10), t11), 0.25f);
      }
      *reinterpret_cast<float2*>(s.s1 + (i * 12 + py) * 12 + 4 * xs + 2 * r) = make_float2(pv[0], pv[1]);
    }
  }
  if constexpr (EXACT) {  // warps 14-15 of a 512-thread CTA, else every thread after its conv1 items
    if (blockDim.x > 448) {
      if (threadIdx.x >= 448) build_shifted(s, img, threadIdx.x - 448, blockDim.x - 448);
    } else {
      build_shifted(s, img, threadIdx.x, blockDim.x);
    }
  }
}

// C2: mconv(s1,k2,b2) -> sigmoid -> avgpool.  One lane per output row (kernel i, row y, 8 columns):
// per (c, ky) a lane loads the 12-float s1 row segment and the 5 weights and does 40 multiply-adds.
// Per output the 150 taps run (c, ky, kx) row-major (nn.cpp:14-33).  Fast mode splits the channel
// sum over a lane pair (c < 3, c >= 3) and combines with a shuffle; EXACT keeps one ordered chain.
// The two rows of each pooling window are neighbouring lane groups and meet through a shuffle.
// WP: weights read as scalars from P instead of the padded Kp copy (the clustered kernel keeps no Kp).
template <bool EXACT, bool WP = false>
__device__ __forceinline__ void stage_conv2_rows(const Smem& s) {
  constexpr int kSplit = EXACT ? 1 : 2;
  const int it = threadIdx.x;
  if (it >= 96 * kSplit) return;  // 3 (EXACT) / 6 (fast) whole warps
  const int item = it / kSplit, part = it % kSplit;
  const int i = item >> 3, y = item & 7;
  float acc[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) acc[o] = 0.0f;
  const int c0 = part * (6 / kSplit), c1 = c0 + 6 / kSplit;
#pragma unroll 1
  for (int c = c0; c < c1; ++c) {
#pragma unroll
    for (int ky = 0; ky < 5; ++ky) {
      const float4* src = reinterpret_cast<const float4*>(s.s1 + (c * 12 + y + ky) * 12);
      const float4 v0 = src[0], v1 = src[1], v2 = src[2];
      const float in[12] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w, v2.x, v2.y, v2.z, v2.w};
      float w[5];
      if constexpr (WP) {
        const float* wp = s.P + kK2 + ((i * 6 + c) * 5 + ky) * 5;
#pragma unroll
        for (int kx = 0; kx < 5; ++kx) w[kx] = wp[kx];
      } else {
        const float4* wp = reinterpret_cast<const float4*>(s.Kp + ((i * 6 + c) * 5 + ky) * 8);
        const float4 w0 = wp[0], w1 = wp[1];
        w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w; w[4] = w1.x;
      }
#pragma unroll
      for (int kx = 0; kx < 5; ++kx)
#pragma unroll
        for (int o = 0; o < 8; ++o) acc[o] = mac<EXACT>(acc[o], in[o + kx], w[kx]);
    }
  }
  if constexpr (!EXACT) {
#pragma unroll
    for (int o = 0; o < 8; ++o) acc[o] += __shfl_xor_sync(0xffffffffu, acc[o], 1);
  }
  const float b = s.P[kB2 + i];
  float t[8], u[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) t[o] = sigmoid_m<EXACT>(fadd(acc[o], b), s.tab);
#pragma unroll
  for (int o = 0; o < 8; ++o) u[o] = __shfl_xor_sync(0xffffffffu, t[o], kSplit);  // row y ^ 1
  if (part) return;
  float4* d = reinterpret_cast<float4*>(s.c2 + (i * 8 + y) * 8);
  d[0] = make_float4(t[0], t[1], t[2], t[3]);
  d[1] = make_float4(t[4], t[5], t[6], t[7]);
  if ((y & 1) == 0) {  // avgpool (nn.cpp:144): ((p00 + p01) + p10) + p11, then * 0.25f
    float pv[4];
#pragma unroll
    for (int px = 0; px < 4; ++px)
      pv[px] = fmul(fadd(fadd(fadd(t[2 * px], t[2 * px + 1]), u[2 * px]), u[2 * px + 1]), 0.25f);
    *reinterpret_cast<float4*>(s.s2 + (i * 4 + (y >> 1)) * 4) = make_float4(pv[0], pv[1], pv[2], pv[3]);
  }
}

// C2 variant with 4-output lanes (kernel i, row y, half-row xh): twice the lanes of stage_conv2_rows,
// so more warps hide the shared-memory latency.  Pool partner (row y^1) is lane ^ (2*kSplit).
template <bool EXACT>
__device__ __forceinline__ void stage_conv2_halves(const Smem& s) {
  constexpr int kSplit = EXACT ? 1 : 2;
  const int it = threadIdx.x;
  if (it >= 192 * kSplit) return;  // 6 (EXACT) / 12 (fast) whole warps
  const int item = it / kSplit, part = it % kSplit;
  const int xh = item & 1, y = (item >> 1) & 7, i = item >> 4;
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  const int c0 = part * (6 / kSplit), c1 = c0 + 6 / kSplit;
#pragma unroll 1
  for (int c = c0; c < c1; ++c) {
#pragma unroll
    for (int ky = 0; ky < 5; ++ky) {
      const float4* src = reinterpret_cast<const float4*>(s.s1 + (c * 12 + y + ky) * 12 + 4 * xh);
      const float4 v0 = src[0], v1 = src[1];
      const float in[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      const float4* wp = reinterpret_cast<const float4*>(s.Kp + ((i * 6 + c) * 5 + ky) * 8);
      const float4 w0 = wp[0], w1 = wp[1];
      const float w[5] = {w0.x, w0.y, w0.z, w0.w, w1.x};
#pragma unroll
      for (int kx = 0; kx < 5; ++kx)
#pragma unroll
        for (int o = 0; o < 4; ++o) acc[o] = mac<EXACT>(acc[o], in[o + kx], w[kx]);
    }
  }
  if constexpr (!EXACT) {
#pragma unroll
    for (int o = 0; o < 4; ++o) acc[o] += __shfl_xor_sync(0xffffffffu, acc[o], 1);
  }
  const float b = s.P[kB2 + i];
  float t[4], u[4];
#pragma unroll
  for (int o = 0; o < 4; ++o) t[o] = sigmoid_m<EXACT>(fadd(acc[o], b), s.tab);
#pragma unroll
  for (int o = 0; o < 4; ++o) u[o] = __shfl_xor_sync(0xffffffffu, t[o], 2 * kSplit);  // row y ^ 1
  if (part) return;
  *reinterpret_cast<float4*>(s.c2 + (i * 8 + y) * 8 + 4 * xh) = make_float4(t[0], t[1], t[2], t[3]);
  if ((y & 1) == 0) {  // avgpool (nn.cpp:144): ((p00 + p01) + p10) + p11, then * 0.25f
    const float p0 = fmul(fadd(fadd(fadd(t[0], t[1]), u[0]), u[1]), 0.25f);
    const float p1 = fmul(fadd(fadd(fadd(t[2], t[3]), u[2]), u[3]), 0.25f);
    *reinterpret_cast<float2*>(s.s2 + (i * 4 + (y >> 1)) * 4 + 2 * xh) = make_float2(p0, p1);
  }
}

template <bool EXACT, int V>
__device__ __forceinline__ void stage_conv2(const Smem& s) {
  if constexpr (!EXACT && TLB_PAIR) stage_conv2_kpair<TLB_C2K>(s);
  else if constexpr (V == 0) stage_conv2_halves<EXACT>(s);
  else if constexpr (V == 2) stage_conv2_rows<EXACT, true>(s);
  else stage_conv2_rows<EXACT>(s);
}

// FC: out[i] = sigmoid(sum_j s2[j]*fc[i][j] + b[i]); also dz = backsigmoid(out - y, out)
// (network.cpp:146-152, nn.cpp:131-133).  EXACT: all 1,920 products in parallel, then one ordered
// 192-term chain per output.  Fast: one warp per output with a shuffle tree.
template <bool EXACT>
__device__ __forceinline__ void stage_fc(const Smem& s, int label, const float* y, bool want_dz) {
  if constexpr (EXACT) {
    for (int idx = threadIdx.x; idx < 1920; idx += blockDim.x)
      s.fcp[idx] = fmul(s.s2[idx % 192], s.P[kFC + idx]);
    __syncthreads();
    if (threadIdx.x < 10) {
      const int i = threadIdx.x;
      const float4* p4 = reinterpret_cast<const float4*>(s.fcp + i * 192);
      float acc = 0.0f;
#pragma unroll 8
      for (int j = 0; j < 48; ++j) {
        const float4 v = p4[j];
        acc = fadd(fadd(fadd(fadd(acc, v.x), v.y), v.z), v.w);
      }
      const float o = sigmoid_m<true>(fadd(acc, s.P[kB + i]), s.tab);
      s.out[i] = o;
      if (want_dz) s.dz[i] = fmul(fmul(fsub(o, target_of(i, label, y)), o), fsub(1.0f, o));
    }
  } else {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = warp; i < 10; i += blockDim.x >> 5) {
      const float* w = s.P + kFC + i * 192;
      float acc = 0.0f;
#pragma unroll
      for (int k = 0; k < 6; ++k) acc = __fmaf_rn(s.s2[lane + 32 * k], w[lane + 32 * k], acc);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) {
        const float o = sigmoid_m<false>(fadd(acc, s.P[kB + i]), s.tab);
        s.out[i] = o;
        if (want_dz) s.dz[i] = fmul(fmul(fsub(o, target_of(i, label, y)), o), fsub(1.0f, o));
      }
    }
  }
}

// net::loss (network.cpp:97-109): 0.5f * sum_i (y_i - out_i)^2, i in order.
__device__ __forceinline__ float example_loss(const Smem& s, int label, const float* y) {
  float acc = 0.0f;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const float d = fsub(target_of(i, label, y), s.out[i]);
    acc = fadd(acc, fmul(d, d));
  }
  return fmul(0.5f, acc);
}

// ---------------------------------------------------------------------------------------------
// Backward stages (net::backward, network.cpp:145-169)
// ---------------------------------------------------------------------------------------------

// Gradient sink: either the per-example row in global memory (reference cell, network.cpp:232)
// or the CTA's running accumulator in shared memory (fast mode, example order within the CTA).
template <bool ACCUM>
__device__ __forceinline__ void put(const Smem& s, float* row, int idx, float v) {
  if constexpr (ACCUM) s.G[idx] = fadd(s.G[idx], v);
  else row[idx] = v;
}

// FC backward: g_fc[i][j] = 0 + s2[j]*dz[i]; g_b = 0 + dz; d_s2[j] = sum_i fc[i][j]*dz[i]
// (backin with singleton error, nn.cpp:193-217, summed over i as network.cpp:135-138), then
// backavgpool (nn.cpp:148-158) and backsigmoid through c2 -> dz2 (into the padded buffer).
// d_s2[j] = sum_i fc[i][j]*dz[i] (FFMA), then backavgpool + backsigmoid through c2 -> dz2 (fast mode).
__device__ __forceinline__ void fc_back_dz2(const Smem& s, int j) {
  float ds = 0.0f;
#pragma unroll
  for (int i = 0; i < 10; ++i) ds = mac<false>(ds, s.P[kFC + i * 192 + j], s.dz[i]);
  const float dc = fmul(ds, 0.25f);
  const int c = j >> 4, py = (j >> 2) & 3, px = j & 3;
#pragma unroll
  for (int dy = 0; dy < 2; ++dy)
#pragma unroll
    for (int dx = 0; dx < 2; ++dx) {
      const int yy = 2 * py + dy, xx = 2 * px + dx;
      const float o = s.c2[(c * 8 + yy) * 8 + xx];
      const float d = fmul(fmul(dc, o), fsub(1.0f, o));
      s.dzp[dzp_at(c, yy + 4, xx + 4)] = d;
      if constexpr (TLB_PAIR && TLB_GK2K) s.Kp[dzk_at(c % 6, yy, xx) + c / 6] = d;
    }
}

template <bool EXACT, bool ACCUM>
__device__ __forceinline__ void stage_fc_back(const Smem& s, float* row) {
  if constexpr (!EXACT && ACCUM) {
    // Fast accumulating kernels: lanes 0-191 run the d_s2 -> dz2 chain while lanes 192+ add the FC
    // gradient into G four columns at a time (480 float4 entries + 10 biases, FFMA).
    for (int t = threadIdx.x; t < 192 + 320; t += blockDim.x) {
      if (t < 192) {
        fc_back_dz2(s, t);
      } else {
        for (int q = t - 192; q < 490; q += 320) {
          if (q < 480) {
            const int i = q / 48, j4 = q - i * 48;
            const float4 sv = *reinterpret_cast<const float4*>(s.s2 + 4 * j4);
            const float d = s.dz[i];
            float4* g = reinterpret_cast<float4*>(s.G + kFC + 4 * q);
            float4 gv = *g;
            gv.x = __fmaf_rn(sv.x, d, gv.x);
            gv.y = __fmaf_rn(sv.y, d, gv.y);
            gv.z = __fmaf_rn(sv.z, d, gv.z);
            gv.w = __fmaf_rn(sv.w, d, gv.w);
            *g = gv;
          } else {
            s.G[kB + q - 480] += s.dz[q - 480];
          }
        }
      }
    }
    return;
  }
  for (int idx = threadIdx.x; idx < 1930; idx += blockDim.x) {
    if (idx < 1920) {
      const int i = idx / 192, j = idx - i * 192;
      put<ACCUM>(s, row, kFC + idx, fadd(0.0f, fmul(s.s2[j], s.dz[i])));
    } else {
      put<ACCUM>(s, row, kB + idx - 1920, fadd(0.0f, s.dz[idx - 1920]));
    }
  }
  for (int j = threadIdx.x; j < 192; j += blockDim.x) {
    float ds = 0.0f;
#pragma unroll
    for (int i = 0; i < 10; ++i) ds = mac<EXACT>(ds, s.P[kFC + i * 192 + j], s.dz[i]);
    const float dc = fmul(ds, 0.25f);
    const int c = j >> 4, py = (j >> 2) & 3, px = j & 3;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const int yy = 2 * py + dy, xx = 2 * px + dx;
        const float o = s.c2[(c * 8 + yy) * 8 + xx];
        const float d = fmul(fmul(dc, o), fsub(1.0f, o));
        s.dzp[dzp_at(c, yy + 4, xx + 4)] = d;
        if constexpr (!EXACT && TLB_PAIR && TLB_GK2K) s.Kp[dzk_at(c % 6, yy, xx) + c / 6] = d;
      }
  }
}

// g_k2[i][c][u][v] = sum_{y,x<8} s1[c][u+y][v+x] * dz2[i][y][x] (conv(s1, dz2[i]), nn.cpp:160;
// 64 taps row-major) and g_b2[i] = sum_all(dz2[i]).  EXACT: one lane per (i,c,u), five ordered chains.
template <bool ACCUM>
__device__ __forceinline__ void gk2_exact(const Smem& s, float* row, int t) {
  if (t < 360) {
    const int i = t / 30, r = t - i * 30, c = r / 5, u = r - c * 5;
    float acc[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 2
    for (int y = 0; y < 8; ++y) {
      const float4* sp = reinterpret_cast<const float4*>(s.s1 + (c * 12 + u + y) * 12);
      const float4 a = sp[0], b = sp[1], cc = sp[2];
      const float sr[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, cc.x, cc.y, cc.z, cc.w};
      const float4* dp = reinterpret_cast<const float4*>(s.dzp + dzp_at(i, y + 4, 4));
      const float4 d0 = dp[0], d1 = dp[1];
      const float dr[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int v = 0; v < 5; ++v) acc[v] = mac<true>(acc[v], sr[v + x], dr[x]);
    }
#pragma unroll
    for (int v = 0; v < 5; ++v) put<ACCUM>(s, row, kK2 + ((i * 6 + c) * 5 + u) * 5 + v, acc[v]);
  } else {
    const int i = t - 360;
    float acc = 0.0f;
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const float4* dp = reinterpret_cast<const float4*>(s.dzp + dzp_at(i, y + 4, 4));
      const float4 d0 = dp[0], d1 = dp[1];
      acc = fadd(fadd(fadd(fadd(acc, d0.x), d0.y), d0.z), d0.w);
      acc = fadd(fadd(fadd(fadd(acc, d1.x), d1.y), d1.z), d1.w);
    }
    put<ACCUM>(s, row, kB2 + i, acc);
  }
}

// Fast g_k2/g_b2 in row form: lane t < 360 -> (c, u) = t / 12, kernel i = t % 12 (the twelve kernels of a
// (c, u) share the s1 rows: broadcast loads), five outputs v over the 64 taps in (y, x) order with FFMA,
// no cross-lane reduction; the (c, u) = (0, 0) lanes also form g_b2[i] (row sums, then over y).
template <bool ACCUM>
__device__ __forceinline__ void gk2_rows(const Smem& s, float* row, int t) {
  const int cu = t / 12, i = t - cu * 12, c = cu / 5, u = cu - c * 5;
  float acc[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
  float bsum = 0.0f;
#pragma unroll kGk2rYUnroll
  for (int y = 0; y < 8; ++y) {
    const float4* sp = reinterpret_cast<const float4*>(s.s1 + (c * 12 + u + y) * 12);
    const float4 a = sp[0], b = sp[1], cc = sp[2];
    const float sr[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, cc.x, cc.y, cc.z, cc.w};
    const float4* dp = reinterpret_cast<const float4*>(s.dzp + dzp_at(i, y + 4, 4));
    const float4 d0 = dp[0], d1 = dp[1];
    const float dr[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
    for (int x = 0; x < 8; ++x)
#pragma unroll
      for (int v = 0; v < 5; ++v) acc[v] = __fmaf_rn(sr[v + x], dr[x], acc[v]);
    if (cu == 0) bsum += ((dr[0] + dr[1]) + (dr[2] + dr[3])) + ((dr[4] + dr[5]) + (dr[6] + dr[7]));
  }
#pragma unroll
  for (int v = 0; v < 5; ++v) put<ACCUM>(s, row, kK2 + ((i * 6 + c) * 5 + u) * 5 + v, acc[v]);
  if (cu == 0) put<ACCUM>(s, row, kB2 + i, bsum);
}

// Fast backin in scatter form, no padded taps.  Lane = (channel c, d_s1 row p, kernel split s): for
// each of its 12/SPLITS kernels i it holds the 25 weights of k2[i][c] and, for every valid tap row u1
// (dz2 row y = p - u1 in 0..7), scatters the 8 dz2 values of row y into the 12 row accumulators:
// acc[x + u2] += k2[i][c][u1][u2] * dz2[i][y][x] -- exactly the 115,200 valid multiply-adds of the
// reference's clipped sums (nn.cpp:169-189), against 259,200 for the padded 2x4 tiles.  Rows are
// ordered by their valid-tap count (p = 4..7 first, 0/11 last) so the lanes of a warp take the same
// trip count.  The SPLITS lanes of a (c, p) combine by xor shuffles; each then finishes 12/SPLITS
// columns (backavgpool + backsigmoid through c1, nn.cpp:148-158 / 131-133).
__device__ __forceinline__ int backin_row_of(int k) {  // k-th row by descending valid-tap count
  constexpr unsigned long long kOrder = 0xB0A192837654ULL;  // nibbles, low first: 4,5,6,7,3,8,2,9,1,10,0,11
  return (int)((kOrder >> (4 * k)) & 0xF);
}

// WP: weights read as scalars from the unpadded P (stride 25 per (i, c): distinct banks across the
// warp's (i, c) pairs) instead of float4s from the padded Kp (stride 40: 8-way bank groups).
template <int SPLITS, bool WP = false>
__device__ __forceinline__ void backin_rows(const Smem& s, int t) {
  constexpr int KPL = 12 / SPLITS;
  const bool valid = t < 72 * SPLITS;  // padding lanes compute combo 0 for the warp-wide shuffles
  const int combo = valid ? t / SPLITS : 0, part = t % SPLITS;
  const int p = backin_row_of(combo / 6), c = combo - (combo / 6) * 6;
  float acc[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) acc[q] = 0.0f;
#pragma unroll kBackinKUnroll
  for (int k = 0; k < KPL; ++k) {
    const int i = part * KPL + k;
    float w[5][5];
    if constexpr (WP) {
      const float* wp = s.P + kK2 + (i * 6 + c) * 25;
#pragma unroll
      for (int u1 = 0; u1 < 5; ++u1)
#pragma unroll
        for (int u2 = 0; u2 < 5; ++u2) w[u1][u2] = wp[u1 * 5 + u2];
    } else {
#pragma unroll
      for (int u1 = 0; u1 < 5; ++u1) {
        const float4* wp = reinterpret_cast<const float4*>(s.Kp + ((i * 6 + c) * 5 + u1) * 8);
        const float4 w0 = wp[0], w1 = wp[1];
        w[u1][0] = w0.x; w[u1][1] = w0.y; w[u1][2] = w0.z; w[u1][3] = w0.w; w[u1][4] = w1.x;
      }
    }
#pragma unroll
    for (int u1 = 0; u1 < 5; ++u1) {
      const int y = p - u1;
      if (y < 0 || y > 7) continue;
      const float4* dp = reinterpret_cast<const float4*>(s.dzp + dzp_at(i, y + 4, 4));
      const float4 d0 = dp[0], d1 = dp[1];
      const float d[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int u2 = 0; u2 < 5; ++u2) acc[x + u2] = __fmaf_rn(w[u1][u2], d[x], acc[x + u2]);
    }
  }
#pragma unroll
  for (int q = 0; q < 12; ++q) {
#pragma unroll
    for (int m = 1; m < SPLITS; m <<= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], m);
  }
  constexpr int QN = 12 / SPLITS;  // d_s1 columns this lane finishes: q0 .. q0 + QN - 1
  const int q0 = part * QN;
  float mine[QN];
#pragma unroll
  for (int k = 0; k < QN; ++k) {  // select acc[q0 + k] without dynamic register indexing
    float v = acc[k];
#pragma unroll
    for (int pp = 1; pp < SPLITS; ++pp)
      if (part == pp) v = acc[pp * QN + k];
    mine[k] = v;
  }
  if (!valid) return;
#pragma unroll
  for (int dy = 0; dy < 2; ++dy) {
    float* cp = s.c1 + c1_at(c, 2 * p + dy, 2 * q0);
#pragma unroll
    for (int k = 0; k < QN; ++k) {
      const float dc = fmul(mine[k], 0.25f);
      float2 v = *reinterpret_cast<float2*>(cp + 2 * k);
      v.x = fmul(fmul(dc, v.x), fsub(1.0f, v.x));
      v.y = fmul(fmul(dc, v.y), fsub(1.0f, v.y));
      *reinterpret_cast<float2*>(cp + 2 * k) = v;
    }
  }
}

// EXACT backin in scatter form, bit-identical to the reference's clipped nested sums (nn.cpp:169-189,
// network.cpp:135-138).  Lane = (channel c, d_s1 row p, kernel split of 3) as in backin_rows.  Per
// kernel i and per valid tap row ky (ascending, = off1 + u1; dz2 row y = p - ky), the twelve row sums
// rs[q] start at +0 and take k2[i][c][ky][kx] * dz2[i][y][q - kx] over the valid kx in ascending order
// (kx outer, x inner: each output sees its kx in order), each product rounded then added (no FMA);
// then b_i[q] = b_i[q] + rs[q] (the outer sum, from +0).  Only valid terms are formed -- the clipped
// sums add exactly these, in this order.  Finally d_s1[q] = ((0 + b_0[q]) + b_1[q]) + ... + b_11[q]:
// the four split lanes pass their per-kernel terms to part 0 by shuffle in kernel order.
__device__ __forceinline__ void backin_rows_exact(const Smem& s, int t) {
  constexpr int SPLITS = 4, KPL = 3;
  const bool valid = t < 72 * SPLITS;
  const int combo = valid ? t / SPLITS : 0, part = t % SPLITS;
  const int p = backin_row_of(combo / 6), c = combo - (combo / 6) * 6;
  float b[KPL][12];
#pragma unroll
  for (int k = 0; k < KPL; ++k) {
    const int i = part * KPL + k;
    const float* wp = s.P + kK2 + (i * 6 + c) * 25;
#pragma unroll
    for (int q = 0; q < 12; ++q) b[k][q] = 0.0f;
#pragma unroll
    for (int ky = 0; ky < 5; ++ky) {
      const int y = p - ky;
      if (y < 0 || y > 7) continue;
      const float4* dp = reinterpret_cast<const float4*>(s.dzp + dzp_at(i, y + 4, 4));
      const float4 d0 = dp[0], d1 = dp[1];
      const float d[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
      float w[5];
#pragma unroll
      for (int kx = 0; kx < 5; ++kx) w[kx] = wp[ky * 5 + kx];
      float rs[12];
#pragma unroll
      for (int q = 0; q < 12; ++q) rs[q] = 0.0f;
#pragma unroll
      for (int kx = 0; kx < 5; ++kx)
#pragma unroll
        for (int x = 0; x < 8; ++x) rs[x + kx] = fadd(rs[x + kx], fmul(w[kx], d[x]));
#pragma unroll
      for (int q = 0; q < 12; ++q) b[k][q] = fadd(b[k][q], rs[q]);
    }
  }
  const int base = (threadIdx.x & 31) & ~(SPLITS - 1);
  float acc[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) acc[q] = 0.0f;
#pragma unroll
  for (int i = 0; i < 12; ++i)
#pragma unroll
    for (int q = 0; q < 12; ++q) acc[q] = fadd(acc[q], __shfl_sync(0xffffffffu, b[i % KPL][q], base + i / KPL));
  if (!valid || part != 0) return;
#pragma unroll
  for (int dy = 0; dy < 2; ++dy) {  // backavgpool (x0.25) + backsigmoid through c1 -> dz1, 24 columns
    float* cp = s.c1 + c1_at(c, 2 * p + dy, 0);
#pragma unroll
    for (int q4 = 0; q4 < 6; ++q4) {
      float4 v = reinterpret_cast<float4*>(cp)[q4];
      const float dc0 = fmul(acc[2 * q4], 0.25f), dc1 = fmul(acc[2 * q4 + 1], 0.25f);
      v.x = fmul(fmul(dc0, v.x), fsub(1.0f, v.x));
      v.y = fmul(fmul(dc0, v.y), fsub(1.0f, v.y));
      v.z = fmul(fmul(dc1, v.z), fsub(1.0f, v.z));
      v.w = fmul(fmul(dc1, v.w), fsub(1.0f, v.w));
      reinterpret_cast<float4*>(cp)[q4] = v;
    }
  }
}

// Fast g_k2 on kernel pairs (TLB_GK2K): lane j < 180 = (channel c, row u) = j / 6, kernel pair ip = j % 6 (the
// six pair lanes of a (c, u) read the same s1 rows: broadcast); five outputs v over the 64 taps (y, x):
// s1[c][u+y][v+x] (broadcast) x (dz2[ip][y][x], dz2[ip+6][y][x]) -> (g_k2[ip][c][u][v], g_k2[ip+6][c][u][v])
// with FFMA2; the (c, u) = (0, 0) lanes also form (g_b2[ip], g_b2[ip+6]).
template <bool ACCUM>
__device__ __forceinline__ void gk2_kpair(const Smem& s, float* row, int j) {
  const int cu = j / 6, ip = j - cu * 6, c = cu / 5, u = cu - c * 5;
  float2 acc[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) acc[v] = make_float2(0.0f, 0.0f);
  float2 bsum = make_float2(0.0f, 0.0f);
#pragma unroll 2
  for (int y = 0; y < 8; ++y) {
    const float4* sp = reinterpret_cast<const float4*>(s.s1 + (c * 12 + u + y) * 12);
    const float4 a = sp[0], b = sp[1], cc = sp[2];
    const float sr[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, cc.x, cc.y, cc.z, cc.w};
    const float4* dp = reinterpret_cast<const float4*>(s.Kp + dzk_at(ip, y, 0));
    float2 d[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 v = dp[q];
      d[2 * q] = make_float2(v.x, v.y);
      d[2 * q + 1] = make_float2(v.z, v.w);
    }
#pragma unroll
    for (int x = 0; x < 8; ++x)
#pragma unroll
      for (int v = 0; v < 5; ++v) acc[v] = __ffma2_rn(bcast2(sr[v + x]), d[x], acc[v]);
    if (cu == 0) {
      const float2 r0 = make_float2((d[0].x + d[1].x) + (d[2].x + d[3].x), (d[0].y + d[1].y) + (d[2].y + d[3].y));
      const float2 r1 = make_float2((d[4].x + d[5].x) + (d[6].x + d[7].x), (d[4].y + d[5].y) + (d[6].y + d[7].y));
      bsum = make_float2(bsum.x + (r0.x + r1.x), bsum.y + (r0.y + r1.y));
    }
  }
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    const int idx = kK2 + ((ip * 6 + c) * 5 + u) * 5 + v;
    put<ACCUM>(s, row, idx, acc[v].x);
    put<ACCUM>(s, row, idx + 900, acc[v].y);  // kernel ip + 6: 6 x 150 floats further
  }
  if (cu == 0) {
    put<ACCUM>(s, row, kB2 + ip, bsum.x);
    put<ACCUM>(s, row, kB2 + ip + 6, bsum.y);
  }
}

// g_k2 lanes done beside the scatter-form backin in conv2_back V14 / V15 (and the variants 10..13).
__host__ __device__ constexpr int gk2_split_lanes(int V) {
  return V == 10 ? 224 : V == 11 ? 160 : V == 12 ? 192 : V == 13 ? 128 : V == 14 ? TLB_GK2R_SPLIT
       : V == 15 ? TLB_EXACT_GK2_SPLIT : 0;
}

// C2 backward stage (the schedules settled by the stage bench, profiles/README.md; the rejected variants
// live in stage_variants.cuh for csrc/stage_bench.cu).
//   V = 14 (fast): scatter-form backin rows (4 kernel splits, weights from P) on warps 0-8 beside g_k2 row
//          lanes 0..TLB_GK2R_SPLIT-1 on warps 9-15; the remaining row lanes run beside the C1 gradient.
//   V = 15 (EXACT): scatter-form exact backin on warps 0-8 beside ordered g_k2 chains 0..TLB_EXACT_GK2_SPLIT-1
//          on warps 9-15; the remaining chains run beside the C1 gradient.
template <bool EXACT, bool ACCUM, int V>
__device__ __forceinline__ void stage_conv2_back(const Smem& s, float* row) {
  static_assert(EXACT ? V == 15 : V == 14, "product schedules: V14 (fast), V15 (EXACT)");
  constexpr int kBeside = (!EXACT && TLB_PAIR && TLB_GK2K) ? (TLB_GK2K_SPLIT + 31) / 32 * 32 : gk2_split_lanes(V);
  for (int it = threadIdx.x; it < 288 + kBeside; it += blockDim.x) {  // whole warps per round
    if constexpr (EXACT) {
      if (it < 288) backin_rows_exact(s, it);
      else gk2_exact<ACCUM>(s, row, it - 288);
    } else if constexpr (TLB_PAIR && TLB_GK2K) {
      if (it < 288) backin_rows<4, true>(s, it);
      else if (it - 288 < TLB_GK2K_SPLIT) gk2_kpair<ACCUM>(s, row, it - 288);
    } else {
      if (it < 288) backin_rows<4, true>(s, it);
      else gk2_rows<ACCUM>(s, row, it - 288);
    }
  }
}

// One EXACT C1-gradient lane: it < 150 -> g_k1[i][u][v] as one ordered 576-term chain (lanes (u, v)-major,
// i minor: a warp reads ~6 shifted-image rows and the 6 dz1 channel rows of one y, each in its own bank
// group); 150 <= it < 156 -> g_b1[i] as the ordered sum of dz1[i].
template <bool ACCUM>
__device__ __forceinline__ void stage_conv1_back_lane_exact(const Smem& s, float* row, int it) {
  const float* dz1 = s.c1;
  if (it < 150) {
    // lane = (u, v) major, i minor: a warp reads ~6 shifted-image rows and the 6 dz1 channel rows
    // of one y, each in its own bank group (conflict-free 128-bit loads)
    const int i = it % 6, r = it / 6, u = r / 5, v = r - u * 5;
    const float4* ib = reinterpret_cast<const float4*>(s.sh + sh_at(v, u));
    const float4* db = reinterpret_cast<const float4*>(dz1 + i * kC1Plane);
    float acc = 0.0f;
    // software pipeline: row y+1 is in flight while the ordered chain consumes row y
    float4 a[6], d[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      a[q] = ib[q];
      d[q] = db[q];
    }
#pragma unroll 1
    for (int y = 0; y < 24; ++y) {
      const int yn = y + 1 < 24 ? y + 1 : y;
      float4 an[6], dn[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        an[q] = ib[yn * 6 + q];
        dn[q] = db[yn * 6 + q];
      }
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        acc = mac<true>(acc, a[q].x, d[q].x);
        acc = mac<true>(acc, a[q].y, d[q].y);
        acc = mac<true>(acc, a[q].z, d[q].z);
        acc = mac<true>(acc, a[q].w, d[q].w);
      }
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        a[q] = an[q];
        d[q] = dn[q];
      }
    }
    put<ACCUM>(s, row, kK1 + i * 25 + r, acc);
  } else {
    const int i = it - 150;
    const float4* dp = reinterpret_cast<const float4*>(dz1 + i * kC1Plane);
    float acc = 0.0f;
#pragma unroll 4
    for (int e = 0; e < 144; ++e) {
      const float4 d = dp[e];
      acc = fadd(fadd(fadd(fadd(acc, d.x), d.y), d.z), d.w);
    }
    put<ACCUM>(s, row, kB1 + i, acc);
  }
}

// C1 backward: g_k1[i][u][v] = sum_{y,x<24} I[u+y][v+x]*dz1[i][y][x]; g_b1[i] = sum dz1[i].
// EXACT: one lane per output, the 576 terms in order, reading the v-shifted image copy so every row
// is aligned 128-bit loads.  Fast: one lane per (i, y) holds all 25 outputs (the dz1 row stays in
// registers and feeds 5 image rows), then a fixed-order combine over the 24 row partials.
// EXACT C1 weight gradient, register-blocked: lane (u, i) of a warp owns the chains of outputs
// (i, u, V0..V0+NV-1) -- the image row u+y (28 floats) and the dz1 row (i, y) are loaded once per y and
// feed NV ordered 576-term chains (each chain still adds its products in the reference order: y, then x).
// Two warps cover v = {0,1,2} and {3,4}; a third holds the six g_b1 chains.
template <bool ACCUM, int V0, int NV>
__device__ __forceinline__ void c1back_exact_vgroup(const Smem& s, const float* img, float* row, int lane) {
  if (lane >= 30) return;
  const int u = lane / 6, i = lane - u * 6;  // i minor: the six dz1 channel rows sit in distinct bank groups
  const float4* ib = reinterpret_cast<const float4*>(img + u * 28);
  const float4* db = reinterpret_cast<const float4*>(s.c1 + i * kC1Plane);
  float acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0f;
  float4 a[7], d[6];
#pragma unroll
  for (int q = 0; q < 7; ++q) a[q] = ib[q];
#pragma unroll
  for (int q = 0; q < 6; ++q) d[q] = db[q];
#pragma unroll 1
  for (int y = 0; y < 24; ++y) {
    const int yn = y + 1 < 24 ? y + 1 : y;
    float4 an[7], dn[6];  // next row in flight while this row's chains run
#pragma unroll
    for (int q = 0; q < 7; ++q) an[q] = ib[yn * 7 + q];
#pragma unroll
    for (int q = 0; q < 6; ++q) dn[q] = db[yn * 6 + q];
    const float ir[28] = {a[0].x, a[0].y, a[0].z, a[0].w, a[1].x, a[1].y, a[1].z, a[1].w, a[2].x, a[2].y,
                          a[2].z, a[2].w, a[3].x, a[3].y, a[3].z, a[3].w, a[4].x, a[4].y, a[4].z, a[4].w,
                          a[5].x, a[5].y, a[5].z, a[5].w, a[6].x, a[6].y, a[6].z, a[6].w};
    const float dr[24] = {d[0].x, d[0].y, d[0].z, d[0].w, d[1].x, d[1].y, d[1].z, d[1].w,
                          d[2].x, d[2].y, d[2].z, d[2].w, d[3].x, d[3].y, d[3].z, d[3].w,
                          d[4].x, d[4].y, d[4].z, d[4].w, d[5].x, d[5].y, d[5].z, d[5].w};
#pragma unroll
    for (int x = 0; x < 24; ++x)
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[v] = mac<true>(acc[v], ir[V0 + v + x], dr[x]);
#pragma unroll
    for (int q = 0; q < 7; ++q) a[q] = an[q];
#pragma unroll
    for (int q = 0; q < 6; ++q) d[q] = dn[q];
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) put<ACCUM>(s, row, kK1 + i * 25 + u * 5 + V0 + v, acc[v]);
}

template <bool ACCUM>
__device__ __forceinline__ void stage_conv1_back_exact_blocked(const Smem& s, const float* img, float* row) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (blockDim.x >= 96) {
    if (warp == 0) c1back_exact_vgroup<ACCUM, 0, 3>(s, img, row, lane);
    else if (warp == 1) c1back_exact_vgroup<ACCUM, 3, 2>(s, img, row, lane);
    else if (warp == 2 && lane < 6) stage_conv1_back_lane_exact<ACCUM>(s, row, 150 + lane);
  }
}

// C1 weight gradient with the conv2 weight gradient on the otherwise idle lanes (EXACT: the C1 chains
// occupy 156 lanes for ~5 us; g_k2/g_b2 need only dz2 and s1, so they no longer share a phase with backin).
// Fast C1 weight gradient run by the first 160 threads only (named barrier 1 between its two phases):
// 144 (i, y) lanes form 25 row partials + the bias row partial, then 156 lanes combine the 24 row
// partials in fixed order.
template <bool ACCUM>
__device__ __forceinline__ void conv1_back_fast_group(const Smem& s, const float* img, float* row) {
  constexpr int kGroup = 160;
  const float* dz1 = s.c1;
  const int it = threadIdx.x;
  if (it < 144) {
    const int i = it / 24, y = it - i * 24;
    const float4* dp = reinterpret_cast<const float4*>(dz1 + c1_at(i, y, 0));
    float dr[24];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const float4 t = dp[q];
      dr[4 * q] = t.x; dr[4 * q + 1] = t.y; dr[4 * q + 2] = t.z; dr[4 * q + 3] = t.w;
    }
    float bias = 0.0f;
#pragma unroll
    for (int x = 0; x < 24; ++x) bias += dr[x];
    float* out = s.red + it * 26;
    out[25] = bias;
#pragma unroll 1
    for (int u = 0; u < 5; ++u) {
      const float4* ip = reinterpret_cast<const float4*>(img + (u + y) * 28);
      float ir[28];
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const float4 t = ip[q];
        ir[4 * q] = t.x; ir[4 * q + 1] = t.y; ir[4 * q + 2] = t.z; ir[4 * q + 3] = t.w;
      }
      float acc[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int x = 0; x < 24; ++x)
#pragma unroll
        for (int v = 0; v < 5; ++v) acc[v] = __fmaf_rn(ir[x + v], dr[x], acc[v]);
#pragma unroll
      for (int v = 0; v < 5; ++v) out[u * 5 + v] = acc[v];
    }
  }
  named_sync(1, kGroup);
  if (it < 156) {
    float acc = 0.0f;
    const int col = it < 150 ? (it % 25) : 25, i = it < 150 ? it / 25 : it - 150;
#pragma unroll 8
    for (int y = 0; y < 24; ++y) acc += s.red[(i * 24 + y) * 26 + col];
    put<ACCUM>(s, row, it < 150 ? kK1 + it : kB1 + i, acc);
  }
}

// Fast C1 weight gradient on 288 lanes (512-thread CTAs): lane pair (i, y) splits the five tap rows
// u = 0..2 | 3..4 (+ the bias row-partial), so phase 1 takes ~390 instead of ~635 issue slots per lane;
// the fixed-order combine over y is unchanged (named barrier 1 over the 288 lanes).
template <bool ACCUM>
__device__ __forceinline__ void conv1_back_fast_group2(const Smem& s, const float* img, float* row) {
  constexpr int kGroup = 288;
  const float* dz1 = s.c1;
  const int it = threadIdx.x;  // < kGroup
  const int pr = it >> 1, h = it & 1;
  const int i = pr / 24, y = pr - i * 24;
  const float4* dp = reinterpret_cast<const float4*>(dz1 + c1_at(i, y, 0));
  float dr[24];
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const float4 t = dp[q];
    dr[4 * q] = t.x; dr[4 * q + 1] = t.y; dr[4 * q + 2] = t.z; dr[4 * q + 3] = t.w;
  }
  float* out = s.red + pr * 26;
  if (h) {
    float bias = 0.0f;
#pragma unroll
    for (int x = 0; x < 24; ++x) bias += dr[x];
    out[25] = bias;
  }
  const int u0 = h ? 3 : 0, un = h ? 2 : 3;
#pragma unroll kC1g2Unroll
  for (int k = 0; k < un; ++k) {
    const int u = u0 + k;
    const float4* ip = reinterpret_cast<const float4*>(img + (u + y) * 28);
    float ir[28];
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      const float4 t = ip[q];
      ir[4 * q] = t.x; ir[4 * q + 1] = t.y; ir[4 * q + 2] = t.z; ir[4 * q + 3] = t.w;
    }
    float acc[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int x = 0; x < 24; ++x)
#pragma unroll
      for (int v = 0; v < 5; ++v) acc[v] = __fmaf_rn(ir[x + v], dr[x], acc[v]);
#pragma unroll
    for (int v = 0; v < 5; ++v) out[u * 5 + v] = acc[v];
  }
  named_sync(1, kGroup);
  if (it < 156) {
    float acc = 0.0f;
    const int col = it < 150 ? (it % 25) : 25, ii = it < 150 ? it / 25 : it - 150;
#pragma unroll 8
    for (int yy = 0; yy < 24; ++yy) acc += s.red[(ii * 24 + yy) * 26 + col];
    put<ACCUM>(s, row, it < 150 ? kK1 + it : kB1 + ii, acc);
  }
}

template <bool EXACT, bool ACCUM, int GLO = 0, bool ROWS = false>
__device__ __forceinline__ void stage_conv1_back_gk2(const Smem& s, const float* img, float* row) {
  constexpr int kGk2 = EXACT ? 372 : ROWS ? 360 : 288;
  const int t = threadIdx.x;
  if constexpr (!EXACT && TLB_PAIR && TLB_GK2K) {  // the C1 gradient beside the remaining g_k2 pair lanes
    if (blockDim.x >= 512) {
      if (t < 288) conv1_back_fast_group2<ACCUM>(s, img, row);
      else for (int j = TLB_GK2K_SPLIT + t - 288; j < 180; j += blockDim.x - 288) gk2_kpair<ACCUM>(s, row, j);
    } else if (t < 160) {
      conv1_back_fast_group<ACCUM>(s, img, row);
    } else {
      for (int j = TLB_GK2K_SPLIT + t - 160; j < 180; j += blockDim.x - 160) gk2_kpair<ACCUM>(s, row, j);
    }
    return;
  }
  if constexpr (!EXACT && TLB_C1BACK_GROUP2) {
    if (blockDim.x >= 512) {  // C1 gradient on warps 0-8, the remaining g_k2 lanes on warps 9+
      if (t < 288) {
        conv1_back_fast_group2<ACCUM>(s, img, row);
      } else {
        for (int item = GLO + t - 288; item < kGk2; item += blockDim.x - 288) gk2_rows<ACCUM>(s, row, item);
      }
      return;
    }
  }
  static_assert(EXACT != ROWS, "fast mode: row-form g_k2 lanes; EXACT: ordered g_k2 chains");
  if constexpr (EXACT && GLO > 0) {  // V15: ordered C1 chains on the first warps, g_k2 chains after them
    constexpr int kC1 = TLB_V15_C1_LANES ? 160 : 96;  // one chain per lane (5 warps) | blocked (3 warps)
    if (t < kC1) {
      if constexpr (TLB_V15_C1_LANES) {
        if (t < 156) stage_conv1_back_lane_exact<ACCUM>(s, row, t);
      } else {
        stage_conv1_back_exact_blocked<ACCUM>(s, img, row);
      }
    } else {
      for (int item = GLO + t - kC1; item < kGk2; item += blockDim.x - kC1) gk2_exact<ACCUM>(s, row, item);
    }
    return;
  }
  if (t < 160) {
    if constexpr (EXACT) {
      if (t < 156) stage_conv1_back_lane_exact<ACCUM>(s, row, t);
    } else {
      conv1_back_fast_group<ACCUM>(s, img, row);
    }
  } else {
    for (int item = GLO + t - 160; item < kGk2; item += blockDim.x - 160) {
      if constexpr (EXACT) gk2_exact<ACCUM>(s, row, item);
      else gk2_rows<ACCUM>(s, row, item);
    }
  }
}

// The product schedules (chosen with paper_1912_05234_b200/csrc/stage_bench.cu; alternatives in
// stage_variants.cuh): conv2 V0 lane halves (EXACT) / V2 row pairs with weights from P (fast); conv2_back
// V15 (EXACT) / V14 (fast), whose remaining g_k2 lanes run beside the C1 gradient.
template <bool EXACT>
struct StageCfg {
  static constexpr int conv2 = EXACT ? 0 : 2;
  static constexpr int conv2_back = EXACT ? 15 : 14;
  static constexpr int gk2_lo = gk2_split_lanes(conv2_back);  // g_k2 lanes already done in conv2_back
  static constexpr bool gk2_rows = !EXACT;                      // fast: row-form g_k2 lanes (gk2_rows)
};

// ---------------------------------------------------------------------------------------------
// Out-of-line stage entry points.  Each stage is compiled as its own function so the register
// allocator schedules it without the persistent kernel's long-lived state (step/job/prefetch
// bookkeeping) occupying registers; the stages re-derive the shared-memory map themselves.
// ---------------------------------------------------------------------------------------------
template <bool EXACT>
__device__ __noinline__ void call_conv1(const float* img) { stage_conv1<EXACT>(smem_view(), img); }
template <bool EXACT>
__device__ __noinline__ void call_conv2() { stage_conv2<EXACT, StageCfg<EXACT>::conv2>(smem_view()); }
template <bool EXACT>
__device__ __noinline__ void call_fc(int label, const float* y, bool want_dz) {
  stage_fc<EXACT>(smem_view(), label, y, want_dz);
}
template <bool EXACT, bool ACCUM>
__device__ __noinline__ void call_fc_back(float* row) { stage_fc_back<EXACT, ACCUM>(smem_view(), row); }
template <bool EXACT, bool ACCUM>
__device__ __noinline__ void call_conv2_back(float* row) {
  stage_conv2_back<EXACT, ACCUM, StageCfg<EXACT>::conv2_back>(smem_view(), row);
}
template <bool EXACT, bool ACCUM>
__device__ __noinline__ void call_conv1_back(const float* img, float* row) {
  stage_conv1_back_gk2<EXACT, ACCUM, StageCfg<EXACT>::gk2_lo, StageCfg<EXACT>::gk2_rows>(smem_view(), img, row);
}

// Whole forward pass of one image (image already in shared memory).  `lab` (train kernels): the label
// sits in shared memory, written by an async copy that thread 0 completed before conv1; it is read only
// after conv1's barrier.
// Byte ingestion (TrainArgs::pixels): the NEXT job's pixel bytes, converted while this job runs conv2.
struct NextBytes {
  int buf;          // its image buffer
  uint32_t parity;  // the mbarrier phase its bytes complete
  float* wb;        // fp32 write-back base (TrainArgs::images_wb); the job index is s.jidx[buf]
};
constexpr int kConv2Lanes = 192;  // conv2 (both modes' variants) runs on threads [0, 192): the rest are idle

// Threads [kConv2Lanes, blockDim) during conv2: if the next job arrives as bytes, wait for them and convert
// (pixel / 255.0f) into its fp32 buffer and the global write-back -- off the critical path of both jobs.
__device__ __forceinline__ void convert_next_bytes(const Smem& s, const NextBytes* nb) {
  if (!nb || (int)threadIdx.x < kConv2Lanes || !s.bst[nb->buf]) return;
  mbar_wait(&s.bar[nb->buf], nb->parity);
  const int t = threadIdx.x - kConv2Lanes, T = blockDim.x - kConv2Lanes;
  const uint32_t* px = reinterpret_cast<const uint32_t*>(s.px + nb->buf * kImg);
  float4* img = reinterpret_cast<float4*>(s.img + nb->buf * kImg);
  float4* wb = nb->wb ? reinterpret_cast<float4*>(nb->wb + s.jidx[nb->buf] * kImg) : nullptr;
  for (int q = t; q < kImg / 4; q += T) {
    const uint32_t w = px[q];
    const float4 v = make_float4(__fdiv_rn((float)(w & 0xffu), 255.0f), __fdiv_rn((float)((w >> 8) & 0xffu), 255.0f),
                                 __fdiv_rn((float)((w >> 16) & 0xffu), 255.0f), __fdiv_rn((float)(w >> 24), 255.0f));
    img[q] = v;
    if (wb) __stcg(wb + q, v);
  }
}

template <bool EXACT>
__device__ __forceinline__ void forward_image(const Smem& s, const float* img, int label, const float* y,
                                              bool want_dz, const int* lab = nullptr, uint64_t* post_conv1 = nullptr,
                                              uint32_t post_conv1_parity = 0, long long wait_limit = 0,
                                              unsigned int* abort = nullptr, const NextBytes* next_bytes = nullptr) {
  call_conv1<EXACT>(img);
  __syncthreads();
  if (lab) label = *lab;
  // clustered kernel: the parameters conv2 and later stages read may still be arriving during conv1
  if (post_conv1) mbar_wait_cluster_guarded(post_conv1, post_conv1_parity, wait_limit, abort);
  mark(s, 3);
  call_conv2<EXACT>();  // includes avgpool
  convert_next_bytes(s, next_bytes);
  __syncthreads();
  mark(s, 4);
  mark(s, 5);
  call_fc<EXACT>(label, y, want_dz);
  __syncthreads();
  mark(s, 6);
}

// Whole backward pass (after forward_image with want_dz).  Ends with a __syncthreads.
template <bool EXACT, bool ACCUM>
__device__ __forceinline__ void backward_image(const Smem& s, const float* img, float* row) {
  call_fc_back<EXACT, ACCUM>(row);
  __syncthreads();
  mark(s, 7);
  call_conv2_back<EXACT, ACCUM>(row);
  __syncthreads();
  mark(s, 8);
  call_conv1_back<EXACT, ACCUM>(img, row);
  __syncthreads();
  mark(s, 9);
}

}  // namespace tlb
