// wide_kernels.cuh -- shapes, parameter layout, GEMM operand functors and the step driver of the widened
// CNN (BASELINE.json configs[4]); see wide_kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tlb {
namespace wide {

// ---- network shape (composition of nn.cpp operators) ----------------------
constexpr int kImgW = 64;                       // input [64,64]
constexpr int kC1N = 32, kC1W = 60;             // c1 [32,60,60]
constexpr int kS1W = 30, kS1Pos = kS1W * kS1W;  // s1 [32,30,30]
constexpr int kC2N = 64, kC2W = 26, kC2Pos = kC2W * kC2W;  // c2 [64,1,26,26]
constexpr int kS2Len = kC2N * 13 * 13;          // s2 [64,1,13,13] = 10,816
constexpr int kClasses = 10;
constexpr int kK2Slice = kC1N * 25;             // 800 = one conv2 kernel [32,5,5]
constexpr int kGk2Rows = kK2Slice + 1;          // + the all-ones row that yields g_b2

// ---- flat parameter / gradient layout, write_flat order k1,b1,k2,b2,fc,b (network.cpp:186-193) -------
constexpr int kOffK1 = 0;
constexpr int kOffB1 = kOffK1 + kC1N * 25;        // 800
constexpr int kOffK2 = kOffB1 + kC1N;             // 832
constexpr int kOffB2 = kOffK2 + kC2N * kK2Slice;  // 52,032
constexpr int kOffFC = kOffB2 + kC2N;             // 52,096
constexpr int kOffBF = kOffFC + kClasses * kS2Len; // 160,256
constexpr int kNParam = kOffBF + kClasses;        // 160,266

constexpr int64_t kFlopPerTrainImage = 2LL * 109918080;  // 109,918,080 MAC
constexpr int64_t kFlopPerFwdImage = 2LL * (2880000 + 34611200 + 108160);

__device__ __forceinline__ float sigmoid_fast(float x) { return __frcp_rn(1.0f + __expf(-x)); }

// dz2 is stored zero-padded by 4 on every side ([m][64][34][34]) so the backin gather needs no bounds
// checks (the reference's clipped sums, nn.cpp:169-189, only ever drop zero products).
constexpr int kDzPad = 4, kDzW = kC2W + 2 * kDzPad, kDzPlane = kDzW * kDzW;  // 34, 1156

// ---- GEMM operand functors: D[m][n] = sum_k A[m][k] * B[n][k] over this split's k range ----------------
// Every operand is separable: A[m][k] = Aptr[a_row(m) + a_col(k)], B[n][k] = Bptr[b_row(n) + b_col(k)], so
// the producers compute a row base once per tile and look column offsets up (kKTab > 0: K is static and
// the offsets are tabulated in shared memory once per CTA).  a(m,k)/b(n,k) are the generic forms.
template <class Op>
struct SepOps {
  __device__ __forceinline__ static float a(const Op& o, int64_t m, int64_t k) {
    return o.a_ones(m) ? 1.0f : o.A[o.a_row(m) + o.a_col(k)];
  }
  __device__ __forceinline__ static float b(const Op& o, int n, int64_t k) { return o.B[o.b_row(n) + o.b_col(k)]; }
};

// conv2 forward: m = (b, y, x) over 26x26 outputs, n = kernel i, k = (c, ky, kx); epilogue + b2, sigmoid.
struct OpConv2Fwd {
  static constexpr bool kAContigM = true;
  static constexpr int N = kC2N;
  static constexpr int kKTab = kK2Slice;
  static constexpr bool kBImage = true;   // B (the weights) is the same for every tile: pre-split image
  static constexpr bool kBDense = false;
  const float* A;  // s1
  const float* B;  // params (k2 rows)
  float* c2;
  int64_t M;
  const float* Bimg;  // tensor-core engine: per-chunk hi|lo swizzled B stages (tc_prepare_b)
  __device__ __forceinline__ void k_range(int, int64_t& k0, int64_t& k1) const {
    k0 = 0;
    k1 = kK2Slice;
  }
  __device__ __forceinline__ bool a_ones(int64_t) const { return false; }
  __device__ __forceinline__ int64_t a_row(int64_t m) const {
    const unsigned mm = (unsigned)m, b = mm / kC2Pos, pos = mm - b * kC2Pos, y = pos / kC2W, x = pos - y * kC2W;
    return (int64_t)b * (kC1N * kS1Pos) + y * kS1W + x;
  }
  __device__ __forceinline__ int a_col(int64_t k) const {
    const unsigned kk = (unsigned)k, c = kk / 25, r = kk - c * 25, ky = r / 5, kx = r - ky * 5;
    return (int)(c * kS1Pos + ky * kS1W + kx);
  }
  __device__ __forceinline__ int64_t b_row(int n) const { return kOffK2 + n * kK2Slice; }
  __device__ __forceinline__ int b_col(int64_t k) const { return (int)k; }
  __device__ __forceinline__ float a(int64_t m, int64_t k) const { return SepOps<OpConv2Fwd>::a(*this, m, k); }
  __device__ __forceinline__ float b(int n, int64_t k) const { return SepOps<OpConv2Fwd>::b(*this, n, k); }
  __device__ __forceinline__ void store(int, int64_t m, int n, float v) const {
    const unsigned mm = (unsigned)m, b = mm / kC2Pos, pos = mm - b * kC2Pos;
    c2[(size_t)(b * kC2N + n) * kC2Pos + pos] = sigmoid_fast(v + B[kOffB2 + n]);
  }
};

// conv2 weight gradient (+ bias via the all-ones row m = 800): m = (c, ky, kx), n = i, k = (b, y, x);
// split-K partials part[z][m][n] reduced in fixed split order.
struct OpGk2 {
  static constexpr bool kAContigM = false;
  static constexpr int N = kC2N;
  static constexpr int kKTab = 0;
  static constexpr bool kBImage = false;
  static constexpr bool kBDense = true;   // B rows contiguous and 16-B aligned: float4 gathers
  static constexpr int64_t M = kGk2Rows;
  const float* A;  // s1
  const float* B;  // dz2t: [64][K] = dz2 transposed to (i, (b, y, x)), written by fc_kernel
  float* part;
  int64_t K;
  int splits;
  __device__ __forceinline__ void k_range(int z, int64_t& k0, int64_t& k1) const {
    const int64_t chunk = ((K + splits - 1) / splits + 31) / 32 * 32;
    k0 = (int64_t)z * chunk;
    k1 = k0 + chunk < K ? k0 + chunk : K;
  }
  __device__ __forceinline__ bool a_ones(int64_t m) const { return m == kK2Slice; }
  __device__ __forceinline__ int64_t a_row(int64_t m) const {
    const unsigned mm = (unsigned)m, c = mm / 25, r = mm - c * 25, ky = r / 5, kx = r - ky * 5;
    return c * kS1Pos + ky * kS1W + kx;
  }
  __device__ __forceinline__ int64_t a_col(int64_t k) const {
    const unsigned kk = (unsigned)k, b = kk / kC2Pos, pos = kk - b * kC2Pos, y = pos / kC2W, x = pos - y * kC2W;
    return (int64_t)b * (kC1N * kS1Pos) + y * kS1W + x;
  }
  // a_col of 16 consecutive k: decompose the first, then step x -> y -> image with carries
  __device__ __forceinline__ void a_cols16(int64_t k, int64_t (&o)[16]) const {
    const unsigned kk = (unsigned)k;
    unsigned b = kk / kC2Pos, pos = kk - b * kC2Pos, y = pos / kC2W, x = pos - y * kC2W;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      o[e] = (int64_t)b * (kC1N * kS1Pos) + y * kS1W + x;
      if (++x == (unsigned)kC2W) {
        x = 0;
        if (++y == (unsigned)kC2W) {
          y = 0;
          ++b;
        }
      }
    }
  }
  __device__ __forceinline__ int64_t b_row(int n) const { return (int64_t)n * K; }
  __device__ __forceinline__ int64_t b_col(int64_t k) const { return k; }
  __device__ __forceinline__ float a(int64_t m, int64_t k) const { return SepOps<OpGk2>::a(*this, m, k); }
  __device__ __forceinline__ float b(int n, int64_t k) const { return SepOps<OpGk2>::b(*this, n, k); }
  __device__ __forceinline__ void store(int z, int64_t m, int n, float v) const {
    part[((int64_t)z * kGk2Rows + m) * kC2N + n] = v;
  }
};

// conv2 backin: m = (b, p, q) over the 30x30 s1 plane, n = channel c, k = (i, u, v) over the 64 kernels'
// 5x5 taps; A = padded dz2[b, i, p+4-u, q+4-v].  Epilogue: backavgpool (x0.25) + backsigmoid through c1
// -> dz1, written in place over c1.
struct OpBackin {
  static constexpr bool kAContigM = true;
  static constexpr int N = kC1N;
  static constexpr int kKTab = kC2N * 25;
  static constexpr bool kBImage = true;
  static constexpr bool kBDense = false;
  const float* A;  // dz2 (padded)
  const float* B;  // params (k2)
  float* c1;
  int64_t M;
  const float* Bimg;
  __device__ __forceinline__ void k_range(int, int64_t& k0, int64_t& k1) const {
    k0 = 0;
    k1 = (int64_t)kC2N * 25;
  }
  __device__ __forceinline__ bool a_ones(int64_t) const { return false; }
  __device__ __forceinline__ int64_t a_row(int64_t m) const {
    const unsigned mm = (unsigned)m, b = mm / kS1Pos, r = mm - b * kS1Pos, pp = r / kS1W, q = r - pp * kS1W;
    return (int64_t)b * (kC2N * kDzPlane) + (pp + kDzPad) * kDzW + q + kDzPad;
  }
  __device__ __forceinline__ int a_col(int64_t k) const {
    const int kk = (int)k, i = kk / 25, u = kk - i * 25, u1 = u / 5, u2 = u - u1 * 5;
    return i * kDzPlane - u1 * kDzW - u2;
  }
  __device__ __forceinline__ int64_t b_row(int n) const { return kOffK2 + n * 25; }
  __device__ __forceinline__ int b_col(int64_t k) const {
    const int kk = (int)k, i = kk / 25, u = kk - i * 25;
    return i * kK2Slice + u;
  }
  __device__ __forceinline__ float a(int64_t m, int64_t k) const { return SepOps<OpBackin>::a(*this, m, k); }
  __device__ __forceinline__ float b(int n, int64_t k) const { return SepOps<OpBackin>::b(*this, n, k); }
  __device__ __forceinline__ void store(int, int64_t m, int n, float v) const {
    const unsigned mm = (unsigned)m, b = mm / kS1Pos, r = mm - b * kS1Pos, pp = r / kS1W, q = r - pp * kS1W;
    const float dc = v * 0.25f;
    float* base = c1 + (size_t)((b * kC1N + n) * kC1W + 2 * pp) * kC1W + 2 * q;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const float o = base[dy * kC1W + dx];
        base[dy * kC1W + dx] = (dc * o) * (1.0f - o);
      }
  }
};

inline int gk2_splits(int64_t m) {
  const int64_t k = m * kC2Pos;
  int64_t s = k / 2048;
  if (s > 42) s = 42;
  return s < 1 ? 1 : (int)s;
}

// ---- one SGD group ------------------------------------------------------------------------------------
struct StepArgs {
  const float* images;    // [m][64*64] of this group
  const int32_t* labels;  // [m]
  float* params;          // [kNParam]
  int64_t m;
  float rate;
  bool tensor;            // GEMM engine: tcgen05 3xTF32 (true) or FP32 CUDA cores (false)
  // workspaces (capacity >= m images)
  float* c1;   // [m][32][60][60], dz1 in place
  float* s1;   // [m][32][30][30]
  float* c2;   // [m][64][26][26]
  float* s2;   // [m][10816]
  float* dz;   // [m][10]
  float* loss; // [m]
  float* dz2;  // [m][64][34][34], zero border of 4 (kDzPad)
  float* dz2t; // [64][m*676]: dz2 transposed (the conv2 weight-gradient GEMM's B operand)
  float* bimg; // tensor-core engine: pre-split B stage images (<= 400 KB)
  float* part;   // [42][801][64] split-K partials of g_k2
  float* part1;  // [m][32][26] conv1 gradient partials
  float* grad;   // [kNParam]
  double* epoch_loss;  // running fp64 epoch loss (nullable)
  int first, last;
  double n_total;
};

cudaError_t step(const StepArgs& a, cudaStream_t st);
cudaError_t forward(const StepArgs& a, float* yhat, cudaStream_t st);
cudaError_t gemm_only(int which, bool tensor, const StepArgs& a, cudaStream_t st);

// tcgen05 engine (wide_tc.cu)
constexpr size_t kBImgBytes = 50 * 2 * 32 * 32 * 4;  // max over ops: chunks x (hi|lo) x N x 32 fp32
cudaError_t tc_gemm(const OpConv2Fwd& op, int splits, cudaStream_t st);
cudaError_t tc_gemm(const OpGk2& op, int splits, cudaStream_t st);
cudaError_t tc_gemm(const OpBackin& op, int splits, cudaStream_t st);

}  // namespace wide
}  // namespace tlb
