// synth_device.cu -- synth::make_digits / synth::make_set (proj/src/synth.cpp:117-161) generated on the
// GPU, byte-identical to the reference for every (n, seed).
//
// The reference draws one sequential std::mt19937_64 stream: per image 4 jitter draws (sx, sy, tx, ty)
// then 784 noise draws (pixel row-major), u01 = (rng() >> 40) * 2^-24.  The stream is rebuilt on the
// device in two kernels:
//   1. chain_kernel (one CTA): seeds the 312-word state (std::mersenne_twister_engine::seed) and runs the
//      twist recurrence serially, one __syncthreads per 312 outputs (each of 156 threads produces words
//      i and i+156 of the next state from the current one; word 311's dependency on the new word 0 is
//      recomputed locally), storing a snapshot of the state array at the start of every image segment;
//   2. segment_kernel (one CTA per segment of L images): resumes from its snapshot, twists forward
//      through a 4-array ring as its images need draws, and synthesises the pixels in parallel --
//      bilinear glyph sample + 0.02 u01 noise, clamp, lround(v * 255) -- in double precision with
//      explicitly rounded operations in the reference's evaluation order (no contraction), so every byte
//      equals the host's (x86-64 baseline: no FMA).
// 1 M images take ~0.15 s on one B200 against ~33 s on the host.
#include <cuda_runtime.h>

#include <algorithm>

#include <cstdint>

#include "tlb_common.cuh"
#include "tlb_launch.h"

namespace tlb {
namespace synth {

constexpr int kN = 312, kHalf = 156;
constexpr uint64_t kMatrixA = 0xB5026F5AA96619E9ULL, kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
constexpr int kDraws = 788;  // per image: 4 jitter + 784 noise (synth.cpp:133-146)

__device__ __forceinline__ uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

__device__ __forceinline__ uint64_t twist_word(uint64_t far, uint64_t a, uint64_t b) {
  const uint64_t y = (a & kUpper) | (b & kLower);
  return far ^ (y >> 1) ^ ((y & 1ULL) ? kMatrixA : 0ULL);
}

// nxt = twist(cur); threads 0..155 each produce nxt[i] and nxt[i + 156].
__device__ __forceinline__ void twist(const uint64_t* cur, uint64_t* nxt) {
  const int i = threadIdx.x;
  if (i < kHalf) {
    const uint64_t lo = twist_word(cur[i + kHalf], cur[i], cur[i + 1]);
    nxt[i] = lo;
    if (i + kHalf + 1 < kN) {
      nxt[i + kHalf] = twist_word(lo, cur[i + kHalf], cur[i + kHalf + 1]);
    } else {  // word 311: needs the new word 0 (thread 0's) -- recompute it here
      const uint64_t n0 = twist_word(cur[kHalf], cur[0], cur[1]);
      nxt[kN - 1] = twist_word(lo, cur[kN - 1], n0);
    }
  }
}

// Segment s starts at draw D = 788 * L * s; its draws come from state S_{D/312 + 1} (the array after
// D/312 + 1 twists) at word D % 312.
__host__ __device__ __forceinline__ int64_t seg_twist(int64_t s, int64_t L) { return (kDraws * L * s) / kN + 1; }

__global__ void __launch_bounds__(160) chain_kernel(uint64_t seed, int64_t segments, int64_t L, uint64_t* snaps) {
  __shared__ uint64_t buf[2][kN];
  if (threadIdx.x == 0) {  // std::mersenne_twister_engine<uint_fast64_t, 64, 312, ...>::seed(seed)
    uint64_t v = seed;
    buf[0][0] = v;
    for (int i = 1; i < kN; ++i) {
      v = 6364136223846793005ULL * (v ^ (v >> 62)) + (uint64_t)i;
      buf[0][i] = v;
    }
  }
  __syncthreads();
  int cur = 0;
  int64_t next_seg = 0;
  int64_t want = segments > 0 ? seg_twist(0, L) : -1;
  for (int64_t t = 1; next_seg < segments; ++t) {
    twist(buf[cur], buf[cur ^ 1]);
    __syncthreads();
    cur ^= 1;
    while (next_seg < segments && t == want) {  // several segments can start inside one array
      for (int i = threadIdx.x; i < kN; i += blockDim.x) snaps[next_seg * kN + i] = buf[cur][i];
      ++next_seg;
      want = next_seg < segments ? seg_twist(next_seg, L) : -1;
    }
  }
}

// Glyph table of synth.cpp:14-94 (5x7 font, bit 4 = leftmost column).
__constant__ uint8_t kFont[10][7] = {
    {0x0E, 0x11, 0x13, 0x15, 0x19, 0x11, 0x0E}, {0x04, 0x0C, 0x04, 0x04, 0x04, 0x04, 0x0E},
    {0x0E, 0x11, 0x01, 0x02, 0x04, 0x08, 0x1F}, {0x0E, 0x11, 0x01, 0x06, 0x01, 0x11, 0x0E},
    {0x02, 0x06, 0x0A, 0x12, 0x1F, 0x02, 0x02}, {0x1F, 0x10, 0x1E, 0x01, 0x01, 0x11, 0x0E},
    {0x06, 0x08, 0x10, 0x1E, 0x11, 0x11, 0x0E}, {0x1F, 0x01, 0x02, 0x02, 0x04, 0x04, 0x04},
    {0x0E, 0x11, 0x11, 0x0E, 0x11, 0x11, 0x0E}, {0x0E, 0x11, 0x11, 0x0F, 0x01, 0x02, 0x0C},
};

__device__ __forceinline__ double font_cell(int digit, int gy, int gx) {
  if (gx < 0 || gx > 4 || gy < 0 || gy > 6) return 0.0;
  return ((kFont[digit][gy] >> (4 - gx)) & 1u) ? 1.0 : 0.0;
}

// glyph_sample (synth.cpp:102-113), evaluated left to right with separately rounded operations.
__device__ __forceinline__ double font_sample(int digit, double gx, double gy) {
  const double fx = floor(gx), fy = floor(gy);
  const int ix = (int)fx, iy = (int)fy;
  const double wx = __dsub_rn(gx, fx), wy = __dsub_rn(gy, fy);
  const double ux = __dsub_rn(1.0, wx), uy = __dsub_rn(1.0, wy);
  double v = __dmul_rn(__dmul_rn(font_cell(digit, iy, ix), ux), uy);
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(font_cell(digit, iy, ix + 1), wx), uy));
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(font_cell(digit, iy + 1, ix), ux), wy));
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(font_cell(digit, iy + 1, ix + 1), wx), wy));
  return v;
}

__device__ __forceinline__ double u01_of(uint64_t w) { return __dmul_rn((double)(temper(w) >> 40), 0x1p-24); }

__global__ void __launch_bounds__(256) segment_kernel(int64_t n, int64_t L, const uint64_t* snaps, uint8_t* pixels,
                                                      float* images, int32_t* labels) {
  __shared__ uint64_t ring[4][kN];  // state arrays S_t .. S_{t+3}: draws [312(t-1), 312(t+3))
  const int64_t s = blockIdx.x;
  const int64_t img0 = s * L, img1 = img0 + L < n ? img0 + L : n;
  int64_t t0 = seg_twist(s, L);  // array index held in ring slot t0 % 4 ... t_hi
  for (int i = threadIdx.x; i < kN; i += blockDim.x) ring[t0 & 3][i] = snaps[s * kN + i];
  int64_t t_hi = t0;  // highest array index present
  __syncthreads();
  for (int64_t img = img0; img < img1; ++img) {
    const int64_t d0 = (int64_t)kDraws * img;                 // first draw of this image
    const int64_t need_hi = (d0 + kDraws - 1) / kN + 1;       // array holding its last draw
    while (t_hi < need_hi) {
      twist(ring[t_hi & 3], ring[(t_hi + 1) & 3]);
      __syncthreads();
      ++t_hi;
    }
    auto draw = [&](int64_t d) -> double {  // draw d lives in array d/312 + 1, word d % 312
      const int64_t t = d / kN + 1;
      return u01_of(ring[t & 3][d - (t - 1) * kN]);
    };
    const int digit = (int)(img % 10);
    // uniform(lo, hi) = lo + (hi - lo) * u01 (synth.cpp:128-129)
    const double sx = __dadd_rn(3.3, __dmul_rn(__dsub_rn(3.7, 3.3), draw(d0)));
    const double sy = __dadd_rn(3.3, __dmul_rn(__dsub_rn(3.7, 3.3), draw(d0 + 1)));
    const double tx = __dadd_rn(-0.8, __dmul_rn(__dsub_rn(0.8, -0.8), draw(d0 + 2)));
    const double ty = __dadd_rn(-0.8, __dmul_rn(__dsub_rn(0.8, -0.8), draw(d0 + 3)));
    for (int p = threadIdx.x; p < 784; p += blockDim.x) {
      const int y = p / 28, x = p - y * 28;
      const double gx = __dadd_rn(__ddiv_rn(__dsub_rn(__dsub_rn((double)x, 13.5), tx), sx), 2.0);
      const double gy = __dadd_rn(__ddiv_rn(__dsub_rn(__dsub_rn((double)y, 13.5), ty), sy), 3.0);
      double v = __dadd_rn(font_sample(digit, gx, gy), __dmul_rn(0.02, draw(d0 + 4 + p)));
      v = fmin(fmax(v, 0.0), 1.0);
      const uint8_t b = (uint8_t)llround(__dmul_rn(v, 255.0));
      if (pixels) pixels[img * 784 + p] = b;
      if (images) images[img * 784 + p] = __fdiv_rn((float)b, 255.0f);  // synth::make_set (synth.cpp:155-161)
    }
    if (threadIdx.x == 0 && labels) labels[img] = digit;
    // the ring slot of array t is overwritten only when t + 4 is produced; every thread is past this
    // image's reads once it reaches the next image's twists (the __syncthreads inside the while loop)
    __syncthreads();
  }
}

int64_t segment_images(int64_t n) {
  int64_t L = (n + 2047) / 2048;
  return L < 8 ? 8 : L;
}

size_t snapshot_bytes(int64_t n) {
  const int64_t L = segment_images(n);
  return (size_t)((n + L - 1) / L) * kN * sizeof(uint64_t);
}

cudaError_t make_digits(int64_t n, uint64_t seed, uint64_t* snaps, uint8_t* pixels, float* images, int32_t* labels,
                        cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t L = segment_images(n), segs = (n + L - 1) / L;
  chain_kernel<<<1, 160, 0, st>>>(seed, segs, L, snaps);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  segment_kernel<<<(unsigned)segs, 256, 0, st>>>(n, L, snaps, pixels, images, labels);
  return cudaGetLastError();
}

}  // namespace synth
// ---- byte ingestion: pixel bytes -> fp32 images ------------------------------------------------------
// pixel / 255.0f with IEEE division (mnist.cpp:57, synth.cpp:158): bit-identical to the host conversion.
// HBM-bound: each thread takes 16 bytes (one 128-bit load) and writes four float4s.
__global__ void __launch_bounds__(256) pixels_to_f32_kernel(const uint8_t* __restrict__ src, float* __restrict__ dst,
                                                            int64_t count) {
  const int64_t nvec = count >> 4;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(src) + v);
    const uint32_t word[4] = {w.x, w.y, w.z, w.w};
    float4* d = reinterpret_cast<float4*>(dst) + 4 * v;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      d[q] = make_float4(__fdiv_rn((float)(word[q] & 0xffu), 255.0f), __fdiv_rn((float)((word[q] >> 8) & 0xffu), 255.0f),
                         __fdiv_rn((float)((word[q] >> 16) & 0xffu), 255.0f), __fdiv_rn((float)(word[q] >> 24), 255.0f));
  }
  // tail (count % 16 bytes) and unaligned callers are handled bytewise by the first threads
  for (int64_t i = (nvec << 4) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __fdiv_rn((float)src[i], 255.0f);
}

__global__ void __launch_bounds__(256) pixels_to_f32_scalar(const uint8_t* __restrict__ src, float* __restrict__ dst,
                                                            int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __fdiv_rn((float)src[i], 255.0f);
}

cudaError_t launch_pixels_to_f32(const uint8_t* src, float* dst, int64_t count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int64_t work = (count + 15) / 16;
  const int grid = (int)std::min<int64_t>((work + 255) / 256, 148 * 8);
  const bool aligned = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
  if (aligned) pixels_to_f32_kernel<<<grid, 256, 0, st>>>(src, dst, count);
  else pixels_to_f32_scalar<<<grid, 256, 0, st>>>(src, dst, count);
  return cudaGetLastError();
}

}  // namespace tlb
