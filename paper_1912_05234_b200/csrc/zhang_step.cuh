// zhang_step.cuh -- one CTA runs the whole Zhang-CNN training cell of one image out of shared memory.
//
// Reference path (proj/src/network.cpp:81-169, kernels proj/src/nn.cpp:96-217):
//   c1 = sigmoid(mconv(I,k1,b1)); s1 = avgpool(c1); c2 = sigmoid(mconv(s1,k2,b2)); s2 = avgpool(c2);
//   out = sigmoid(mconv(s2,fc,b)); loss = 1/2 sum (y-out)^2; hand backprop FC -> C2 -> C1.
//
// Every stage below maps the reference's per-output computation onto CTA threads.  With EXACT=true
// each output is produced by ONE thread in exactly the reference's summation order with separately
// rounded products (no FMA), the glibc expf restatement and IEEE division, so results are bitwise
// identical to the reference (SURVEY.md §8(a) numerics contract).  With EXACT=false the same stages
// use FFMA and split the long C1 weight-gradient sums across threads (within the 1e-4 tolerance).
//
// Shared-memory working set per CTA (floats): params 3904 | image x2 1568 | c1 3456 | s1 864 |
// c2 768 | s2 192 | out 16 | dz 16 | red 1088 | grad accumulator 3904  (= 63 KB + tables).
#pragma once

#include "tlb_common.cuh"

namespace tlb {

struct Smem {
  float* P;
  float* img;  // two image buffers of kImg floats (double-buffered TMA ring)
  float* c1;  // c1, then dz1 in place
  float* s1;
  float* c2;  // c2, then dz2 in place
  float* s2;
  float* out;
  float* dz;
  float* red;
  float* G;
  float* dzp;  // dz2 zero-padded by 4 on every side: [12][16][16]; border stays 0
  uint64_t* tab;
  uint64_t* bar;
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

constexpr int kDzp = 12 * 16 * 16;
constexpr int kSmemFloats = kPStride + 2 * kImg + 3456 + 864 + 768 + 192 + 16 + 16 + 1088 + kPStride + kDzp;
constexpr size_t kSmemBytes = sizeof(float) * kSmemFloats + 32 * sizeof(uint64_t) + 2 * sizeof(uint64_t);

__device__ __forceinline__ Smem carve_smem(float* base) {
  Smem s;
  float* p = base;
  s.P = p; p += kPStride;
  s.img = p; p += 2 * kImg;
  s.c1 = p; p += 3456;
  s.s1 = p; p += 864;
  s.c2 = p; p += 768;
  s.s2 = p; p += 192;
  s.out = p; p += 16;
  s.dz = p; p += 16;
  s.red = p; p += 1088;
  s.G = p; p += kPStride;
  s.dzp = p; p += kDzp;
  s.tab = reinterpret_cast<uint64_t*>(p);
  s.bar = s.tab + 32;
  s.tr = nullptr;
  return s;
}

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

// Parameters (3,898 floats, padded) global -> shared.  __ldcg: other CTAs rewrote them in the
// previous step's SGD phase, so bypass L1.
__device__ __forceinline__ void load_params(const Smem& s, const float* params) {
  const float4* src = reinterpret_cast<const float4*>(params);
  float4* dst = reinterpret_cast<float4*>(s.P);
  constexpr int kBatch = 4;  // issue every load before the first shared store
  for (int base = threadIdx.x; base < kPStride / 4; base += kBatch * blockDim.x) {
    float4 v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (base + u * (int)blockDim.x < kPStride / 4) v[u] = __ldcg(src + base + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (base + u * (int)blockDim.x < kPStride / 4) dst[base + u * blockDim.x] = v[u];
  }
}

// ---------------------------------------------------------------------------------------------
// Forward stages (net::forward, network.cpp:81-95)
// ---------------------------------------------------------------------------------------------

// C1: mconv(I,k1,b1) -> sigmoid -> avgpool, fused.  Item = (channel i, pooled row py, 8-wide
// column strip xs): the thread computes the 2x8 conv outputs feeding 4 pooled outputs.
// Per output: taps (ky,kx) row-major (nn.cpp:28-33), then + b1[i] (nn.cpp:123).
template <bool EXACT>
__device__ __forceinline__ void stage_conv1(const Smem& s, const float* img) {
  for (int it = threadIdx.x; it < 216; it += blockDim.x) {
    const int i = it / 36, r = it - i * 36, py = r / 3, xs = r - py * 3;
    const int y0 = 2 * py, x0 = 8 * xs;
    const float* k = s.P + kK1 + i * 25;
    float a0[8], a1[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) a0[o] = a1[o] = 0.0f;
#pragma unroll
    for (int rr = 0; rr < 6; ++rr) {
      const float4* src = reinterpret_cast<const float4*>(img + (y0 + rr) * 28 + x0);
      const float4 v0 = src[0], v1 = src[1], v2 = src[2];
      const float in[12] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w, v2.x, v2.y, v2.z, v2.w};
      if (rr < 5) {
#pragma unroll
        for (int kx = 0; kx < 5; ++kx) {
          const float w = k[rr * 5 + kx];
#pragma unroll
          for (int o = 0; o < 8; ++o) a0[o] = mac<EXACT>(a0[o], in[o + kx], w);
        }
      }
      if (rr >= 1) {
#pragma unroll
        for (int kx = 0; kx < 5; ++kx) {
          const float w = k[(rr - 1) * 5 + kx];
#pragma unroll
          for (int o = 0; o < 8; ++o) a1[o] = mac<EXACT>(a1[o], in[o + kx], w);
        }
      }
    }
    const float b = s.P[kB1 + i];
    float t0[8], t1[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      t0[o] = sigmoid_m<EXACT>(fadd(a0[o], b), s.tab);
      t1[o] = sigmoid_m<EXACT>(fadd(a1[o], b), s.tab);
    }
    float4* d0 = reinterpret_cast<float4*>(s.c1 + (i * 24 + y0) * 24 + x0);
    float4* d1 = reinterpret_cast<float4*>(s.c1 + (i * 24 + y0 + 1) * 24 + x0);
    d0[0] = make_float4(t0[0], t0[1], t0[2], t0[3]);
    d0[1] = make_float4(t0[4], t0[5], t0[6], t0[7]);
    d1[0] = make_float4(t1[0], t1[1], t1[2], t1[3]);
    d1[1] = make_float4(t1[4], t1[5], t1[6], t1[7]);
    float pv[4];
#pragma unroll
    for (int px = 0; px < 4; ++px)  // avgpool (nn.cpp:144): ((p00+p01)+p10)+p11, then *0.25f
      pv[px] = fmul(fadd(fadd(fadd(t0[2 * px], t0[2 * px + 1]), t1[2 * px]), t1[2 * px + 1]), 0.25f);
    *reinterpret_cast<float4*>(s.s1 + (i * 12 + py) * 12 + 4 * xs) = make_float4(pv[0], pv[1], pv[2], pv[3]);
  }
}

// C2: mconv(s1,k2,b2) -> sigmoid.  Item = (kernel i, row y, 4-wide half-row xh); per output the
// 150 taps run (c, ky, kx) row-major (nn.cpp:14-33).
template <bool EXACT>
__device__ __forceinline__ void stage_conv2(const Smem& s) {
  for (int it = threadIdx.x; it < 192; it += blockDim.x) {
    const int i = it >> 4, r = it & 15, y = r >> 1, xh = r & 1;
    const float* k = s.P + kK2 + i * 150;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 1
    for (int c = 0; c < 6; ++c) {
#pragma unroll
      for (int ky = 0; ky < 5; ++ky) {
        const float4* src = reinterpret_cast<const float4*>(s.s1 + (c * 12 + y + ky) * 12 + 4 * xh);
        const float4 v0 = src[0], v1 = src[1];
        const float in[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int kx = 0; kx < 5; ++kx) {
          const float w = k[(c * 5 + ky) * 5 + kx];
#pragma unroll
          for (int o = 0; o < 4; ++o) acc[o] = mac<EXACT>(acc[o], in[o + kx], w);
        }
      }
    }
    const float b = s.P[kB2 + i];
    float t[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) t[o] = sigmoid_m<EXACT>(fadd(acc[o], b), s.tab);
    *reinterpret_cast<float4*>(s.c2 + (i * 8 + y) * 8 + 4 * xh) = make_float4(t[0], t[1], t[2], t[3]);
  }
}

__device__ __forceinline__ void stage_pool2(const Smem& s) {
  for (int t = threadIdx.x; t < 192; t += blockDim.x) {
    const int c = t >> 4, py = (t >> 2) & 3, px = t & 3;
    const float* q = s.c2 + (c * 8 + 2 * py) * 8 + 2 * px;
    s.s2[t] = fmul(fadd(fadd(fadd(q[0], q[1]), q[8]), q[9]), 0.25f);
  }
}

__device__ __forceinline__ float target_of(int i, int label, const float* y) {
  return y ? y[i] : (i == label ? 1.0f : 0.0f);  // mnist::one_hot (mnist.cpp:161-167)
}

// FC: out[i] = sigmoid(sum_j s2[j]*fc[i][j] + b[i]); also dz = backsigmoid(out - y, out)
// (network.cpp:146-152, nn.cpp:131-133).  EXACT: one thread per output, j in order.
template <bool EXACT>
__device__ __forceinline__ void stage_fc(const Smem& s, int label, const float* y, bool want_dz) {
  if constexpr (EXACT) {
    if (threadIdx.x < 10) {
      const int i = threadIdx.x;
      const float* w = s.P + kFC + i * 192;
      float acc = 0.0f;
#pragma unroll 8
      for (int j = 0; j < 192; ++j) acc = mac<true>(acc, s.s2[j], w[j]);
      const float o = sigmoid_m<EXACT>(fadd(acc, s.P[kB + i]), s.tab);
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
        const float o = sigmoid_m<EXACT>(fadd(acc, s.P[kB + i]), s.tab);
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
// backavgpool (nn.cpp:148-158) and backsigmoid through c2 -> dz2 (in place over c2).
template <bool EXACT, bool ACCUM>
__device__ __forceinline__ void stage_fc_back(const Smem& s, float* row) {
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
        const int y = 2 * py + dy, x = 2 * px + dx;
        const float o = s.c2[(c * 8 + y) * 8 + x];
        s.dzp[(c * 16 + y + 4) * 16 + x + 4] = fmul(fmul(dc, o), fsub(1.0f, o));
      }
  }
}

// C2 backward: g_k2 = conv(s1, dz2[i]) (64 taps, (y,x) row-major), g_b2 = sum_all(dz2[i]),
// d_s1 = sum_i backin(dz2[i], k2[i], s1), then backavgpool + backsigmoid through c1 -> dz1 (in place).
//
// backin runs over the zero-padded dz2 (uniform 5x5 taps, register-blocked 4 outputs per thread).
// The reference's clipped nested sums (nn.cpp:169-189: per i, row sums over u2 from 0, outer sum over
// u1 from 0, then acc += per-i result) only ever see the padded zero products prepended or appended
// to a row/outer sum, and x + (+-0) == x (with +0 + -0 == +0), so EXACT stays bit-identical while
// executing 259,200 instead of 115,200 multiply-adds per image.
template <bool EXACT, bool ACCUM>
__device__ __forceinline__ void stage_conv2_back(const Smem& s, float* row) {
  for (int it = threadIdx.x; it < 588; it += blockDim.x) {
    if (it < 216) {
      const int c = it / 36, r = it - c * 36, p = r / 3, qq = r - p * 3;
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 1
      for (int i = 0; i < 12; ++i) {
        const float* kk = s.P + kK2 + (i * 6 + c) * 25;
        float outer[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int u1 = 0; u1 < 5; ++u1) {
          const float4* dp = reinterpret_cast<const float4*>(s.dzp + (i * 16 + p - u1 + 4) * 16 + 4 * qq);
          const float4 a = dp[0], b = dp[1];
          const float d[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
          float rs[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
          for (int u2 = 0; u2 < 5; ++u2) {
            const float w = kk[u1 * 5 + u2];
#pragma unroll
            for (int o = 0; o < 4; ++o) {
              if constexpr (EXACT) rs[o] = mac<true>(rs[o], w, d[o - u2 + 4]);
              else acc[o] = __fmaf_rn(w, d[o - u2 + 4], acc[o]);
            }
          }
          if constexpr (EXACT) {
#pragma unroll
            for (int o = 0; o < 4; ++o) outer[o] = fadd(outer[o], rs[o]);
          }
        }
        if constexpr (EXACT) {
#pragma unroll
          for (int o = 0; o < 4; ++o) acc[o] = fadd(acc[o], outer[o]);
        }
      }
      // backavgpool (x0.25) + backsigmoid through c1 for the 2x8 block this thread owns
#pragma unroll
      for (int dy = 0; dy < 2; ++dy) {
        float4* cp = reinterpret_cast<float4*>(s.c1 + (c * 24 + 2 * p + dy) * 24 + 8 * qq);
        const float4 v0 = cp[0], v1 = cp[1];
        float cv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const float dc = fmul(acc[x >> 1], 0.25f);
          cv[x] = fmul(fmul(dc, cv[x]), fsub(1.0f, cv[x]));
        }
        cp[0] = make_float4(cv[0], cv[1], cv[2], cv[3]);
        cp[1] = make_float4(cv[4], cv[5], cv[6], cv[7]);
      }
    } else if (it < 576) {
      const int t = it - 216, i = t / 30, r = t - i * 30, c = r / 5, u = r - c * 5;
      float acc[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 2
      for (int y = 0; y < 8; ++y) {
        const float4* sp = reinterpret_cast<const float4*>(s.s1 + (c * 12 + u + y) * 12);
        const float4 a = sp[0], b = sp[1], cc = sp[2];
        const float sr[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, cc.x, cc.y, cc.z, cc.w};
        const float4* dp = reinterpret_cast<const float4*>(s.dzp + (i * 16 + y + 4) * 16 + 4);
        const float4 d0 = dp[0], d1 = dp[1];
        const float dr[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
        for (int x = 0; x < 8; ++x)
#pragma unroll
          for (int v = 0; v < 5; ++v) acc[v] = mac<EXACT>(acc[v], sr[v + x], dr[x]);
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) put<ACCUM>(s, row, kK2 + ((i * 6 + c) * 5 + u) * 5 + v, acc[v]);
    } else {
      const int i = it - 576;
      float acc = 0.0f;
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        const float4* dp = reinterpret_cast<const float4*>(s.dzp + (i * 16 + y + 4) * 16 + 4);
        const float4 d0 = dp[0], d1 = dp[1];
        acc = fadd(fadd(fadd(fadd(acc, d0.x), d0.y), d0.z), d0.w);
        acc = fadd(fadd(fadd(fadd(acc, d1.x), d1.y), d1.z), d1.w);
      }
      put<ACCUM>(s, row, kB2 + i, acc);
    }
  }
}

// C1 backward: g_k1[i][u][v] = sum_{y,x<24} I[u+y][v+x]*dz1[i][y][x]; g_b1[i] = sum dz1[i].
// EXACT: one thread per output, 576 terms in order.  Fast: 4-row partials + fixed-order combine.
template <bool EXACT, bool ACCUM>
__device__ __forceinline__ void stage_conv1_back(const Smem& s, const float* img, float* row) {
  const float* dz1 = s.c1;
  if constexpr (EXACT) {
    for (int it = threadIdx.x; it < 156; it += blockDim.x) {
      if (it < 150) {
        const int i = it / 25, r = it - i * 25, u = r / 5, v = r - u * 5;
        float acc = 0.0f;
#pragma unroll 1
        for (int y = 0; y < 24; ++y) {
          const float* ir = img + (u + y) * 28 + v;
          const float4* dp = reinterpret_cast<const float4*>(dz1 + (i * 24 + y) * 24);
#pragma unroll
          for (int x4 = 0; x4 < 6; ++x4) {
            const float4 d = dp[x4];
            acc = mac<true>(acc, ir[4 * x4 + 0], d.x);
            acc = mac<true>(acc, ir[4 * x4 + 1], d.y);
            acc = mac<true>(acc, ir[4 * x4 + 2], d.z);
            acc = mac<true>(acc, ir[4 * x4 + 3], d.w);
          }
        }
        put<ACCUM>(s, row, kK1 + it, acc);
      } else {
        const int i = it - 150;
        const float4* dp = reinterpret_cast<const float4*>(dz1 + i * 576);
        float acc = 0.0f;
#pragma unroll 4
        for (int e = 0; e < 144; ++e) {
          const float4 d = dp[e];
          acc = fadd(fadd(fadd(fadd(acc, d.x), d.y), d.z), d.w);
        }
        put<ACCUM>(s, row, kB1 + i, acc);
      }
    }
  } else {
    for (int it = threadIdx.x; it < 216; it += blockDim.x) {
      if (it < 180) {
        const int i = it / 30, r = it - i * 30, u = r / 6, yq = r - u * 6;
        float acc[5] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 1
        for (int y = 4 * yq; y < 4 * yq + 4; ++y) {
          const float4* ip = reinterpret_cast<const float4*>(img + (u + y) * 28);
          float ir[28];
#pragma unroll
          for (int q = 0; q < 7; ++q) {
            const float4 t = ip[q];
            ir[4 * q] = t.x; ir[4 * q + 1] = t.y; ir[4 * q + 2] = t.z; ir[4 * q + 3] = t.w;
          }
          const float4* dp = reinterpret_cast<const float4*>(dz1 + (i * 24 + y) * 24);
#pragma unroll
          for (int x4 = 0; x4 < 6; ++x4) {
            const float4 d = dp[x4];
            const float dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
            for (int xx = 0; xx < 4; ++xx)
#pragma unroll
              for (int v = 0; v < 5; ++v) acc[v] = __fmaf_rn(ir[4 * x4 + xx + v], dv[xx], acc[v]);
          }
        }
#pragma unroll
        for (int v = 0; v < 5; ++v) s.red[it * 5 + v] = acc[v];
      } else {
        const int j = it - 180, i = j / 6, yq = j - i * 6;
        const float4* dp = reinterpret_cast<const float4*>(dz1 + i * 576 + yq * 96);
        float acc = 0.0f;
#pragma unroll 4
        for (int e = 0; e < 24; ++e) {
          const float4 d = dp[e];
          acc += (d.x + d.y) + (d.z + d.w);
        }
        s.red[900 + j] = acc;
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 156; t += blockDim.x) {
      float acc = 0.0f;
      if (t < 150) {
        const int i = t / 25, r = t - i * 25, u = r / 5, v = r - u * 5;
#pragma unroll
        for (int yq = 0; yq < 6; ++yq) acc += s.red[((i * 30) + u * 6 + yq) * 5 + v];
        put<ACCUM>(s, row, kK1 + t, acc);
      } else {
        const int i = t - 150;
#pragma unroll
        for (int yq = 0; yq < 6; ++yq) acc += s.red[900 + i * 6 + yq];
        put<ACCUM>(s, row, kB1 + i, acc);
      }
    }
  }
}

// Whole forward pass of one image (image already in shared memory).
template <bool EXACT>
__device__ __forceinline__ void forward_image(const Smem& s, const float* img, int label, const float* y,
                                              bool want_dz) {
  stage_conv1<EXACT>(s, img);
  __syncthreads();
  mark(s, 3);
  stage_conv2<EXACT>(s);
  __syncthreads();
  mark(s, 4);
  stage_pool2(s);
  __syncthreads();
  mark(s, 5);
  stage_fc<EXACT>(s, label, y, want_dz);
  __syncthreads();
  mark(s, 6);
}

// Whole backward pass (after forward_image with want_dz).  Ends with a __syncthreads.
template <bool EXACT, bool ACCUM>
__device__ __forceinline__ void backward_image(const Smem& s, const float* img, float* row) {
  stage_fc_back<EXACT, ACCUM>(s, row);
  __syncthreads();
  mark(s, 7);
  stage_conv2_back<EXACT, ACCUM>(s, row);
  __syncthreads();
  mark(s, 8);
  stage_conv1_back<EXACT, ACCUM>(s, img, row);
  __syncthreads();
  mark(s, 9);
}

}  // namespace tlb
