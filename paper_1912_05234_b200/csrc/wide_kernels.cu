// wide_kernels.cu -- the widened CNN of BASELINE.json configs[4] (conv1 32@5x5, conv2 64@32x5x5, 64x64
// inputs, FC 10 from [64,1,13,13]; 160,266 parameters), trained with the reference's per-group
// semantics (network.cpp:209-251: per-example forward/backward, batch-summed gradient, sgd_step) but
// laid out B200-first: activations no longer fit one SM (c1 alone is 460 KB per image), so a step runs
// layer by layer over the whole group with HBM/L2-resident activations, and the three 34.6 M-MAC
// contractions per image are GEMMs over the group:
//
//   conv2 forward   D[(b,y,x), i]        = sum_{(c,ky,kx)} s1[b,c,y+ky,x+kx] * k2[i,c,ky,kx]   K = 800
//   conv2 backin    D[(b,p,q), c]        = sum_{(i,u,v)}   dz2[b,i,p-u,q-v] * k2[i,c,u,v]     K = 1600
//   conv2 weights   D[(c,ky,kx)|1, i]    = sum_{(b,y,x)}   s1[b,c,y+ky,x+kx] * dz2[b,i,y,x]    K = 676 B
//
// Each GEMM is an operand-gather functor (implicit im2col, never materialised) + an epilogue functor
// (bias + sigmoid, backavgpool + backsigmoid through c1, split-K partial).  Two GEMM engines share them:
// the FP32 CUDA-core engine here (register-tiled SIMT, FFMA) and the tcgen05 engine in
// wide_tc.cu (3xTF32 on the 5th-gen tensor cores, TMEM accumulators) -- BASELINE configs[4] asks
// whether the tensor cores pay off at K = 800/1600; bench/sweep measure both.
//
// Every batch reduction runs in a fixed order (deterministic run to run); parity against the reference's
// composed nn:: operators (oracle/widened.py) is within the north-star 1e-4 relative tolerance.
#include <cuda_runtime.h>

#include <cstdint>

#include "tlb_common.cuh"
#include "wide_kernels.cuh"

namespace tlb {
namespace wide {

// ------------------------------------------------------------------------------------------------
// conv1 + bias + sigmoid + avgpool: one CTA per (image, group of 8 kernels).  Thread item = (pooled
// row py, 4-column strip xs): it keeps the 6x8 input window in registers and produces the 2x4 block of
// c1 and the 1x2 block of s1 for each of the 8 kernels (taps (ky,kx) row-major as nn.cpp:28-33).
// ------------------------------------------------------------------------------------------------
constexpr int kC1Group = 8;

__global__ void __launch_bounds__(256) conv1_kernel(const float* __restrict__ images, const float* __restrict__ p,
                                                    float* __restrict__ c1, float* __restrict__ s1) {
  __shared__ __align__(16) float img[kImgW * kImgW];
  __shared__ float w[kC1Group * 25 + kC1Group];
  const int b = blockIdx.x, g = blockIdx.y;
  const float4* src = reinterpret_cast<const float4*>(images + (int64_t)b * kImgW * kImgW);
  for (int i = threadIdx.x; i < kImgW * kImgW / 4; i += blockDim.x) reinterpret_cast<float4*>(img)[i] = __ldg(src + i);
  for (int i = threadIdx.x; i < kC1Group * 25; i += blockDim.x) w[i] = __ldg(p + kOffK1 + g * kC1Group * 25 + i);
  if (threadIdx.x < kC1Group) w[kC1Group * 25 + threadIdx.x] = __ldg(p + kOffB1 + g * kC1Group + threadIdx.x);
  __syncthreads();
  for (int it = threadIdx.x; it < 30 * 15; it += blockDim.x) {
    const int py = it / 15, xs = it - py * 15, y0 = 2 * py, x0 = 4 * xs;
    float win[6][8];
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      const float4 a = *reinterpret_cast<const float4*>(img + (y0 + r) * kImgW + x0);
      const float4 c = *reinterpret_cast<const float4*>(img + (y0 + r) * kImgW + x0 + 4);
      win[r][0] = a.x; win[r][1] = a.y; win[r][2] = a.z; win[r][3] = a.w;
      win[r][4] = c.x; win[r][5] = c.y; win[r][6] = c.z; win[r][7] = c.w;
    }
#pragma unroll 1
    for (int k = 0; k < kC1Group; ++k) {
      float acc[2][4] = {};
#pragma unroll
      for (int ky = 0; ky < 5; ++ky)
#pragma unroll
        for (int kx = 0; kx < 5; ++kx) {
          const float wv = w[k * 25 + ky * 5 + kx];
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int o = 0; o < 4; ++o) acc[r][o] = __fmaf_rn(win[r + ky][o + kx], wv, acc[r][o]);
        }
      const float bias = w[kC1Group * 25 + k];
      float t[2][4];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int o = 0; o < 4; ++o) t[r][o] = __frcp_rn(1.0f + __expf(-(acc[r][o] + bias)));
      const int ch = g * kC1Group + k;
      float* dst = c1 + ((int64_t)(b * kC1N + ch) * kC1W + y0) * kC1W + x0;
      *reinterpret_cast<float4*>(dst) = make_float4(t[0][0], t[0][1], t[0][2], t[0][3]);
      *reinterpret_cast<float4*>(dst + kC1W) = make_float4(t[1][0], t[1][1], t[1][2], t[1][3]);
      const float p0 = (((t[0][0] + t[0][1]) + t[1][0]) + t[1][1]) * 0.25f;
      const float p1 = (((t[0][2] + t[0][3]) + t[1][2]) + t[1][3]) * 0.25f;
      *reinterpret_cast<float2*>(s1 + ((int64_t)(b * kC1N + ch) * kS1W + py) * kS1W + 2 * xs) = make_float2(p0, p1);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// FP32 CUDA-core GEMM engine: D[M,N] (+)= A[M,K] B[N,K]^T over k in this CTA's split, operands gathered
// by the op functor, 128 x BN tile, BK = 16, 256 threads with an 8 x (BN/16) register tile, register
// prefetch of the next k-chunk while the current one is multiplied.
// ------------------------------------------------------------------------------------------------
template <class Op, int BN>
__global__ void __launch_bounds__(256) simt_gemm_kernel(Op op) {
  constexpr int BM = 128, BK = 16, TN = BN / 16;
  constexpr int AL = BM * BK / 256, BL = BN * BK / 256;  // gathered elements per thread per chunk
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  int64_t k0, k1;
  op.k_range(blockIdx.z, k0, k1);
  float acc[8][TN];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) acc[r][c] = 0.0f;
  float ra[AL], rb[BL];
  auto gather = [&](int64_t kb) {
#pragma unroll
    for (int j = 0; j < AL; ++j) {
      int64_t m, k;
      if constexpr (Op::kAContigM) {
        m = m0 + (tid & (BM - 1));
        k = kb + (tid >> 7) + 2 * j;
      } else {
        k = kb + (tid & (BK - 1));
        m = m0 + (tid >> 4) + 16 * j;
      }
      ra[j] = (m < op.M && k < k1) ? op.a(m, k) : 0.0f;
    }
#pragma unroll
    for (int j = 0; j < BL; ++j) {
      const int64_t k = kb + (tid & (BK - 1));
      const int n = n0 + (tid >> 4) + 16 * j;
      rb[j] = (n < op.N && k < k1) ? op.b(n, k) : 0.0f;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int j = 0; j < AL; ++j) {
      if constexpr (Op::kAContigM) As[(tid >> 7) + 2 * j][tid & (BM - 1)] = ra[j];
      else As[tid & (BK - 1)][(tid >> 4) + 16 * j] = ra[j];
    }
#pragma unroll
    for (int j = 0; j < BL; ++j) Bs[tid & (BK - 1)][(tid >> 4) + 16 * j] = rb[j];
  };
  if (k0 < k1) gather(k0);
  for (int64_t kb = k0; kb < k1; kb += BK) {
    __syncthreads();
    stash();
    __syncthreads();
    if (kb + BK < k1) gather(kb + BK);  // next chunk's loads overlap this chunk's FFMAs
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float bv[TN];
      if constexpr (TN == 4) {
        const float4 b0 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
        bv[0] = b0.x; bv[1] = b0.y; bv[2] = b0.z; bv[3] = b0.w;
      } else {
        const float2 b0 = *reinterpret_cast<const float2*>(&Bs[kk][tx * 2]);
        bv[0] = b0.x; bv[1] = b0.y;
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) acc[r][c] = __fmaf_rn(av[r], bv[c], acc[r][c]);
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int64_t m = m0 + ty * 8 + r;
    if (m >= op.M) continue;
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      const int n = n0 + tx * TN + c;
      if (n < op.N) op.store(blockIdx.z, m, n, acc[r][c]);
    }
  }
}

template <class Op, int BN>
cudaError_t simt_gemm(const Op& op, int splits, cudaStream_t st) {
  const dim3 grid((unsigned)((op.M + 127) / 128), (unsigned)((op.N + BN - 1) / BN), (unsigned)splits);
  simt_gemm_kernel<Op, BN><<<grid, 256, 0, st>>>(op);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// Per-image FC layer: avgpool(c2) -> s2, out = sigmoid(fc . s2 + b), loss and dz (network.cpp:97-109,
// 146-152), then d_s2 = sum_o fc[o] dz[o] (backin with a singleton error, kernel order), backavgpool and
// backsigmoid through c2 -> dz2.  One 512-thread CTA per image; s2 stays in shared memory.
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(512) fc_kernel(const float* __restrict__ c2, const float* __restrict__ p,
                                                 const int32_t* __restrict__ labels, float* __restrict__ s2g,
                                                 float* __restrict__ dzg, float* __restrict__ lossg,
                                                 float* __restrict__ dz2, float* __restrict__ dz2t, int64_t m) {
  __shared__ float s2[kS2Len];
  __shared__ float red[16][kClasses];
  __shared__ float dz[kClasses];
  const int b = blockIdx.x;
  const float* c2b = c2 + (int64_t)b * kC2N * kC2Pos;
  for (int j = threadIdx.x; j < kS2Len; j += blockDim.x) {
    const int i = j / 169, r = j - i * 169, py = r / 13, px = r - py * 13;
    const float* q = c2b + i * kC2Pos + (2 * py) * kC2W + 2 * px;
    const float v = (((q[0] + q[1]) + q[kC2W]) + q[kC2W + 1]) * 0.25f;
    s2[j] = v;
    s2g[(int64_t)b * kS2Len + j] = v;
  }
  __syncthreads();
  float part[kClasses];
#pragma unroll
  for (int o = 0; o < kClasses; ++o) part[o] = 0.0f;
  for (int j = threadIdx.x; j < kS2Len; j += blockDim.x) {
    const float v = s2[j];
#pragma unroll
    for (int o = 0; o < kClasses; ++o) part[o] = __fmaf_rn(v, __ldg(p + kOffFC + o * kS2Len + j), part[o]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 0; o < kClasses; ++o) {
    float v = part[o];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp][o] = v;
  }
  __syncthreads();
  if (threadIdx.x < kClasses) {
    const int o = threadIdx.x;
    float z = 0.0f;
    for (int w = 0; w < 16; ++w) z += red[w][o];
    const float out = __frcp_rn(1.0f + __expf(-(z + __ldg(p + kOffBF + o))));
    const float y = (o == labels[b]) ? 1.0f : 0.0f;
    dz[o] = ((out - y) * out) * (1.0f - out);
    dzg[b * kClasses + o] = dz[o];
    red[0][o] = (y - out) * (y - out);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float acc = 0.0f;
    for (int o = 0; o < kClasses; ++o) acc += red[0][o];
    lossg[b] = 0.5f * acc;
  }
  for (int j = threadIdx.x; j < kS2Len; j += blockDim.x) {
    float ds = 0.0f;
#pragma unroll
    for (int o = 0; o < kClasses; ++o) ds = __fmaf_rn(__ldg(p + kOffFC + o * kS2Len + j), dz[o], ds);
    const float dc = ds * 0.25f;
    const int i = j / 169, r = j - i * 169, py = r / 13, px = r - py * 13;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const int pos = (2 * py + dy) * kC2W + 2 * px + dx;
        const float o = c2[((int64_t)b * kC2N + i) * kC2Pos + pos];
        const float v = (dc * o) * (1.0f - o);
        dz2[((int64_t)b * kC2N + i) * kDzPlane + (2 * py + dy + kDzPad) * kDzW + 2 * px + dx + kDzPad] = v;
        dz2t[(int64_t)i * (m * kC2Pos) + (int64_t)b * kC2Pos + pos] = v;
      }
  }
}

// g_fc[o][j] = sum_b s2[b][j] dz[b][o] and g_b[o] = sum_b dz[b][o], example order.
__global__ void gfc_kernel(const float* __restrict__ s2, const float* __restrict__ dz, int64_t m, float* __restrict__ g) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < (int64_t)kClasses * kS2Len) {
    const int o = (int)(t / kS2Len), j = (int)(t - (int64_t)o * kS2Len);
    float acc = 0.0f;
    for (int64_t b = 0; b < m; ++b) acc = __fmaf_rn(s2[b * kS2Len + j], dz[b * kClasses + o], acc);
    g[kOffFC + t] = acc;
  } else if (t < (int64_t)kClasses * kS2Len + kClasses) {
    const int o = (int)(t - (int64_t)kClasses * kS2Len);
    float acc = 0.0f;
    for (int64_t b = 0; b < m; ++b) acc += dz[b * kClasses + o];
    g[kOffBF + o] = acc;
  }
}

// Split-K partials of the conv2 weight/bias gradient -> g_k2[i][c][ky][kx], g_b2[i] (fixed split order).
__global__ void gk2_reduce_kernel(const float* __restrict__ part, int splits, float* __restrict__ g) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= kGk2Rows * kC2N) return;
  float acc = 0.0f;
  for (int z = 0; z < splits; ++z) acc += part[(int64_t)z * kGk2Rows * kC2N + t];
  const int m = t / kC2N, i = t - m * kC2N;
  if (m < kK2Slice) g[kOffK2 + i * kK2Slice + m] = acc;
  else g[kOffB2 + i] = acc;
}

// conv1 weight/bias gradient partials per (image, kernel): 25 taps over the 60x60 dz1 plane + its sum.
__global__ void __launch_bounds__(256) gk1_kernel(const float* __restrict__ images, const float* __restrict__ dz1,
                                                  float* __restrict__ part) {
  __shared__ __align__(16) float img[kImgW * kImgW];
  __shared__ float red[8][26];
  const int b = blockIdx.x, i = blockIdx.y;
  const float4* src = reinterpret_cast<const float4*>(images + (int64_t)b * kImgW * kImgW);
  for (int t = threadIdx.x; t < kImgW * kImgW / 4; t += blockDim.x) reinterpret_cast<float4*>(img)[t] = __ldg(src + t);
  __syncthreads();
  const float* d = dz1 + (int64_t)(b * kC1N + i) * kC1W * kC1W;
  float acc[26];
#pragma unroll
  for (int k = 0; k < 26; ++k) acc[k] = 0.0f;
  for (int pos = threadIdx.x; pos < kC1W * kC1W; pos += blockDim.x) {
    const int y = pos / kC1W, x = pos - y * kC1W;
    const float dv = d[pos];
#pragma unroll
    for (int u = 0; u < 5; ++u)
#pragma unroll
      for (int v = 0; v < 5; ++v) acc[u * 5 + v] = __fmaf_rn(img[(u + y) * kImgW + v + x], dv, acc[u * 5 + v]);
    acc[25] += dv;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 26; ++k) {
    float v = acc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 26) {
    float v = 0.0f;
    for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
    part[((int64_t)b * kC1N + i) * 26 + threadIdx.x] = v;
  }
}

// Sum the per-image conv1 partials (example order), the group's fp64 loss (example order), then
// sgd_step (network.cpp:171-180) over all 160,266 parameters.
__global__ void gk1_reduce_kernel(const float* __restrict__ part, int64_t m, float* __restrict__ g) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= kC1N * 26) return;
  float acc = 0.0f;
  for (int64_t b = 0; b < m; ++b) acc += part[b * kC1N * 26 + t];
  const int i = t / 26, k = t - i * 26;
  if (k < 25) g[kOffK1 + i * 25 + k] = acc;
  else g[kOffB1 + i] = acc;
}

__global__ void sgd_kernel(float* __restrict__ p, const float* __restrict__ g, float rate, float m) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < kNParam) p[t] = __fsub_rn(p[t], __fmul_rn(rate, __fdiv_rn(g[t], m)));
}

__global__ void loss_kernel(const float* __restrict__ loss, int64_t m, double* __restrict__ epoch_loss, int first,
                            int last, double n_total) {
  double acc = first ? 0.0 : epoch_loss[0];
  for (int64_t b = 0; b < m; ++b) acc += (double)loss[b];
  epoch_loss[0] = last ? acc / n_total : acc;
}

// ------------------------------------------------------------------------------------------------
// Host driver: one SGD group.
// ------------------------------------------------------------------------------------------------
cudaError_t step(const StepArgs& a, cudaStream_t st) {
  const int64_t m = a.m;
  cudaError_t e;
  conv1_kernel<<<dim3((unsigned)m, kC1N / kC1Group), 256, 0, st>>>(a.images, a.params, a.c1, a.s1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  OpConv2Fwd f{a.s1, a.params, a.c2, m * kC2Pos, a.bimg};
  if ((e = a.tensor ? tc_gemm(f, 1, st) : simt_gemm<OpConv2Fwd, 64>(f, 1, st)) != cudaSuccess) return e;
  fc_kernel<<<(unsigned)m, 512, 0, st>>>(a.c2, a.params, a.labels, a.s2, a.dz, a.loss, a.dz2, a.dz2t, m);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  gfc_kernel<<<(kClasses * kS2Len + kClasses + 255) / 256, 256, 0, st>>>(a.s2, a.dz, m, a.grad);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  OpGk2 gk{a.s1, a.dz2t, a.part, m * kC2Pos, gk2_splits(m)};
  if ((e = a.tensor ? tc_gemm(gk, gk.splits, st) : simt_gemm<OpGk2, 64>(gk, gk.splits, st)) != cudaSuccess) return e;
  gk2_reduce_kernel<<<(kGk2Rows * kC2N + 255) / 256, 256, 0, st>>>(a.part, gk.splits, a.grad);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  OpBackin bi{a.dz2, a.params, a.c1, m * kS1Pos, a.bimg};
  if ((e = a.tensor ? tc_gemm(bi, 1, st) : simt_gemm<OpBackin, 32>(bi, 1, st)) != cudaSuccess) return e;
  gk1_kernel<<<dim3((unsigned)m, kC1N), 256, 0, st>>>(a.images, a.c1, a.part1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  gk1_reduce_kernel<<<(kC1N * 26 + 127) / 128, 128, 0, st>>>(a.part1, m, a.grad);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  sgd_kernel<<<(kNParam + 255) / 256, 256, 0, st>>>(a.params, a.grad, a.rate, (float)m);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (a.epoch_loss) {
    loss_kernel<<<1, 1, 0, st>>>(a.loss, m, a.epoch_loss, a.first, a.last, a.n_total);
    e = cudaGetLastError();
  }
  return e;
}

// Forward only (inference): conv1, conv2 GEMM, then the FC head without the backward part.
__global__ void __launch_bounds__(512) fc_forward_kernel(const float* __restrict__ c2, const float* __restrict__ p,
                                                         float* __restrict__ yhat) {
  __shared__ float s2[kS2Len];
  __shared__ float red[16][kClasses];
  const int b = blockIdx.x;
  const float* c2b = c2 + (int64_t)b * kC2N * kC2Pos;
  for (int j = threadIdx.x; j < kS2Len; j += blockDim.x) {
    const int i = j / 169, r = j - i * 169, py = r / 13, px = r - py * 13;
    const float* q = c2b + i * kC2Pos + (2 * py) * kC2W + 2 * px;
    s2[j] = (((q[0] + q[1]) + q[kC2W]) + q[kC2W + 1]) * 0.25f;
  }
  __syncthreads();
  float part[kClasses];
#pragma unroll
  for (int o = 0; o < kClasses; ++o) part[o] = 0.0f;
  for (int j = threadIdx.x; j < kS2Len; j += blockDim.x) {
    const float v = s2[j];
#pragma unroll
    for (int o = 0; o < kClasses; ++o) part[o] = __fmaf_rn(v, __ldg(p + kOffFC + o * kS2Len + j), part[o]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 0; o < kClasses; ++o) {
    float v = part[o];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp][o] = v;
  }
  __syncthreads();
  if (threadIdx.x < kClasses) {
    float z = 0.0f;
    for (int w = 0; w < 16; ++w) z += red[w][threadIdx.x];
    yhat[b * kClasses + threadIdx.x] = __frcp_rn(1.0f + __expf(-(z + __ldg(p + kOffBF + threadIdx.x))));
  }
}

cudaError_t forward(const StepArgs& a, float* yhat, cudaStream_t st) {
  const int64_t m = a.m;
  conv1_kernel<<<dim3((unsigned)m, kC1N / kC1Group), 256, 0, st>>>(a.images, a.params, a.c1, a.s1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  OpConv2Fwd f{a.s1, a.params, a.c2, m * kC2Pos, a.bimg};
  if ((e = a.tensor ? tc_gemm(f, 1, st) : simt_gemm<OpConv2Fwd, 64>(f, 1, st)) != cudaSuccess) return e;
  fc_forward_kernel<<<(unsigned)m, 512, 0, st>>>(a.c2, a.params, yhat);
  return cudaGetLastError();
}

// Stand-alone GEMM entry points for the engine comparison (bench / tests): run one of the three
// contractions with either engine on the caller's activations.
cudaError_t gemm_only(int which, bool tensor, const StepArgs& a, cudaStream_t st) {
  const int64_t m = a.m;
  if (which == 0) {
    OpConv2Fwd f{a.s1, a.params, a.c2, m * kC2Pos, a.bimg};
    return tensor ? tc_gemm(f, 1, st) : simt_gemm<OpConv2Fwd, 64>(f, 1, st);
  }
  if (which == 1) {
    OpGk2 gk{a.s1, a.dz2t, a.part, m * kC2Pos, gk2_splits(m)};
    return tensor ? tc_gemm(gk, gk.splits, st) : simt_gemm<OpGk2, 64>(gk, gk.splits, st);
  }
  OpBackin bi{a.dz2, a.params, a.c1, m * kS1Pos, a.bimg};
  return tensor ? tc_gemm(bi, 1, st) : simt_gemm<OpBackin, 32>(bi, 1, st);
}

}  // namespace wide
}  // namespace tlb
