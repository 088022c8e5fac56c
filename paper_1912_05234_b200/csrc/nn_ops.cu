// nn_ops.cu -- the reference's rank-polymorphic layer ops (tloom::nn, proj/src/nn.cpp:37-217) as
// generic sm_100a kernels: one thread per output element, each computing the reference's exact
// per-element summation order (bitwise identical).  These serve the drop-in op API (tlb_nn_*); the
// training hot path uses the fused fixed-shape kernels in zhang_kernels.cu instead.
#include <cuda_runtime.h>

#include <cstdint>

#include "tlb_common.cuh"
#include "tlb_launch.h"

namespace tlb {

struct Shp {
  int64_t e[8];
  int r;
};

__host__ __device__ inline int64_t shp_count(const Shp& s) {
  int64_t c = 1;
  for (int a = 0; a < s.r; ++a) c *= s.e[a];
  return c;
}

__device__ inline void shp_strides(const Shp& s, int64_t* st) {
  int64_t acc = 1;
  for (int a = s.r - 1; a >= 0; --a) {
    st[a] = acc;
    acc *= s.e[a];
  }
}

__device__ inline void unflatten(const Shp& s, int64_t flat, int64_t* iv) {
  for (int a = s.r - 1; a >= 0; --a) {
    iv[a] = s.e[a] > 0 ? flat % s.e[a] : 0;
    if (s.e[a] > 0) flat /= s.e[a];
  }
}

__device__ inline void load_tab(uint64_t* tab) {
  if (threadIdx.x < 32) tab[threadIdx.x] = exp_tab_entry(threadIdx.x);
  __syncthreads();
}

// conv / mconv (nn.cpp:96-125): out[i, iv] = (sum over row-major taps ov of in[iv+ov]*k[i][ov]) (+ b[i]).
__global__ void conv_kernel(const float* in, Shp is, const float* k, Shp ks, Shp os, const float* bias,
                            int64_t nk, float* out) {
  const int64_t per = shp_count(os), total = per * nk, nt = shp_count(ks);
  int64_t ist[8];
  shp_strides(is, ist);
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = o / per, rem = o - i * per;
    int64_t iv[8], ov[8];
    unflatten(os, rem, iv);
    int64_t base = 0;
    for (int a = 0; a < is.r; ++a) base += iv[a] * ist[a];
    const float* kk = k + i * nt;
    float acc = 0.0f;
    for (int64_t t = 0; t < nt; ++t) {
      unflatten(ks, t, ov);
      int64_t off = 0;
      for (int a = 0; a < ks.r; ++a) off += ov[a] * ist[a];
      acc = __fadd_rn(acc, __fmul_rn(in[base + off], kk[t]));
    }
    out[o] = bias ? __fadd_rn(acc, bias[i]) : acc;
  }
}

__global__ void sigmoid_kernel(const float* x, int64_t n, float* out) {
  __shared__ uint64_t tab[32];
  load_tab(tab);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sigmoid_ref(x[i], tab);
}

// backsigmoid (nn.cpp:131-133): d * o * (1 - o)
__global__ void backsigmoid_kernel(const float* d, const float* o, int64_t n, float* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __fmul_rn(__fmul_rn(d[i], o[i]), __fsub_rn(1.0f, o[i]));
}

// avgpool (nn.cpp:135-146) over the trailing two axes.
__global__ void avgpool_kernel(const float* in, Shp is, Shp os, float* out) {
  const int64_t n = shp_count(os);
  int64_t st[8];
  shp_strides(is, st);
  const int r = is.r;
  const int64_t row = st[r - 2];
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t iv[8];
    unflatten(os, o, iv);
    int64_t base = 0;
    for (int a = 0; a < r; ++a) base += iv[a] * st[a] * (a >= r - 2 ? 2 : 1);
    const float s = __fadd_rn(__fadd_rn(__fadd_rn(in[base], in[base + 1]), in[base + row]), in[base + row + 1]);
    out[o] = __fmul_rn(s, 0.25f);
  }
}

// backavgpool (nn.cpp:148-158): out[iv] = d[iv with trailing coords halved] * 0.25f
__global__ void backavgpool_kernel(const float* d, Shp ds, Shp os, float* out) {
  const int64_t n = shp_count(os);
  int64_t st[8];
  shp_strides(ds, st);
  const int r = ds.r;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t iv[8];
    unflatten(os, o, iv);
    int64_t base = 0;
    for (int a = 0; a < r; ++a) base += (a >= r - 2 ? iv[a] / 2 : iv[a]) * st[a];
    out[o] = __fmul_rn(d[base], 0.25f);
  }
}

struct Box {
  const float* d;
  const float* k;
  int64_t dst[8], kst[8], cnt[8];
  int r;
};

// BackinBox::sum (nn.cpp:169-189): nested per-axis sums, innermost axis first, each level starting
// from 0.0f.  Iterative (explicit per-level accumulators) instead of device recursion.
__device__ float box_sum(const Box& b, int64_t dbase, int64_t kbase) {
  float acc[8];
  int64_t u[8], doff[8], koff[8];
  int l = 0;
  acc[0] = 0.0f;
  u[0] = 0;
  doff[0] = dbase;
  koff[0] = kbase;
  for (;;) {
    float done;
    if (l == b.r - 1) {
      float s = 0.0f;
      for (int64_t v = 0; v < b.cnt[l]; ++v) s = __fadd_rn(s, __fmul_rn(b.k[koff[l] + v], b.d[doff[l] - v]));
      done = s;
    } else if (u[l] < b.cnt[l]) {
      doff[l + 1] = doff[l] - u[l] * b.dst[l];
      koff[l + 1] = koff[l] + u[l] * b.kst[l];
      ++l;
      acc[l] = 0.0f;
      u[l] = 0;
      continue;
    } else {
      done = acc[l];
    }
    if (l == 0) return done;
    --l;
    acc[l] = __fadd_rn(acc[l], done);
    ++u[l];
  }
}

// backin (nn.cpp:193-217): clipped correlation of the error with the kernel.
__global__ void backin_kernel(const float* d, Shp ds, const float* k, Shp ks, Shp os, float* out) {
  const int64_t n = shp_count(os);
  Box b;
  b.d = d;
  b.k = k;
  b.r = os.r;
  shp_strides(ds, b.dst);
  shp_strides(ks, b.kst);
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    if (os.r == 0) {
      out[0] = __fmul_rn(d[0], k[0]);
      continue;
    }
    int64_t iv[8];
    unflatten(os, o, iv);
    int64_t dbase = 0, kbase = 0;
    Box bb = b;
    for (int a = 0; a < os.r; ++a) {
      const int64_t i = iv[a];
      const int64_t off = i < ds.e[a] ? 0 : i - ds.e[a] + 1;
      int64_t c = ds.e[a] < i + 1 ? ds.e[a] : i + 1;
      if (ks.e[a] - off < c) c = ks.e[a] - off;
      bb.cnt[a] = c;
      dbase += (i - off) * b.dst[a];
      kbase += off * b.kst[a];
    }
    out[o] = box_sum(bb, dbase, kbase);
  }
}

// net::loss (network.cpp:97-109) per row: 0.5f * sum_i (y_i - yhat_i)^2, i in order.
__global__ void loss_kernel(const float* yhat, const float* y, int64_t n, float* out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.0f;
    for (int i = 0; i < 10; ++i) {
      const float d = __fsub_rn(y[r * 10 + i], yhat[r * 10 + i]);
      acc = __fadd_rn(acc, __fmul_rn(d, d));
    }
    out[r] = __fmul_rn(0.5f, acc);
  }
}

// sum_all (tensor.cpp:310-314): sequential from 0.0f (one thread; exact order).
__global__ void sum_all_kernel(const float* x, int64_t n, float* out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    float acc = 0.0f;
    for (int64_t i = 0; i < n; ++i) acc = __fadd_rn(acc, x[i]);
    *out = acc;
  }
}

__global__ void expf_kernel(const float* x, int64_t n, float* out) {
  __shared__ uint64_t tab[32];
  load_tab(tab);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = glibc_expf(x[i], tab);
}

__global__ void expf_range_kernel(uint32_t start, int64_t n, float* out) {
  __shared__ uint64_t tab[32];
  load_tab(tab);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = glibc_expf(__uint_as_float(start + (uint32_t)i), tab);
}

// ---- launchers ---------------------------------------------------------------------------------
static Shp mk(const int64_t* e, int r) {
  Shp s{};
  s.r = r;
  for (int a = 0; a < r; ++a) s.e[a] = e[a];
  return s;
}

static int blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return (int)b;
}

cudaError_t nn_conv(const float* in, const int64_t* is, const float* k, const int64_t* ks, int r,
                    const float* bias, int64_t nk, float* out, cudaStream_t st) {
  int64_t os[8];
  for (int a = 0; a < r; ++a) os[a] = is[a] - ks[a] + 1;
  const Shp O = mk(os, r);
  const int64_t total = shp_count(O) * nk;
  if (total > 0) conv_kernel<<<blocks_for(total), 256, 0, st>>>(in, mk(is, r), k, mk(ks, r), O, bias, nk, out);
  return cudaGetLastError();
}

cudaError_t nn_sigmoid(const float* x, int64_t n, float* out, cudaStream_t st) {
  if (n > 0) sigmoid_kernel<<<blocks_for(n), 256, 0, st>>>(x, n, out);
  return cudaGetLastError();
}

cudaError_t nn_backsigmoid(const float* d, const float* o, int64_t n, float* out, cudaStream_t st) {
  if (n > 0) backsigmoid_kernel<<<blocks_for(n), 256, 0, st>>>(d, o, n, out);
  return cudaGetLastError();
}

cudaError_t nn_avgpool(const float* in, const int64_t* s, int r, float* out, cudaStream_t st) {
  int64_t os[8];
  for (int a = 0; a < r; ++a) os[a] = a >= r - 2 ? s[a] / 2 : s[a];
  const Shp O = mk(os, r);
  const int64_t n = shp_count(O);
  if (n > 0) avgpool_kernel<<<blocks_for(n), 256, 0, st>>>(in, mk(s, r), O, out);
  return cudaGetLastError();
}

cudaError_t nn_backavgpool(const float* d, const int64_t* s, int r, float* out, cudaStream_t st) {
  int64_t os[8];
  for (int a = 0; a < r; ++a) os[a] = a >= r - 2 ? s[a] * 2 : s[a];
  const Shp O = mk(os, r);
  const int64_t n = shp_count(O);
  if (n > 0) backavgpool_kernel<<<blocks_for(n), 256, 0, st>>>(d, mk(s, r), O, out);
  return cudaGetLastError();
}

cudaError_t nn_backin(const float* d, const int64_t* ds, const float* k, const int64_t* ks, int r, float* out,
                      cudaStream_t st) {
  int64_t os[8];
  for (int a = 0; a < r; ++a) os[a] = ds[a] + ks[a] - 1;
  const Shp O = mk(os, r);
  const int64_t n = shp_count(O);
  if (n > 0) backin_kernel<<<blocks_for(n), 128, 0, st>>>(d, mk(ds, r), k, mk(ks, r), O, out);
  return cudaGetLastError();
}

cudaError_t nn_loss(const float* yhat, const float* y, int64_t n, float* out, cudaStream_t st) {
  if (n > 0) loss_kernel<<<blocks_for(n), 256, 0, st>>>(yhat, y, n, out);
  return cudaGetLastError();
}

cudaError_t nn_sum_all(const float* x, int64_t n, float* out, cudaStream_t st) {
  sum_all_kernel<<<1, 32, 0, st>>>(x, n, out);
  return cudaGetLastError();
}

cudaError_t nn_expf(const float* x, int64_t n, float* out, cudaStream_t st) {
  if (n > 0) expf_kernel<<<blocks_for(n), 256, 0, st>>>(x, n, out);
  return cudaGetLastError();
}

cudaError_t nn_expf_range(uint32_t start_bits, int64_t n, float* out, cudaStream_t st) {
  if (n > 0) expf_range_kernel<<<blocks_for(n), 256, 0, st>>>(start_bits, n, out);
  return cudaGetLastError();
}

}  // namespace tlb
