// stage_bench.cu -- developer micro-benchmark for the per-image stages of zhang_step.cuh.
//
// One 512-thread CTA per SM (148 CTAs, like the batch-100 train kernel) repeats one stage `iters`
// times on deterministic pseudo-random shared-memory contents; thread 0 measures clock64 across the
// loop.  Prints one JSON line per (mode, stage, variant) with the median cycles and us per call.
// Not part of the product library; build: python -m paper_1912_05234_b200.build --bench
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "stage_variants.cuh"

using namespace tlb;

enum Stage { kConv1, kConv2V0, kConv2V1, kFc, kFcBack, kC2BackV0, kC2BackV1, kC2BackV2, kC2BackV3, kC1Back, kForward,
             kBackwardV0, kBackwardV1, kBackinV4, kBackinV5, kC1BackGk2, kBackwardV4, kBackwardV5, kC2BackV6, kC2BackV7, kBackwardV6, kBackwardV7, kC2BackV8, kBackwardV8,
             kBackinV9, kBackwardV9, kC2BackV10, kBackwardV10, kBackwardV11, kBackwardV12, kBackwardV13, kConv2V2, kBackwardV14,
             kBackwardProduct, kC2BackProduct, kC1BackProduct, kNumStages };
static const char* kNames[kNumStages] = {"conv1", "conv2_v0_halves", "conv2_v1_rows", "fc", "fc_back",
                                         "conv2_back_v0_quads", "conv2_back_v1_items", "conv2_back_v2_pairs", "conv2_back_v3_ws", "conv1_back",
                                         "forward_image", "backward_v0", "backward_v1",
                                         "backin_only_v4_items", "backin_only_v5_quads", "c1back_with_gk2",
                                         "backward_v4", "backward_v5", "conv2_back_v6_rows2", "conv2_back_v7_rows4",
                                         "backward_v6", "backward_v7", "conv2_back_v8_rows4p", "backward_v8",
                                         "backin_only_v9_rows4p", "backward_v9", "conv2_back_v10_split_gk2",
                                         "backward_v10", "backward_v11_gk160", "backward_v12_gk192",
                                         "backward_v13_gk128", "conv2_v2_rows_p", "backward_v14_gk2rows",
                                         "backward_product", "conv2_back_product", "conv1_back_product"};

__device__ __forceinline__ float hrand(unsigned int x) {  // deterministic value in [0, 1)
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return (x >> 8) * (1.0f / 16777216.0f);
}

__device__ void fill(const Smem& s) {
  const int t = threadIdx.x, n = blockDim.x;
  for (int i = t; i < kPStride; i += n) s.P[i] = i < kNParam ? (hrand(i) - 0.5f) * 0.2f : 0.0f;
  for (int i = t; i < 2 * kImg; i += n) s.img[i] = hrand(i + 10000);
  for (int i = t; i < kC1Floats; i += n) s.c1[i] = 0.3f + 0.4f * hrand(i + 20000);
  for (int i = t; i < 864; i += n) s.s1[i] = 0.3f + 0.4f * hrand(i + 30000);
  for (int i = t; i < 768; i += n) s.c2[i] = 0.3f + 0.4f * hrand(i + 40000);
  for (int i = t; i < 192; i += n) s.s2[i] = 0.3f + 0.4f * hrand(i + 50000);
  if (t < 16) { s.out[t] = 0.5f; s.dz[t] = (hrand(t + 60000) - 0.5f) * 0.1f; }
  for (int i = t; i < kPStride; i += n) s.G[i] = 0.0f;
  __syncthreads();
  for (int idx = t; idx < kKp; idx += n) {
    const int row = idx >> 3, k = idx & 7;
    s.Kp[idx] = k < 5 ? s.P[kK2 + row * 5 + k] : 0.0f;
  }
#if TLB_PAIR
  __syncthreads();
#endif
  for (int q = t; q < 12 * 64; q += n) {
    const int i = q >> 6, y = (q >> 3) & 7, x = q & 7;
    s.dzp[dzp_at(i, y + 4, x + 4)] = (hrand(q + 70000) - 0.5f) * 0.01f;
  }
  build_shifted(s, s.img, t, n);
  __syncthreads();
}

template <bool EXACT, int STAGE>
__device__ __forceinline__ void run_stage(const Smem& s, float* row) {
  constexpr bool A = !EXACT;
  if constexpr (STAGE == kBackwardProduct) {
    backward_image<EXACT, A>(s, s.img, row);
    return;
  }
  if constexpr (STAGE == kC2BackProduct) {
    call_conv2_back<EXACT, A>(row);
    return;
  }
  if constexpr (STAGE == kC1BackProduct) {
    call_conv1_back<EXACT, A>(s.img, row);
    return;
  }
  if constexpr (STAGE == kConv1) stage_conv1<EXACT>(s, s.img);
  else if constexpr (STAGE == kConv2V0) stage_conv2<EXACT, 0>(s);
  else if constexpr (STAGE == kConv2V1) stage_conv2<EXACT, 1>(s);
  else if constexpr (STAGE == kConv2V2) stage_conv2<EXACT, 2>(s);
  else if constexpr (STAGE == kFc) stage_fc<EXACT>(s, 3, nullptr, true);
  else if constexpr (STAGE == kFcBack) stage_fc_back<EXACT, A>(s, row);
  else if constexpr (STAGE == kC2BackV0) stage_conv2_back_legacy<EXACT, A, 0>(s, row);
  else if constexpr (STAGE == kC2BackV1) stage_conv2_back_legacy<EXACT, A, 1>(s, row);
  else if constexpr (STAGE == kC2BackV2) stage_conv2_back_legacy<EXACT, A, 2>(s, row);
  else if constexpr (STAGE == kC2BackV3) stage_conv2_back_legacy<EXACT, A, 3>(s, row);
  else if constexpr (STAGE == kC1Back) stage_conv1_back<EXACT, A>(s, s.img, row);
  else if constexpr (STAGE == kForward) forward_image<EXACT>(s, s.img, 3, nullptr, true);
  else if constexpr (STAGE == kBackinV4) stage_conv2_back_legacy<EXACT, A, 4>(s, row);
  else if constexpr (STAGE == kBackinV5) stage_conv2_back_legacy<EXACT, A, 5>(s, row);
  else if constexpr (STAGE == kC1BackGk2) stage_conv1_back_gk2_legacy<EXACT, A>(s, s.img, row);
  else if constexpr (STAGE == kC2BackV6 || STAGE == kC2BackV7) {
    if constexpr (!EXACT) stage_conv2_back_legacy<false, A, STAGE == kC2BackV6 ? 6 : 7>(s, row);
  } else if constexpr (STAGE == kBackwardV6 || STAGE == kBackwardV7 || STAGE == kBackwardV8) {
    if constexpr (!EXACT) {
      stage_fc_back<EXACT, A>(s, row);
      __syncthreads();
      stage_conv2_back_legacy<false, A, STAGE == kBackwardV6 ? 6 : STAGE == kBackwardV7 ? 7 : 8>(s, row);
      __syncthreads();
      stage_conv1_back<EXACT, A>(s, s.img, row);
    }
  } else if constexpr (STAGE == kC2BackV8) {
    if constexpr (!EXACT) stage_conv2_back_legacy<false, A, 8>(s, row);
  } else if constexpr (STAGE == kBackinV9) {
    if constexpr (!EXACT) stage_conv2_back_legacy<false, A, 9>(s, row);
  } else if constexpr (STAGE == kC2BackV10) {
    if constexpr (!EXACT) stage_conv2_back_legacy<false, A, 10>(s, row);
  } else if constexpr (STAGE == kBackwardV9 || STAGE == kBackwardV10 || STAGE == kBackwardV11 ||
                       STAGE == kBackwardV12 || STAGE == kBackwardV13 || STAGE == kBackwardV14) {
    if constexpr (!EXACT) {
      constexpr int V = STAGE == kBackwardV9 ? 9 : STAGE == kBackwardV10 ? 10 : STAGE == kBackwardV11 ? 11
                      : STAGE == kBackwardV12 ? 12 : STAGE == kBackwardV13 ? 13 : 14;
      stage_fc_back<EXACT, A>(s, row);
      __syncthreads();
      stage_conv2_back_legacy<false, A, V>(s, row);
      __syncthreads();
      stage_conv1_back_gk2_legacy<false, A, gk2_split_lanes(V), V == 14>(s, s.img, row);
    }
  }
  else if constexpr (STAGE == kBackwardV4 || STAGE == kBackwardV5) {
    stage_fc_back<EXACT, A>(s, row);
    __syncthreads();
    stage_conv2_back_legacy<EXACT, A, STAGE == kBackwardV4 ? 4 : 5>(s, row);
    __syncthreads();
    stage_conv1_back_gk2_legacy<EXACT, A>(s, s.img, row);
  } else if constexpr (STAGE == kBackwardV0) {
    stage_fc_back<EXACT, A>(s, row);
    __syncthreads();
    stage_conv2_back_legacy<EXACT, A, 0>(s, row);
    __syncthreads();
    stage_conv1_back<EXACT, A>(s, s.img, row);
  } else {
    stage_fc_back<EXACT, A>(s, row);
    __syncthreads();
    stage_conv2_back_legacy<EXACT, A, 1>(s, row);
    __syncthreads();
    stage_conv1_back<EXACT, A>(s, s.img, row);
  }
}

template <bool EXACT, int STAGE>
__global__ void __launch_bounds__(kThreads, 1) stage_kernel(float* rows, unsigned long long* cycles, int iters) {
  const Smem s = carve_smem(tlb_smem);
  smem_setup(s);
  fill(s);
  float* row = rows + (size_t)blockIdx.x * kPStride;
  run_stage<EXACT, STAGE>(s, row);  // warm-up
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
    run_stage<EXACT, STAGE>(s, row);
    __syncthreads();
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// One fresh fast run of STAGE (accumulating into G): dump c1 (dz1 after backin) and G.
template <int STAGE>
__global__ void __launch_bounds__(kThreads, 1) verify_kernel(float* out) {
  const Smem s = carve_smem(tlb_smem);
  smem_setup(s);
  fill(s);
  run_stage<false, STAGE>(s, nullptr);
  __syncthreads();
  for (int i = threadIdx.x; i < kC1Floats; i += blockDim.x) out[i] = s.c1[i];
  for (int i = threadIdx.x; i < kPStride; i += blockDim.x) out[kC1Floats + i] = s.G[i];
}

template <int STAGE>
std::vector<float> run_verify(float* d_out) {
  auto k = verify_kernel<STAGE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  k<<<1, kThreads, kSmemBytes>>>(d_out);
  cudaDeviceSynchronize();
  std::vector<float> got(kC1Floats + kPStride);
  cudaMemcpy(got.data(), d_out, got.size() * sizeof(float), cudaMemcpyDeviceToHost);
  return got;
}

template <int STAGE, int REF>
void verify(float* d_out) {
  const std::vector<float> want = run_verify<REF>(d_out), got = run_verify<STAGE>(d_out);
  double md = 0, mv = 0;
  for (size_t i = 0; i < got.size(); ++i) {
    md = std::max(md, (double)std::fabs(got[i] - want[i]));
    mv = std::max(mv, (double)std::fabs(want[i]));
  }
  printf("{\"verify\": \"%s vs %s\", \"max_abs_diff\": %.3e, \"max_abs\": %.3e, \"err\": \"%s\"}\n", kNames[STAGE],
         kNames[REF], md, mv, cudaGetErrorString(cudaGetLastError()));
}

template <bool EXACT, int STAGE>
void measure(float* rows, unsigned long long* d_cycles, int sms, int iters, double mhz) {
  auto k = stage_kernel<EXACT, STAGE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  k<<<sms, kThreads, kSmemBytes>>>(rows, d_cycles, iters);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<unsigned long long> c(sms);
  cudaMemcpy(c.data(), d_cycles, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  std::sort(c.begin(), c.end());
  const double med = (double)c[sms / 2] / iters, mx = (double)c[sms - 1] / iters;
  printf("{\"mode\": \"%s\", \"stage\": \"%s\", \"cycles\": %.0f, \"us\": %.3f, \"us_max_cta\": %.3f, \"err\": \"%s\"}\n",
         EXACT ? "exact" : "fast", kNames[STAGE], med, med / mhz, mx / mhz, cudaGetErrorString(e));
}

template <bool EXACT>
void all(float* rows, unsigned long long* d_cycles, int sms, int iters, double mhz) {
  measure<EXACT, kConv1>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kConv2V0>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kConv2V1>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kConv2V2>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kFc>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kFcBack>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kC2BackV0>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kC2BackV1>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kC2BackV2>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kC2BackV3>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kC1Back>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kForward>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kBackwardV0>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kBackwardV1>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kBackinV4>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kBackinV5>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kC1BackGk2>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kBackwardV4>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kBackwardV5>(rows, d_cycles, sms, iters, mhz);
  if constexpr (!EXACT) {
    measure<EXACT, kC2BackV6>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kC2BackV7>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kBackwardV6>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kBackwardV7>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kC2BackV8>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kBackwardV8>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kBackinV9>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kBackwardV9>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kC2BackV10>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kBackwardV10>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kBackwardV11>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kBackwardV12>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kBackwardV13>(rows, d_cycles, sms, iters, mhz);
    measure<EXACT, kBackwardV14>(rows, d_cycles, sms, iters, mhz);
  }
  measure<EXACT, kC2BackProduct>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kC1BackProduct>(rows, d_cycles, sms, iters, mhz);
  measure<EXACT, kBackwardProduct>(rows, d_cycles, sms, iters, mhz);
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 100;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* rows;
  unsigned long long* d_cycles;
  cudaMalloc(&rows, (size_t)sms * kPStride * sizeof(float));
  cudaMalloc(&d_cycles, sms * sizeof(unsigned long long));
  const double mhz = 1965.0;
  {  // numerics of the fast variants against V1 (same inputs)
    float* d_out;
    cudaMalloc(&d_out, (kC1Floats + kPStride) * sizeof(float));
    verify<kC2BackV6, kC2BackV1>(d_out);
    verify<kC2BackV7, kC2BackV1>(d_out);
    verify<kC2BackV8, kC2BackV1>(d_out);
    verify<kBackwardV9, kBackwardV1>(d_out);
    verify<kBackwardV10, kBackwardV1>(d_out);
    verify<kBackwardV11, kBackwardV1>(d_out);
    verify<kBackwardV13, kBackwardV1>(d_out);
    verify<kBackwardV14, kBackwardV1>(d_out);
    cudaFree(d_out);
  }
  all<false>(rows, d_cycles, sms, iters, mhz);
  all<true>(rows, d_cycles, sms, iters, mhz);
  return 0;
}
