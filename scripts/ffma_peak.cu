// ffma_peak.cu -- measured FP32 FFMA peak of this B200 (the denominator of the FFMA-bound rooflines).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ffma_peak scripts/ffma_peak.cu
//   build/ffma_peak            -> one JSON line
//
// Every thread runs 16 independent FFMA chains (enough ILP to cover the 4-cycle FFMA latency at 4+ warps
// per SM sub-partition), `iters` rounds, on 148 x k CTAs of 512 threads (k = resident CTAs per SM).  The
// SM clock during the run is derived from CTA 0's clock64 delta over the event-timed interval, so the
// line carries both the achieved TFLOP/s and the clock it was reached at.  Repeated `reps` times; best
// and median are reported.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void __launch_bounds__(512) ffma_kernel(float* out, int iters, float a, float b,
                                                   unsigned long long* cycles) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = (float)(threadIdx.x + k);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = __fmaf_rn(x[k], a, b);
  }
  const long long t1 = clock64();
  float s = 0.0f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == 12345.678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // keep the chains live
  if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
}

// Packed variant: 8 independent f32x2 chains (16 floats) per thread, fma.rn.f32x2 (SASS FFMA2, sm_100):
// the same 16 FMAs per round in half the issued instructions.
__global__ void __launch_bounds__(512) ffma2_kernel(float* out, int iters, float a, float b,
                                                    unsigned long long* cycles) {
  unsigned long long x[8], av, bv;
  asm("mov.b64 %0, {%1,%1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1,%1};" : "=l"(bv) : "f"(b));
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float lo = (float)(threadIdx.x + 2 * k), hi = (float)(threadIdx.x + 2 * k + 1);
    asm("mov.b64 %0, {%1,%2};" : "=l"(x[k]) : "f"(lo), "f"(hi));
  }
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[k]) : "l"(av), "l"(bv));
  }
  const long long t1 = clock64();
  float s = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float lo, hi;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[k]));
    s += lo + hi;
  }
  if (s == 12345.678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
}

int main(int argc, char** argv) {
  const bool packed = argc > 3 && argv[3][0] == '2';
  const int iters = argc > 1 ? atoi(argv[1]) : 4096;
  const int reps = argc > 2 ? atoi(argv[2]) : 20;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int per_sm = 0;
  auto kern = packed ? ffma2_kernel : ffma_kernel;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 512, 0);
  const int grid = prop.multiProcessorCount * per_sm;
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, sizeof(float) * grid * 512);
  cudaMalloc(&cyc, sizeof(unsigned long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<<<grid, 512>>>(out, iters, 0.999f, 0.001f, cyc);
  std::vector<double> tf, mhz;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, 512>>>(out, iters, 0.999f, 0.001f, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double flop = 2.0 * 16 * 8 * (double)iters * grid * 512;
    tf.push_back(flop / (ms * 1e-3) / 1e12);
    mhz.push_back((double)c / (ms * 1e-3) / 1e6);
  }
  cudaError_t err = cudaGetLastError();
  std::vector<double> s = tf;
  std::sort(s.begin(), s.end());
  std::vector<double> m = mhz;
  std::sort(m.begin(), m.end());
  const double nominal_at_mhz = prop.multiProcessorCount * 128.0 * 2.0 * m[m.size() / 2] * 1e6 / 1e12;
  printf("{\"what\": \"%s\", \"sm_count\": %d, \"ctas_per_sm\": %d, \"threads\": 512, \"iters\": %d, "
         "\"reps\": %d, \"tflops_best\": %.3f, \"tflops_median\": %.3f, \"sm_mhz_median\": %.1f, "
         "\"nominal_tflops_at_that_clock\": %.3f, \"frac_of_nominal\": %.4f, \"cuda\": \"%s\"}\n",
         packed ? "fp32 ffma2 (fma.rn.f32x2) peak" : "fp32 ffma peak", prop.multiProcessorCount, per_sm, iters, reps, s.back(), s[s.size() / 2], m[m.size() / 2], nominal_at_mhz,
         s[s.size() / 2] / nominal_at_mhz, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
