// tlb_common.cuh -- shared constants and sm_100a device helpers for the tensorloom-B200 kernels.
//
// Layout constants mirror the reference's Zhang network (proj/src/network.cpp:17-23) and its flat
// gradient/parameter order (write_flat, network.cpp:186-193).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tlb {

// ---- flat parameter / gradient layout (k1, b1, k2, b2, fc, b) -------------------------------
constexpr int kK1 = 0, kB1 = 150, kK2 = 156, kB2 = 1956, kFC = 1968, kB = 3888;
constexpr int kNParam = 3898;  // kGradFloats, network.cpp:184
constexpr int kPStride = 3904;  // padded row (16-B multiple): params, grad rows, partials
constexpr int kLossSlot = 3898; // per-example loss rides in the padding of a grad row

// ---- per-image activation layout (net::ActCache, network.hpp:35-42) -------------------------
constexpr int kC1 = 0, kS1 = 3456, kC2 = 4320, kS2 = 5088, kOut = 5280;
constexpr int kNAct = 5290;
constexpr int kImg = 784;  // 28x28 fp32 = 3,136 B per image

// ---- arithmetic: EXACT = reference order, no contraction (the bitwise parity mode) ----------
template <bool EXACT>
__device__ __forceinline__ float mac(float acc, float a, float b) {
  if constexpr (EXACT) return __fadd_rn(acc, __fmul_rn(a, b));
  else return __fmaf_rn(a, b, acc);
}
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }

// glibc 2.39 expf (the reference's std::exp(float), IFUNC FMA variant), restated bit-exactly:
// oracle/tloom_oracle.c:orc_expf_port is checked against host libm on every float in [-104, 89],
// and this device copy against host libm by tests/test_gpu_parity.py.  `tab` is the 32-entry
// exp2 table (in shared memory so divergent lookups do not serialise on the constant cache).
__device__ __forceinline__ float glibc_expf(float x, const uint64_t* tab) {
  const uint32_t ux = __float_as_uint(x);
  const uint32_t abstop = (ux >> 20) & 0x7ffu;
  if (abstop >= 0x42bu) {  // |x| >= 88 or nan
    if (ux == 0xff800000u) return 0.0f;
    if (abstop >= 0x7f8u) return __fadd_rn(x, x);
    if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
    if (x < -0x1.9fe368p6f) return 0.0f;
  }
  const double xd = (double)x;
  const double kInvLn2N = 0x1.71547652b82fep+5, kShift = 0x1.8p+52;
  double kd = __fma_rn(kInvLn2N, xd, kShift);
  const uint64_t ki = (uint64_t)__double_as_longlong(kd);
  kd = __dsub_rn(kd, kShift);
  const double r = __fma_rn(kInvLn2N, xd, -kd);
  const uint64_t t = tab[ki & 31u] + (ki << 47);
  const double s = __longlong_as_double((long long)t);
  const double z = __fma_rn(0x1.c6af84b912394p-20, r, 0x1.ebfce50fac4f3p-13);
  const double r2 = __dmul_rn(r, r);
  double y = __fma_rn(0x1.62e42ff0c52d6p-6, r, 1.0);
  y = __fma_rn(z, r2, y);
  y = __dmul_rn(y, s);
  return __double2float_rn(y);
}

// nn::sigmoid (nn.cpp:127-129): 1.0f / (1.0f + expf(-x)).  1.0f / y correctly rounded is exactly
// the IEEE reciprocal __frcp_rn(y), so the divide costs a reciprocal, not a general division.
__device__ __forceinline__ float sigmoid_ref(float x, const uint64_t* tab) {
  return __frcp_rn(__fadd_rn(1.0f, glibc_expf(-x, tab)));
}

// Mode-dependent logistic: EXACT = the reference's bits; fast = ex2.approx-based exp and the MUFU
// reciprocal (rcp.approx, ~1 ulp; 1 + e^-x >= 1, so no subnormal input, and inputs above 2^126 flush
// the result to +0 as the logistic should) -- two MUFU ops instead of the IEEE reciprocal sequence.
__device__ __forceinline__ float rcp_approx(float y) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));
  return r;
}
template <bool EXACT>
__device__ __forceinline__ float sigmoid_m(float x, const uint64_t* tab) {
  if constexpr (EXACT) return sigmoid_ref(x, tab);
  else return rcp_approx(1.0f + __expf(-x));
}

// glibc's __exp2f_data.tab (N = 32): asuint64(2^(i/32)) - (i << 47); copied to shared memory.
__constant__ uint64_t kExpTab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL,
};
__device__ __forceinline__ uint64_t exp_tab_entry(int i) { return kExpTab[i]; }

// ---- non-negative 64-bit quotient / remainder with a 32-bit fast path ------------------------------
// The persistent kernels recompute step/example indices per job on every thread; the 64-bit integer
// division is a ~100-instruction software routine, the 32-bit one a few instructions.
__host__ __device__ __forceinline__ int64_t udiv(int64_t a, int64_t b) {
#ifdef __CUDA_ARCH__
  if ((((uint64_t)a | (uint64_t)b) >> 32) == 0) return (int64_t)((uint32_t)a / (uint32_t)b);
#endif
  return a / b;
}
__host__ __device__ __forceinline__ int64_t umod(int64_t a, int64_t b) { return a - udiv(a, b) * b; }

// ---- static_chunk (runtime.cpp:138-145): ceil-block split of [0,n) over `workers` -------------
__host__ __device__ __forceinline__ void static_chunk(int64_t n, int workers, int w, int64_t& lo,
                                                      int64_t& hi) {
  if (n <= workers) {  // block of 1 (or 0): no division
    lo = w < n ? w : n;
    hi = w + 1 < n ? w + 1 : n;
    return;
  }
  const int64_t block = udiv(n + workers - 1, workers);
  lo = (int64_t)w * block;
  if (lo > n) lo = n;
  hi = lo + block;
  if (hi > n) hi = n;
}

// ---- PTX helpers: shared addresses, mbarrier, 1-D bulk TMA, grid barrier --------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TLB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TLB_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 4-byte global -> shared async copy (own commit group); the issuing thread completes it with
// cp_async_wait_all() and a later CTA barrier publishes it.
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// cp.async.bulk global -> shared, completion signalled on `bar` (TMA 1-D bulk copy; SASS UBLKCP).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Sense-free grid barrier for a cooperative (co-resident) launch.  `target` advances by gridDim.x
// on every call; the counter is zeroed by the host before each launch.
// Device-wide nanosecond clock (same time base on every SM; profiling stamps).
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}

__device__ __forceinline__ void grid_sync(unsigned int* counter, unsigned int& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
    while (v < target) {
      __nanosleep(32);  // back off so 148 pollers do not starve the arrivals on the same L2 line
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
    }
  }
  __syncthreads();
}

// Named CTA barriers (id 0 is __syncthreads): producers arrive, consumers sync (or vice versa).
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- thread-block clusters / distributed shared memory ----------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// Full cluster barrier with release/acquire semantics on shared::cluster (DSMEM) accesses.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Address of the same shared-memory object in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t dsmem_map(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 dsmem_ld4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ void dsmem_st4(uint32_t addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
// Asynchronous DSMEM stores into CTA `rank`'s shared memory that complete_tx on that CTA's mbarrier
// (addr and bar are shared::cluster addresses from dsmem_map): the receiver waits on its own mbarrier
// for the expected byte count instead of a cluster-wide release/acquire barrier.
__device__ __forceinline__ void st_async_v4(uint32_t addr, float4 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async_f32(uint32_t addr, float v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(addr), "f"(v), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async_f64(uint32_t addr, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(addr), "d"(v),
               "r"(bar)
               : "memory");
}
// Wait for phase `parity` of a local mbarrier whose transactions come from other CTAs of the cluster.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TLB_WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TLB_WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Bounded variant (fused data parallelism: a cluster peer that gave up on a dead GPU never pushes):
// false after `limit` cycles without the phase completing.
__device__ __forceinline__ bool mbar_wait_cluster_for(uint64_t* bar, uint32_t parity, long long limit) {
  const long long t0 = clock64();
  for (;;) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return true;
    if (clock64() - t0 > limit) return false;
  }
}
// Guarded wait of the single-GPU clustered kernel: returns when the phase completes, or -- so that a
// co-tenant that starves a cluster, or any other protocol failure, fails the call instead of hanging the
// device -- after `limit` cycles, raising *abort; once *abort is raised every guarded wait of the launch
// falls through at once (the host then reports the failure).  The abort word is polled only every 256
// tries, so the common wait (a few hundred cycles) pays no global-memory round trip.
__device__ __forceinline__ void mbar_wait_cluster_guarded(uint64_t* bar, uint32_t parity, long long limit,
                                                          unsigned int* abort) {
  long long t0 = 0;
  for (unsigned int n = 0;; ++n) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (n == 0) t0 = clock64();
    if ((n & 255u) == 255u) {
      if (*reinterpret_cast<volatile unsigned int*>(abort)) return;
      if (clock64() - t0 > limit) {
        atomicExch(abort, 1u);
        return;
      }
    }
  }
}

__device__ __forceinline__ void dsmem_st(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ double dsmem_ld_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}

}  // namespace tlb
