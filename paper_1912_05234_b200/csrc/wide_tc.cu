// wide_tc.cu -- tcgen05 (5th-gen tensor core) GEMM engine for the widened CNN's three conv2 contractions,
// fp32-accurate through 3xTF32: every operand x is split into hi = x with the low 13 mantissa bits
// cleared (exactly TF32) and lo = x - hi (exact in fp32), and D += Ahi*Bhi + Ahi*Blo + Alo*Bhi, all
// accumulated in fp32 in TMEM (the dropped Alo*Blo term and lo's own TF32 truncation are ~2^-21 relative).
//
// One 128 x N tile per CTA (N = 64 or 32 = the whole GEMM width), K streamed in 32-float chunks through a
// 4-stage shared-memory ring:
//   warps 0-7  producers: gather the chunk's A (128 x 32) and B (N x 32) operands through the op functor
//              (implicit im2col, never materialised in HBM), split hi/lo, store them in the K-major
//              SWIZZLE_128B layout the UMMA descriptors describe, fence.proxy.async, arrive on full[s];
//   warp 8     one elected lane issues 4 k-steps x 3 tcgen05.mma.kind::tf32 (M=128, N, K=8) per chunk
//              into the TMEM accumulator and tcgen05.commit's the stage back to the producers;
//   warps 0-3  epilogue: tcgen05.ld (32 lanes x 32 bit, one accumulator row per thread) -> op.store.
#include <cuda_runtime.h>

#include <cstdint>

#include "tlb_common.cuh"
#include "wide_kernels.cuh"

namespace tlb {
namespace wide {
namespace {

constexpr int kBM = 128, kBK = 32, kStages = 2;  // 2 stages x 2 CTAs per SM: twice the gathers in flight
constexpr int kProducers = 256, kThreadsTC = kProducers + 32;

template <int N>
struct TcCfg {
  static constexpr int kABytes = kBM * kBK * 4;  // 16 KB
  static constexpr int kBBytes = N * kBK * 4;
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kSmem = kStages * kStageBytes + 1024;  // + alignment slack (SW128 atoms: 1 KB)
  // + the column-offset tables of ops with a static K (int32 A and B offsets)
  static constexpr int kTmemCols = N < 32 ? 32 : N;
  // kind::tf32 instruction descriptor: D f32 (bits 4-5 = 1), A/B tf32 (bits 7-9, 10-12 = 2), both
  // K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28.
  static constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                                     ((uint32_t)(kBM >> 4) << 24);
};

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: rows of 128 B, 8-row atoms 1024 B apart (SBO),
// version 1 (sm_100), layout type 2.  LBO is unused when the tile's K extent is one swizzle atom.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
}

// 16-byte chunk j of row r in a K-major SWIZZLE_128B tile.
__device__ __forceinline__ uint32_t sw128_off(int r, int j) { return (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4)); }

template <class Op>
constexpr int tc_smem_bytes() {
  return kStages * TcCfg<Op::N>::kStageBytes + 2 * (Op::kKTab > 0 ? Op::kKTab : 1) * (int)sizeof(int) +
         (2 * kStages + 2) * 8;
}

template <class Op>
__global__ void __launch_bounds__(kThreadsTC, 2) tc_gemm_kernel(Op op) {
  constexpr int N = Op::N;
  using Cfg = TcCfg<N>;
  constexpr int kTab = Op::kKTab > 0 ? Op::kKTab : 1;
  // Dynamic shared memory only (no static __shared__), so the window starts 1024-B aligned and every
  // pointer below stays in the shared state space (LDS/STS, not generic LD/ST):
  //   [stages x (Ahi|Alo|Bhi|Blo)] [A/B column tables] [mbarriers full/empty/done] [TMEM slot]
  extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
  uint8_t* const base = tc_smem_raw;
  uint64_t* const full = reinterpret_cast<uint64_t*>(base + kStages * Cfg::kStageBytes + 2 * kTab * sizeof(int));
  uint64_t* const empty = full + kStages;
  uint64_t* const done_bar = empty + kStages;
  uint32_t* const tmem_slot_p = reinterpret_cast<uint32_t*>(done_bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.x * kBM;
  int64_t k0, k1;
  op.k_range(blockIdx.z, k0, k1);
  const int nchunks = k1 > k0 ? (int)((k1 - k0 + kBK - 1) / kBK) : 0;

  int* const acol = reinterpret_cast<int*>(base + kStages * Cfg::kStageBytes);  // [kKTab] when K is static
  int* const bcol = acol + kTab;
  if constexpr (Op::kKTab > 0) {
    for (int k = tid; k < Op::kKTab; k += blockDim.x) {
      acol[k] = (int)op.a_col(k);
      bcol[k] = (int)op.b_col(k);
    }
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], kProducers + (Op::kBImage ? 1 : 0));  // + the B image's expect_tx arrival
      mbar_init(&empty[s], 1);
    }
    mbar_init(done_bar, 1);
    fence_barrier_init();
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot_p)),
                 "r"(Cfg::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_p;

  if (warp < 8) {
    // ---- producers: thread t owns A row t % 128 (16 of the chunk's 32 k) and B row t % N (32*N/256 k).
    // All of a chunk's gathers are issued before any is consumed, and chunk c+1's gathers are in flight
    // while chunk c is split and stored (register double-buffer), so L2 latency overlaps the stores. ----
    constexpr int kPerRowB = kProducers / N;  // threads per B row (4 or 8)
    constexpr int kBElems = kBK / kPerRowB;   // B elements per thread per chunk (8 or 4)
    const int ra_r = tid & (kBM - 1), ra_kh = tid >> 7;
    // B row / part: dense rows take consecutive threads along the row (coalesced float4 gathers)
    const int rb_r = Op::kBDense ? tid / kPerRowB : tid % N, rb_part = Op::kBDense ? tid % kPerRowB : tid / N;
    const int64_t m = m0 + ra_r;
    const bool mv = m < op.M, ones = op.a_ones(m);
    const float* __restrict__ Ap = op.A + (mv && !ones ? op.a_row(m) : 0);
    const float* __restrict__ Bp = op.B + op.b_row(rb_r);
    const int64_t kbeg = k0, kend = k1;
    float va[16], vb[kBElems];
    // A[m][k] = Ap[col(k)], B[n][k] = Bp[col(k)]: one add + one load per element
    auto gather = [&](int c, float (&a)[16], float (&b)[kBElems]) {
      const int64_t kb = kbeg + (int64_t)c * kBK;
      int64_t ac[16];
      if constexpr (Op::kKTab == 0) op.a_cols16(kb + ra_kh * 16, ac);  // one decomposition, then a walk
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int64_t k = kb + ra_kh * 16 + e;
        float v = 0.0f;
        if (mv && k < kend) {
          if constexpr (Op::kKTab > 0) v = ones ? 1.0f : Ap[acol[k]];
          else v = ones ? 1.0f : Ap[ac[e]];
        }
        a[e] = v;
      }
      if constexpr (Op::kBDense) {
#pragma unroll
        for (int e = 0; e < kBElems; e += 4) {
          const int64_t k = kb + rb_part * kBElems + e;  // K, split bounds and row starts are multiples of 4
          const float4 v = k < kend ? __ldg(reinterpret_cast<const float4*>(Bp + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
          b[e] = v.x; b[e + 1] = v.y; b[e + 2] = v.z; b[e + 3] = v.w;
        }
      } else if constexpr (!Op::kBImage) {
#pragma unroll
        for (int e = 0; e < kBElems; ++e) {
          const int64_t k = kb + rb_part * kBElems + e;
          float v = 0.0f;
          if (k < kend) {
            if constexpr (Op::kKTab > 0) v = Bp[bcol[k]];
            else v = Bp[op.b_col(k)];
          }
          b[e] = v;
        }
      }
    };
    // prefetch distance 2: chunks c+1 and c+2 are in flight while chunk c is stored
    float na[16], nb[kBElems];
    if (nchunks > 0) gather(0, va, vb);
    if (nchunks > 1) gather(1, na, nb);
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % kStages;
      float n2a[16], n2b[kBElems];
      if (c + 2 < nchunks) gather(c + 2, n2a, n2b);
      if (c >= kStages) mbar_wait(&empty[s], ((c / kStages) - 1) & 1);
      uint8_t* st = base + s * Cfg::kStageBytes;
      uint8_t *ahi = st, *alo = st + Cfg::kABytes, *bhi = st + 2 * Cfg::kABytes, *blo = bhi + Cfg::kBBytes;
      if constexpr (Op::kBImage) {
        if (tid == 0) {  // the pre-split B stage (hi|lo, already swizzled) by one 1-D TMA bulk copy
          mbar_arrive_expect_tx(&full[s], 2 * Cfg::kBBytes);
          tma_load_1d(bhi, reinterpret_cast<const uint8_t*>(op.Bimg) + (size_t)c * 2 * Cfg::kBBytes, 2 * Cfg::kBBytes,
                      &full[s]);
        }
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        float h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_tf32(va[4 * jj + e], h[e], l[e]);
        const uint32_t o = sw128_off(ra_r, ra_kh * 4 + jj);
        *reinterpret_cast<float4*>(ahi + o) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(alo + o) = make_float4(l[0], l[1], l[2], l[3]);
      }
#pragma unroll
      for (int jj = 0; jj < (Op::kBImage ? 0 : kBElems / 4); ++jj) {
        float h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_tf32(vb[4 * jj + e], h[e], l[e]);
        const uint32_t o = sw128_off(rb_r, rb_part * (kBElems / 4) + jj);
        *reinterpret_cast<float4*>(bhi + o) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(blo + o) = make_float4(l[0], l[1], l[2], l[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core reads
      mbar_arrive(&full[s]);
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        va[e] = na[e];
        na[e] = n2a[e];
      }
#pragma unroll
      for (int e = 0; e < kBElems; ++e) {
        vb[e] = nb[e];
        nb[e] = n2b[e];
      }
    }
  } else if (lane == 0) {
    // ---- MMA issuer (warp 8, one lane) ----
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % kStages;
      mbar_wait(&full[s], (c / kStages) & 1);
      tc_fence_after();
      const uint32_t st = smem_u32(base + s * Cfg::kStageBytes);
      const uint32_t ahi = st, alo = st + Cfg::kABytes, bhi = st + 2 * Cfg::kABytes, blo = bhi + Cfg::kBBytes;
#pragma unroll
      for (int kk = 0; kk < kBK / 8; ++kk) {  // K = 8 tf32 = 32 B per MMA inside the 128 B swizzle row
        const uint32_t o = kk * 32;
        mma_tf32(tmem, sw128_desc(ahi + o), sw128_desc(bhi + o), Cfg::kIdesc, (c > 0 || kk > 0) ? 1u : 0u);
        mma_tf32(tmem, sw128_desc(ahi + o), sw128_desc(blo + o), Cfg::kIdesc, 1u);
        mma_tf32(tmem, sw128_desc(alo + o), sw128_desc(bhi + o), Cfg::kIdesc, 1u);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(done_bar);
  }

  // ---- epilogue (warps 0-3: TMEM lanes 32w..32w+31 = tile rows) ----
  if (warp < 4) {
    mbar_wait(done_bar, 0);
    tc_fence_after();
    const int r = warp * 32 + lane;
    const int64_t m = m0 + r;
#pragma unroll 1
    for (int col = 0; col < N; col += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)col, v);
      if (nchunks == 0) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.0f;
      }
      if (m < op.M) {
#pragma unroll
        for (int j = 0; j < 16; ++j) op.store(blockIdx.z, m, col + j, v[j]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kTmemCols));
  }
}

// B stage images for ops whose B (the conv2 weights) is shared by every tile: chunk c, row n, k-in-chunk kk
// -> hi|lo fp32 at the SWIZZLE_128B position the UMMA descriptor expects.  Rebuilt per group (the weights
// change every SGD step); 51,200 elements.
template <class Op>
__global__ void bimg_kernel(Op op, int64_t K) {
  constexpr int N = Op::N;
  using Cfg = TcCfg<N>;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nch = (K + kBK - 1) / kBK;
  if (t >= nch * N * kBK) return;
  const int kk = (int)(t % kBK), n = (int)((t / kBK) % N);
  const int64_t c = t / ((int64_t)kBK * N), k = c * kBK + kk;
  const float v = k < K ? op.B[op.b_row(n) + op.b_col(k)] : 0.0f;
  float hi, lo;
  split_tf32(v, hi, lo);
  uint8_t* img = reinterpret_cast<uint8_t*>(const_cast<float*>(op.Bimg)) + (size_t)c * 2 * Cfg::kBBytes;
  const uint32_t off = sw128_off(n, kk >> 2) + (kk & 3) * 4;
  *reinterpret_cast<float*>(img + off) = hi;
  *reinterpret_cast<float*>(img + Cfg::kBBytes + off) = lo;
}

template <class Op>
cudaError_t launch_tc(const Op& op, int splits, cudaStream_t st) {
  if constexpr (Op::kBImage) {
    int64_t k0 = 0, K = 0;
    // static K: the op's k_range does not depend on the split
    K = Op::kKTab;
    (void)k0;
    const int64_t total = ((K + kBK - 1) / kBK) * Op::N * kBK;
    bimg_kernel<Op><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(op, K);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  constexpr int kSmem = tc_smem_bytes<Op>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const dim3 grid((unsigned)((op.M + kBM - 1) / kBM), 1, (unsigned)splits);
  tc_gemm_kernel<Op><<<grid, kThreadsTC, kSmem, st>>>(op);
  return cudaGetLastError();
}

}  // namespace

cudaError_t tc_gemm(const OpConv2Fwd& op, int splits, cudaStream_t st) { return launch_tc(op, splits, st); }
cudaError_t tc_gemm(const OpGk2& op, int splits, cudaStream_t st) { return launch_tc(op, splits, st); }
cudaError_t tc_gemm(const OpBackin& op, int splits, cudaStream_t st) { return launch_tc(op, splits, st); }

}  // namespace wide
}  // namespace tlb
