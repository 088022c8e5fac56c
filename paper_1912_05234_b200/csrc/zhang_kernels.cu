// zhang_kernels.cu -- sm_100a kernels for the reference's hot path (net::train / forward / backward /
// evaluate, proj/src/network.cpp:81-280) and their host-side launchers.
//
//  * train_kernel<EXACT>  persistent cooperative kernel: runs a whole range of SGD steps (epochs x
//                         groups) in ONE launch.  Per step: each CTA takes a static_chunk of the
//                         group's examples (runtime.cpp:138-145), runs forward+backward per image in
//                         shared memory, writes its gradient rows (EXACT: one row per example, the
//                         reference's parallel_build cell) or one per-CTA partial (fast); grid barrier;
//                         fixed-order reduction + sgd_step over the 3,898 parameters and the fp64
//                         epoch-loss sum (network.cpp:236-248); grid barrier.
//  * train_cluster_kernel the fast persistent kernel for groups that fit one image per CTA: 8-CTA
//                         clusters, DSMEM (st.async + mbarrier) exchange, packed fixed-point
//                         accumulators in L2, parameters resident in shared memory (see below).
//  * cells_kernel<EXACT>  per-example forward(+backward) rows / activations (net::forward/backward).
//  * eval_kernel<EXACT>   forward + argmax + correct count (net::predict / net::evaluate).
//  * sgd_kernel           net::sgd_step on a reduced gradient (also the post-allreduce step of DP).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "tlb_launch.h"
#include "train_common.cuh"
#include "zhang_step.cuh"

namespace tlb {


// Issuer thread: start the job's image TMA into buffer `buf` and an async copy of its label into s.lab[buf]
// -- the label's L2 latency overlaps the previous image's stages instead of preceding the forward pass.
// The issuer completes the copy (cp_async_wait_all) when the job starts, before issuing the next one;
// the forward pass reads s.lab[buf] only after its first CTA barrier (forward_image's `lab`).
__device__ __forceinline__ void issue_job(const Smem& s, const TrainArgs& a, int buf, const Job& j) {
  const int64_t idx = job_index(a, j);  // once: the index math is a serial chain on the issuer lane
  wait_ready_at(a, j.step, idx);
  cp_async4(s.lab + buf, a.labels + idx);
  s.bst[buf] = step_bytes(a, j.step) ? 1 : 0;
  if (s.bst[buf]) {  // byte ingestion: the image's 784 bytes (converted while the previous job runs conv2)
    s.jidx[buf] = idx;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&s.bar[buf], kImg);
    tma_load_1d(s.px + buf * kImg, a.pixels + idx * kImg, kImg, &s.bar[buf]);
  } else {
    // a byte-ingesting launch wrote this fp32 image back with generic stores in its first epoch
    if (a.pixels) asm volatile("fence.proxy.async.global;" ::: "memory");
    issue_image(s, buf, a.images + idx * kImg);
  }
}

// Byte ingestion, the launch's first job of this CTA (no previous job converted it): every thread waits
// for its bytes and converts them.  Later jobs are converted during their predecessor's conv2.
__device__ __forceinline__ void first_bytes(const Smem& s, const TrainArgs& a, bool valid, const Job& j) {
  if (!valid || !step_bytes(a, j.step)) return;
  __syncthreads();  // the issuer's s.jidx[0]
  mbar_wait(&s.bar[0], 0);
  convert_pixels(s.px, s.img, (a.images_wb ? a.images_wb + s.jidx[0] * kImg : nullptr), 1, threadIdx.x, blockDim.x);
  __syncthreads();
}

// sgd_step (network.cpp:171-180) for one parameter, or the shard's gradient sum in DP mode.
// The step's weights are still in shared memory (loaded at the step start), so no L2 read here.
__device__ __forceinline__ void finish_param(const Smem& s, const TrainArgs& a, int j, float acc, int64_t m) {
  if (a.grad_out) {
    a.grad_out[j] = acc;
  } else {
    __stcg(a.params + j, fsub(s.P[j], fmul(a.rate, __fdiv_rn(acc, (float)m))));
  }
}

// Ordered reduction of this CTA's parameter slice over `nrows` gradient rows, then sgd_step.
template <bool EXACT>
__device__ __forceinline__ void reduce_slice(const Smem& s, const TrainArgs& a, int64_t nrows, int64_t m) {
  int64_t j0, j1;
  static_chunk(kNParam, gridDim.x, blockIdx.x, j0, j1);
  constexpr int kLanes = EXACT ? 1 : 8;  // fast: 8 lanes per parameter + fixed shuffle tree
  float* stage = s.c1;                   // c1|s1|c2|s2 are contiguous: >= 5,280 free floats
  const int t = threadIdx.x, per = blockDim.x / kLanes;
  for (int64_t jb = j0; jb < j1; jb += per) {
    const int W = (int)min((int64_t)per, j1 - jb);
    const int R = 5280 / W;
    const int j = t / kLanes, l = t % kLanes;
    float acc = 0.0f;
    for (int64_t r0 = 0; r0 < nrows; r0 += R) {
      const int rr = (int)min((int64_t)R, nrows - r0);
      __syncthreads();
      // thread -> (column c, first row); every load of a thread is in flight before its first
      // shared store, so the L2 round trip is paid once per chunk (no per-element division)
      const int step = blockDim.x / W, c = t % W, rt = t / W;
      if (rt < step) {
        constexpr int kBatch = 8;
        for (int rb = rt; rb < rr; rb += kBatch * step) {
          float v[kBatch];
#pragma unroll
          for (int u = 0; u < kBatch; ++u) {
            const int rw = rb + u * step;
            if (rw < rr) v[u] = __ldcg(a.work + (r0 + rw) * kPStride + jb + c);
          }
#pragma unroll
          for (int u = 0; u < kBatch; ++u) {
            const int rw = rb + u * step;
            if (rw < rr) stage[rw * W + c] = v[u];
          }
        }
      }
      __syncthreads();
      if (r0 == 0) mark(s, 14);
      if (j < W) {
        if constexpr (EXACT) {
#pragma unroll 4
          for (int r = 0; r < rr; ++r) acc = fadd(acc, stage[r * W + j]);
        } else {
          for (int r = l; r < rr; r += kLanes) acc += stage[r * W + j];
        }
      }
    }
    if constexpr (!EXACT) {
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    }
    if (jb == j0) mark(s, 15);
    if (j < W && l == 0) finish_param(s, a, (int)jb + j, acc, m);
  }
}

// fp64 loss sum of the group (network.cpp:239-242).  EXACT: per-example losses in example order;
// fast: per-CTA partial sums in CTA order.  Updates the epoch mean at the group that ends the epoch.
template <bool EXACT>
__device__ __forceinline__ void reduce_loss(const Smem& s, const TrainArgs& a, int64_t m, int64_t nrows, int64_t ks,
                                            int64_t ep) {
  double l = 0.0;
  if (!a.grad_out && ks != 0) l = a.epoch_loss[ep];
  if constexpr (EXACT) {
    float* stage = s.c1;  // activations are dead after the backward pass (s.red is fast-mode only)
    for (int64_t e0 = 0; e0 < m; e0 += 1024) {
      const int n = (int)min((int64_t)1024, m - e0);
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) stage[i] = __ldcg(a.losses + e0 + i);
      __syncthreads();
      if (threadIdx.x == 0)
        for (int i = 0; i < n; ++i) l = __dadd_rn(l, (double)stage[i]);
    }
  } else {
    double* stage = reinterpret_cast<double*>(s.c1);  // fp64 CTA partials, staged in one round trip
    for (int64_t r0 = 0; r0 < nrows; r0 += 512) {
      const int n = (int)min((int64_t)512, nrows - r0);
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) stage[i] = __ldcg(a.loss_part + r0 + i);
      __syncthreads();
      if (threadIdx.x == 0)
        for (int i = 0; i < n; ++i) l = __dadd_rn(l, stage[i]);
    }
  }
  if (threadIdx.x == 0) {
    if (a.grad_out) a.loss_out[0] = l;
    else a.epoch_loss[ep] = (ks == a.steps_per_epoch - 1) ? __ddiv_rn(l, (double)a.n) : l;
  }
}


// ---- in-process multi-GPU (TrainArgs::md_n > 1) -----------------------------------------------------
// Grid barrier over every CTA of every device: arrivals on device 0's counter (system scope: the peers
// reach it over NVLink), bounded by dp_timeout_cycles -- a device that never arrives sets dp_error and the
// host call fails instead of hanging.
__device__ __forceinline__ void md_sync(const TrainArgs& a, unsigned int& target) {
  __syncthreads();
  target += gridDim.x * (unsigned int)a.md_n;
  if (threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(a.md_bar) : "memory");
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a.md_bar) : "memory");
    const long long t0 = clock64();
    while ((int)(v - target) < 0) {
      if (clock64() - t0 > a.dp_timeout_cycles) {
        atomicExch(a.dp_error, 1u);
        break;
      }
      __nanosleep(64);
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a.md_bar) : "memory");
    }
  }
  __syncthreads();
}

// Row r (0 <= r < total) of the step's gradient rows across devices: EXACT = example r of the group (device
// d holds static_chunk(m, md_n, d) of it, local row r - lo_d); fast = the CTA partials of device 0, then of
// device 1, ... (nrows_d = CTAs with examples on device d).  Returns the row's base pointer.
template <bool EXACT>
__device__ __forceinline__ const float* md_row(const TrainArgs& a, int64_t m, int64_t r) {
  int d = 0;
  for (; d < a.md_n - 1; ++d) {
    int64_t lo, hi;
    static_chunk(m, a.md_n, d, lo, hi);
    int64_t cnt = hi - lo;
    if constexpr (!EXACT) {  // CTA partial rows of device d
      const int64_t block = cnt > 0 ? udiv(cnt + gridDim.x - 1, gridDim.x) : 1;
      cnt = cnt > 0 ? udiv(cnt + block - 1, block) : 0;
    }
    if (r < cnt) break;
    r -= cnt;
  }
  return a.md_work[d] + r * kPStride;
}

__device__ __forceinline__ int64_t md_total_rows(const TrainArgs& a, int64_t m, bool exact) {
  if (exact) return m;
  int64_t total = 0;
  for (int d = 0; d < a.md_n; ++d) {
    int64_t lo, hi;
    static_chunk(m, a.md_n, d, lo, hi);
    const int64_t cnt = hi - lo;
    const int64_t block = cnt > 0 ? udiv(cnt + gridDim.x - 1, gridDim.x) : 1;
    total += cnt > 0 ? udiv(cnt + block - 1, block) : 0;
  }
  return total;
}

// Phase 2 across devices: global CTA gb owns parameters static_chunk(3898, md_n * grid, gb); rows are staged
// through shared memory (one L2/NVLink round trip per chunk), then each parameter's sum runs in row order
// (EXACT: a single fp32 chain in example order = the reference's; fast: 8 lanes + a fixed tree) and the
// update goes to every device's parameter copy.
template <bool EXACT>
__device__ __forceinline__ void md_reduce_slice(const Smem& s, const TrainArgs& a, int64_t m) {
  const int Gt = gridDim.x * a.md_n, gb = a.dp_rank * gridDim.x + blockIdx.x;
  int64_t j0, j1;
  static_chunk(kNParam, Gt, gb, j0, j1);
  const int64_t nrows = md_total_rows(a, m, EXACT);
  constexpr int kLanes = EXACT ? 1 : 8;
  float* stage = s.c1;  // c1|s1|c2|s2 are contiguous: >= 5,280 free floats
  const int t = threadIdx.x, per = blockDim.x / kLanes;
  for (int64_t jb = j0; jb < j1; jb += per) {
    const int W = (int)min((int64_t)per, j1 - jb);
    const int R = 5280 / W;
    const int j = t / kLanes, l = t % kLanes;
    float acc = 0.0f;
    for (int64_t r0 = 0; r0 < nrows; r0 += R) {
      const int rr = (int)min((int64_t)R, nrows - r0);
      __syncthreads();
      for (int q = t; q < rr * W; q += blockDim.x) {
        const int rw = q / W, c = q - rw * W;
        stage[rw * W + c] = __ldcg(md_row<EXACT>(a, m, r0 + rw) + jb + c);
      }
      __syncthreads();
      if (j < W) {
        if constexpr (EXACT) {
          for (int r = 0; r < rr; ++r) acc = fadd(acc, stage[r * W + j]);
        } else {
          for (int r = l; r < rr; r += kLanes) acc += stage[r * W + j];
        }
      }
    }
    if constexpr (!EXACT) {
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    }
    if (j < W && l == 0) {
      const int pj = (int)jb + j;
      if (a.grad_out) {
        a.grad_out[pj] = acc;
      } else {
        const float w = fsub(s.P[pj], fmul(a.rate, __fdiv_rn(acc, (float)m)));
        for (int d = 0; d < a.md_n; ++d) __stcg(a.md_params[d] + pj, w);
      }
    }
  }
}

// fp64 loss of the group across devices (global CTA md_n * grid - 1): EXACT per-example losses in example
// order, fast CTA partials in (device, CTA) order; the epoch value goes to every device's epoch_loss.
template <bool EXACT>
__device__ __forceinline__ void md_reduce_loss(const Smem& s, const TrainArgs& a, int64_t m, int64_t ks, int64_t ep) {
  if (threadIdx.x != 0) return;
  double l = ks != 0 ? a.epoch_loss[ep] : 0.0;
  for (int d = 0; d < a.md_n; ++d) {
    int64_t lo, hi;
    static_chunk(m, a.md_n, d, lo, hi);
    const int64_t cnt = hi - lo;
    if constexpr (EXACT) {
      for (int64_t e = 0; e < cnt; ++e) l = __dadd_rn(l, (double)__ldcg(a.md_losses[d] + e));
    } else {
      const int64_t block = cnt > 0 ? udiv(cnt + gridDim.x - 1, gridDim.x) : 1;
      const int64_t rows = cnt > 0 ? udiv(cnt + block - 1, block) : 0;
      for (int64_t r = 0; r < rows; ++r) l = __dadd_rn(l, __ldcg(a.md_loss_part[d] + r));
    }
  }
  const double v = (ks == a.steps_per_epoch - 1) ? __ddiv_rn(l, (double)a.n) : l;
  for (int d = 0; d < a.md_n; ++d) a.md_epoch_loss[d][ep] = v;
}

template <bool EXACT>
__global__ void __launch_bounds__(kThreads, 1) train_kernel(TrainArgs a) {
  Smem s = carve_smem(tlb_smem);
  smem_setup(s);
  unsigned int target = 0;
  const int G = gridDim.x;
  unsigned long long* const trace = blockIdx.x == 0 ? a.trace : nullptr;

  Job pf;
  bool pf_valid = first_job(a, a.step_begin, pf);
  // The prefetch issuer is lane 0 of the last warp: conv1 leaves that warp idle (448 item lanes), so
  // the next job's index math, label copy and TMA issue stay off the first stage's critical path.
  const bool issuer = threadIdx.x == blockDim.x - 32;
  if (issuer && pf_valid) issue_job(s, a, 0, pf);
  first_bytes(s, a, pf_valid, pf);
  uint32_t consumed = 0;

  // group index within the epoch and epoch of step st, advanced incrementally (no per-step division)
  int64_t ks = umod(a.step_begin, a.steps_per_epoch), ep = udiv(a.step_begin, a.steps_per_epoch);
  for (int64_t st = a.step_begin; st < a.step_end; ++st, ks = ks + 1 == a.steps_per_epoch ? (++ep, 0) : ks + 1) {
    int64_t l_lo, l_hi;
    local_range_k(a, ks, l_lo, l_hi);
    const int64_t m = l_hi - l_lo;
    int64_t lo, hi;
    static_chunk(m, G, blockIdx.x, lo, hi);
    s.tr = trace ? trace + (st - a.step_begin) * 16 : nullptr;
    mark(s, 0);

    // ---- phase 1: per-example forward + backward out of shared memory ----
    load_params<EXACT>(s, a.params);
    if constexpr (!EXACT)
      for (int i = threadIdx.x; i < kPStride; i += blockDim.x) s.G[i] = 0.0f;
    __syncthreads();
    mark(s, 1);
    double cta_loss = 0.0;  // fast mode: this CTA's losses, example order, fp64
    for (int64_t e = lo; e < hi; ++e) {
      const int buf = consumed & 1;
      mbar_wait(&s.bar[buf], (consumed >> 1) & 1);
      mark(s, 2);
      if (issuer) {
        cp_async_wait_all();  // this job's label (published by conv1's barrier)
        s.bst[buf ^ 1] = 0;   // (issue_job sets it for a next job that arrives as bytes)
        if (pf_valid) {
          Job nx = pf;
          if (next_job(a, nx)) {
            issue_job(s, a, buf ^ 1, nx);
            pf = nx;
          } else {
            pf_valid = false;
          }
        }
      }
      const NextBytes nb{buf ^ 1, ((consumed + 1) >> 1) & 1, a.images_wb};
      forward_image<EXACT>(s, s.img + buf * kImg, -1, nullptr, true, s.lab + buf, nullptr, 0, 0, nullptr,
                           a.pixels ? &nb : nullptr);
      if (threadIdx.x == 0) {
        const float l = example_loss(s, s.lab[buf], nullptr);
        if constexpr (EXACT) a.losses[e] = l;
        else cta_loss = __dadd_rn(cta_loss, (double)l);
      }
      backward_image<EXACT, !EXACT>(s, s.img + buf * kImg, EXACT ? a.work + e * kPStride : nullptr);
      ++consumed;
    }
    if constexpr (!EXACT) {
      if (lo < hi) {
        float4* dst = reinterpret_cast<float4*>(a.work + (int64_t)blockIdx.x * kPStride);
        const float4* src = reinterpret_cast<const float4*>(s.G);
        for (int i = threadIdx.x; i < kPStride / 4; i += blockDim.x) __stcg(dst + i, src[i]);
        if (threadIdx.x == 0) a.loss_part[blockIdx.x] = cta_loss;
      }
    }
    mark(s, 10);
    if (a.md_n > 1) {  // in-process multi-GPU: the reduction spans every device (see md_reduce_slice)
      const int64_t mg = group_size_k(a, ks);
      md_sync(a, target);
      md_reduce_slice<EXACT>(s, a, mg);
      if (a.dp_rank == a.md_n - 1 && blockIdx.x == G - 1) md_reduce_loss<EXACT>(s, a, mg, ks, ep);
      __syncthreads();
      md_sync(a, target);
      continue;
    }
    grid_sync(a.barrier, target);
    mark(s, 11);

    // ---- phase 2: fixed-order batch reduction + sgd_step (network.cpp:236-244) ----
    // CTA b owns parameters static_chunk(3898, G, b); its rows are staged through shared memory
    // (the activation buffers are free now) so the ordered sums run out of SMEM, not L2.
    int64_t nrows = m;  // EXACT: one row per example (reference order); fast: CTA partials in CTA order
    if constexpr (!EXACT) {
      const int64_t block = udiv(m + G - 1, G);
      nrows = m > 0 ? udiv(m + block - 1, block) : 0;
    }
    reduce_slice<EXACT>(s, a, nrows, m);
    if (blockIdx.x == G - 1) reduce_loss<EXACT>(s, a, m, nrows, ks, ep);
    __syncthreads();
    mark(s, 12);
    grid_sync(a.barrier, target);
    mark(s, 13);
  }
}

// ------------------------------------------------------------------------------------------------
// train_cluster_kernel: the fast-mode persistent train kernel for groups that fit one image per CTA
// (batch <= grid).  CTAs form clusters of 8 (distributed shared memory); per step:
//   1. each CTA runs forward+backward of its image, accumulating the gradient in its shared G;
//   2. CTA q pushes slice r (488 floats) of its G into the receive buffer of owner CTA r (st.async
//      DSMEM stores completing on r's mbarrier); owner r waits for them and sums the 8 slices in rank order;
//   3. owner r adds its cluster partial into ONE global accumulator as 2^-32 fixed point
//      (red.global.add.u64: integer addition is associative, so the sum is the same whatever order
//      the clusters arrive in -- deterministic run to run).  Single GPU: each word also counts its
//      contributions (packed words, kPackBias); fused DP: the owner bumps the slice-r arrival counter;
//   4. owner r of every cluster waits until all clusters have contributed to slice r (no grid-wide
//      barrier: per-word counts, or the 8-way slice counter), reads the slice total and applies
//      sgd_step (network.cpp:171-180) to its copy of slice r;
//   5. owner r pushes its updated slice into every CTA of its cluster (st.async on their mbarriers:
//      slice 0 -- everything conv1 reads -- on its own barrier); a CTA waits for slice 0 before the
//      next conv1 and for the other six foreign slices after it (single GPU; fused DP waits for all).
// The parameters never round-trip through L2 between steps.  Accumulators are triple-buffered by
// step; with counters, buffer (s+1) % 3 is zeroed by cluster 0 during step s before it signals step s
// (every CTA that adds into it in step s+1 has observed that signal); packed words are never zeroed.
// Not the reference's example-order chain: EXACT mode keeps train_kernel<true>.
// ------------------------------------------------------------------------------------------------
#ifndef TLB_POLL_NS
#define TLB_POLL_NS 32  // back-off between the packed-word polls of the single-GPU exchange (ns)
#endif
#ifndef TLB_CLUSTER
#define TLB_CLUSTER 8  // CTAs per cluster (16 = the non-portable cluster size: A/B)
#endif
constexpr int kCluster = TLB_CLUSTER;
#ifndef TLB_PUSH_EARLY
#define TLB_PUSH_EARLY 1  // single GPU: each owner thread pushes its updated parameter as soon as its word completed
#endif
#ifndef TLB_DP_PENDING
#define TLB_DP_PENDING 1
#endif
#ifndef TLB_DP_PUSH_EARLY
#define TLB_DP_PUSH_EARLY 1
#endif
#ifndef TLB_STEP_NOBAR
#define TLB_STEP_NOBAR 1  // with TLB_PUSH_EARLY: no CTA barrier at the step start (G zeroed after the push)
#endif
static_assert(kCluster == 8 || kCluster == 16, "cluster of 8 or 16 CTAs");
constexpr int kSlice = kPStride / kCluster;  // 488 floats per owner CTA
constexpr int kSlice4 = kSlice / 4;
static_assert(kSlice % 4 == 0, "slice must be float4-aligned");
constexpr double kFix = 4294967296.0;  // 2^32 (both schemes: the fused-DP counters and the packed words
                                       // give bitwise the same sums)
// Packed accumulator word (single GPU): each cluster adds llrint(sum * 2^32) + 2^51, so a word that has
// received K contributions since it was last read differs from that read by K * 2^51 + S with
// |S| < 2^50 (|sums| < 2^18): K = (diff + 2^50) >> 51, S = diff - K * 2^51, all modulo 2^64 -- the
// count needs no separate counter and the words never need zeroing.  A word of buffer s % 3 gets its
// next contributions only in step s + 3, after every cluster completed step s + 2, i.e. after every
// reader of step s.  2^-32 resolution: ~1e-10 absolute on gradient sums (fast mode).
#ifndef TLB_PACKED_ACC
#define TLB_PACKED_ACC 1
#endif
constexpr double kPackFix = kFix;
constexpr double kPackUnfix = 1.0 / kPackFix;
constexpr long long kPackBias = 1ll << 51;
constexpr double kUnfix = 1.0 / kFix;
// Cluster-kernel global workspace (in TrainArgs::work): [3][kPStride] u64 gradient accumulators,
// [3] u64 loss accumulators, [kCluster] u32 slice arrival counters (zeroed by the host per launch).
constexpr int64_t kAccWords = 3 * (int64_t)kPStride + 3;

// Fixed-point accumulation: device scope on one GPU, system scope when the accumulator may be a peer
// GPU's memory (fused data parallelism over NVLink).
__device__ __forceinline__ void red_add_u64(unsigned long long* p, long long v, bool sys) {
  if (sys) asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Range guard of one cluster's fixed-point contribution: the packed words decode their contribution count
// only while the step's total stays inside (-2^50, 2^50), so each of the `contributors` words is kept
// below 2^50 / contributors (|gradient sum| < 2^18 / contributors); an out-of-range or non-finite sum is
// clamped -- the count stays exact, so no wait can hang -- and flagged, and the host call fails.
__device__ __forceinline__ double fix_guard(double v, uint32_t contributors, unsigned int* err) {
  const double lim = 1125899906842624.0 / (double)contributors;  // 2^50 / contributors
  if (fabs(v) < lim) return v;
  if (err) atomicExch(err, 1u);
  return v > 0.0 ? lim - 1.0 : -(lim - 1.0);  // NaN -> the negative bound
}

__device__ __forceinline__ unsigned long long ld_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kThreads, 1) train_cluster_kernel(TrainArgs a) {
  static_assert(StageCfg<false>::conv2_back != 3, "the DSMEM receive buffer reuses the backin term buffer");
  static_assert(StageCfg<false>::conv2 == 2 && StageCfg<false>::conv2_back >= 9,
                "the clustered kernel keeps no padded k2 copy (Kp): its stages must read k2 from P");
  Smem s = carve_smem(tlb_smem);
  float* const rx = s.term;   // [8 source ranks][488]: slices pushed to this CTA (it owns slice `rank`)
  __shared__ double loss_rx[kCluster + 1];  // rank 0: the 8 CTAs' fp64 loss sums of the step (pushed);
                                             // [kCluster]: this CTA's DP-timeout flag
  // xbar[0]: the step's gradient slices (and, on rank 0, losses) have landed in rx / loss_rx;
  // xbar[1]: parameter slice 0 (k1, b1: all conv1 reads) has landed in P; xbar[2]: the other foreign
  // slices have.  On one GPU a step waits for xbar[1] only and the next step's conv1 runs while slices
  // 1-7 arrive; it waits for xbar[2] after conv1.  Peers write with st.async
  // (complete_tx on these barriers), so no cluster-wide release/acquire barrier sits in the step.
  __shared__ __align__(8) uint64_t xbar[3];
  smem_setup(s);
  if (threadIdx.x == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    mbar_init(&xbar[2], 1);
    fence_barrier_init();
  }
  cluster_sync_all();  // every CTA of the cluster is running (barriers initialised) before peers store into it
  const uint32_t rank = cluster_rank(), cid = cluster_id(), ncl = cluster_count();
  const int G = gridDim.x;
  // This CTA owns gradient slice `rank`: its accumulator and arrival counter (local, or on the peer
  // GPU rank % dp_world in fused data-parallel mode), and the loss accumulator (rank 0's).
  const bool dp = a.dp_world > 0;
  const int world = dp ? a.dp_world : 1;
  unsigned long long* const acc = a.slice_acc[rank];  // [3][kPStride]
  unsigned long long* const lacc = a.loss_acc;        // [3]
  unsigned int* const cnt = a.slice_cnt[rank];
  const bool owner = !dp || (int)(rank % (uint32_t)world) == a.dp_rank;  // zeroes its slice's next buffer
  unsigned long long* const trace = blockIdx.x == 0 ? a.trace : nullptr;

  Job pf;
  bool pf_valid = first_job(a, a.step_begin, pf);
  // The prefetch issuer is lane 0 of the last warp: conv1 leaves that warp idle (448 item lanes), so
  // the next job's index math, label copy and TMA issue stay off the first stage's critical path.
  const bool issuer = threadIdx.x == blockDim.x - 32;
  if (issuer && pf_valid) issue_job(s, a, 0, pf);
  first_bytes(s, a, pf_valid, pf);
  uint32_t consumed = 0;
  load_params<false>(s, a.params);  // once: afterwards the parameters live in shared memory
  // Barrier-free step start (single GPU, early push): G is zeroed right after each step's gradient push
  // (here for the first step) and rank 0 pushes its own slice 0 to itself as well, so a CTA starts the next
  // conv1 as soon as slice 0 has landed -- its own owner threads still finishing their slices do not hold
  // it back (their own-slice writes are ordered before conv2 by conv1's barrier).
  const bool nobar = TLB_PUSH_EARLY && TLB_STEP_NOBAR && TLB_PACKED_ACC && !dp && a.grad_out == nullptr;
  // fused data parallelism: the same per-thread early push after the slice counter completed
  const bool dp_early = TLB_PUSH_EARLY && TLB_DP_PUSH_EARLY && dp && a.grad_out == nullptr;
  const bool dp_pend = dp_early && TLB_DP_PENDING;  // fused DP: wait for slices 1-7 after conv1 as well
  if (nobar) {
    for (int i = threadIdx.x; i < kPStride; i += blockDim.x) s.G[i] = 0.0f;
    __syncthreads();
  }

  // group index within the epoch and epoch of step st, advanced incrementally (no per-step division)
  int64_t ks = umod(a.step_begin, a.steps_per_epoch), ep = udiv(a.step_begin, a.steps_per_epoch);
  // Single-GPU launches use packed accumulators (count + fixed-point sum in one word, see kPackBias);
  // fused data parallelism keeps the per-slice arrival counters.  packed_prevK: this thread's word of
  // buffer K as last read (the words are never zeroed: each step reads the difference).
  const bool packed = TLB_PACKED_ACC && !dp && a.grad_out == nullptr;
  unsigned long long packed_prev0 = 0ull, packed_prev1 = 0ull, packed_prev2 = 0ull;
  // CTA 0's loss thread: the epoch's running loss sum (a launch may start mid-epoch: resume it)
  double loss_run = (blockIdx.x == 0 && threadIdx.x == kSlice && !a.grad_out && ks != 0) ? a.epoch_loss[ep] : 0.0;
  for (int64_t st = a.step_begin; st < a.step_end; ++st, ks = ks + 1 == a.steps_per_epoch ? (++ep, 0) : ks + 1) {
    const int64_t ls = st - a.step_begin;  // local step
    const uint64_t seq = a.seq_base + (uint64_t)ls;  // steps on these accumulators: buffer seq % 3
    int64_t l_lo, l_hi;
    local_range_k(a, ks, l_lo, l_hi);
    const int64_t m = l_hi - l_lo, m_global = group_size_k(a, ks);
    int64_t lo, hi;
    static_chunk(m, G, blockIdx.x, lo, hi);
    s.tr = trace ? trace + ls * 16 : nullptr;
    mark(s, 0);
    if (!nobar) {
      for (int i = threadIdx.x; i < kPStride; i += blockDim.x) s.G[i] = 0.0f;
      __syncthreads();
    }
    mark(s, 1);
    double cta_loss = 0.0;
    for (int64_t e = lo; e < hi; ++e) {
      const int buf = consumed & 1;
      mbar_wait(&s.bar[buf], (consumed >> 1) & 1);
      mark(s, 2);
      if (issuer) {
        cp_async_wait_all();  // this job's label (published by conv1's barrier)
        s.bst[buf ^ 1] = 0;   // (issue_job sets it for a next job that arrives as bytes)
        if (pf_valid) {
          Job nx = pf;
          if (next_job(a, nx)) {
            issue_job(s, a, buf ^ 1, nx);
            pf = nx;
          } else {
            pf_valid = false;
          }
        }
      }
      // (single GPU: parameter slices 1-7 of the previous step's update land during conv1)
      const bool pending = (!dp || dp_pend) && ls > 0;
      const NextBytes nb{buf ^ 1, ((consumed + 1) >> 1) & 1, a.images_wb};
      forward_image<false>(s, s.img + buf * kImg, -1, nullptr, true, s.lab + buf, pending ? &xbar[2] : nullptr,
                           (uint32_t)((ls - 1) & 1), a.dp_timeout_cycles, a.dp_error, a.pixels ? &nb : nullptr);
      if (threadIdx.x == 0) cta_loss = __dadd_rn(cta_loss, (double)example_loss(s, s.lab[buf], nullptr));
      backward_image<false, true>(s, s.img + buf * kImg, nullptr);
      ++consumed;
    }
    // A CTA without an image this step still completes the previous step's slice 1-7 phase before it
    // re-arms that barrier below (an arrival on an incomplete phase would corrupt its count).
    if ((!dp || dp_pend) && ls > 0 && lo >= hi)
      mbar_wait_cluster_guarded(&xbar[2], (uint32_t)((ls - 1) & 1), a.dp_timeout_cycles, a.dp_error);
    // ---- 2. push slice q of G to its owner q; owner sums the 8 received slices (rank order) ----
    // (nobar: a CTA that trained no image this step passed no barrier since zeroing G: order that first)
    if (nobar && lo >= hi) __syncthreads();
    const uint32_t parity = (uint32_t)(ls & 1);
    if (threadIdx.x == 0) st_async_f64(dsmem_map(&loss_rx[rank], 0), cta_loss, dsmem_map(&xbar[0], 0));
    for (int i = threadIdx.x; i < kCluster * kSlice4; i += blockDim.x) {
      const int q = i / kSlice4, o = 4 * (i - q * kSlice4);
      st_async_v4(dsmem_map(rx + (int)rank * kSlice + o, q), *reinterpret_cast<const float4*>(s.G + q * kSlice + o),
                  dsmem_map(&xbar[0], q));
    }
    // Early push (below): no CTA barrier follows the exchange any more, so order every thread's reads of G
    // here before any thread can reach the next step's zeroing of G (the threads wait for xbar[0] next anyway).
    if (packed && TLB_PUSH_EARLY) __syncthreads();
    if (nobar)  // every read of G (the pushes above) is complete: zero it for the next step's backward
      for (int i = threadIdx.x; i < kPStride; i += blockDim.x) s.G[i] = 0.0f;
    mark(s, 9);
    if (threadIdx.x == 0)
      mbar_arrive_expect_tx(&xbar[0], kCluster * kSlice * sizeof(float) + (rank == 0 ? kCluster * sizeof(double) : 0));
    if (!dp) {
      mbar_wait_cluster_guarded(&xbar[0], parity, a.dp_timeout_cycles, a.dp_error);  // every slice pushed to this owner
    } else if (__syncthreads_or(!mbar_wait_cluster_for(&xbar[0], parity, a.dp_timeout_cycles))) {
      if (threadIdx.x == 0) atomicExch(a.dp_error, 1u);  // a cluster peer gave up (dead peer GPU)
      return;
    }
    mark(s, 10);
    const int b = (int)(seq % 3), bn = (int)((seq + 1) % 3);
    const int j = (int)rank * kSlice + (int)threadIdx.x;  // this thread's parameter (threads < 488)
    if (threadIdx.x < kSlice) {
      float sum = rx[threadIdx.x];
#pragma unroll
      for (int q = 1; q < kCluster; ++q) sum += rx[q * kSlice + threadIdx.x];
      const double fx = fix_guard((double)sum * kFix, ncl * (uint32_t)world, a.fix_err);
      if (packed) {
        red_add_u64(acc + b * kPStride + j, __double2ll_rn(fx) + kPackBias, false);
      } else {
        red_add_u64(acc + b * kPStride + j, __double2ll_rn(fx), dp);
        if (cid == 0 && owner) acc[bn * kPStride + j] = 0ull;  // next step's accumulator
      }
    }
    if (rank == 0 && threadIdx.x == kSlice) {
      double l = 0.0;
      for (int q = 0; q < kCluster; ++q) l = __dadd_rn(l, loss_rx[q]);
      const double fx = fix_guard(l * kFix, ncl * (uint32_t)world, a.fix_err);
      if (packed) {
        red_add_u64(lacc + b, __double2ll_rn(fx) + kPackBias, false);
      } else {
        red_add_u64(lacc + b, __double2ll_rn(fx), dp);
        if (cid == 0 && (!dp || a.dp_rank == 0)) lacc[bn] = 0ull;
      }
    }
    if (packed) {
      // ---- 3/4 (single GPU). Each accumulator word counts its own contributions (see kPackBias): the
      // owner threads wait for their words' ncl-th contribution and read the sum in the same L2 round
      // trip -- no arrival counter, no barrier between the adds and the SGD.  Lane 0 of a warp polls
      // first (its word completes with the others of the burst), then each lane confirms its own.
      mark(s, 14);
      int64_t dsum = 0;
      if (threadIdx.x < kSlice || (blockIdx.x == 0 && threadIdx.x == kSlice)) {
        const unsigned long long* w = threadIdx.x < kSlice ? acc + b * kPStride + j : lacc + b;
        unsigned long long prev = b == 0 ? packed_prev0 : b == 1 ? packed_prev1 : packed_prev2;
        const unsigned long long want = (unsigned long long)ncl;
        auto count_of = [&](unsigned long long v) { return (v - prev + (1ull << 50)) >> 51; };
        unsigned long long v;
        // bounded: a word that never completes (a starved cluster) raises the abort word instead of hanging
        const long long t0 = clock64();
        auto poll = [&]() {
          for (unsigned int n = 0;; ++n) {
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(w) : "memory");
            if (count_of(v) >= want) return;
            if ((n & 63u) == 63u &&
                (*reinterpret_cast<volatile unsigned int*>(a.dp_error) || clock64() - t0 > a.dp_timeout_cycles)) {
              atomicExch(a.dp_error, 1u);
              return;
            }
            if (TLB_POLL_NS > 0) __nanosleep(TLB_POLL_NS);
          }
        };
        if ((threadIdx.x & 31) == 0) poll();
        __syncwarp(__activemask());
        poll();
        dsum = (int64_t)(v - prev - want * (unsigned long long)kPackBias);
        if (b == 0) packed_prev0 = v;
        else if (b == 1) packed_prev1 = v;
        else packed_prev2 = v;
      }
      mark(s, 11);
      float pnew = threadIdx.x < kSlice ? s.P[j] : 0.0f;
      if (threadIdx.x < kSlice && j < kNParam) {
        const float gsum = (float)((double)dsum * kPackUnfix);
        pnew = fsub(pnew, fmul(a.rate, __fdiv_rn(gsum, (float)m_global)));
        if (!(nobar && rank == 0)) s.P[j] = pnew;  // rank 0 under nobar: written by its own push below
        if (cid == 0) __stcg(a.params + j, pnew);
      }
      if (TLB_PUSH_EARLY && threadIdx.x < kSlice) {
        // ---- 5 (early). push this parameter into the 7 peers right away (no CTA barrier between the
        // per-word polls and the push): slice 0 to the peers' xbar[1], slices 1-7 to their xbar[2];
        // under nobar rank 0 also pushes slice 0 into itself (its threads wait for it on xbar[1])
        uint64_t* const pbar = rank == 0 ? &xbar[1] : &xbar[2];
#pragma unroll
        for (int qi = 0; qi < kCluster - 1; ++qi) {
          const int q = qi < (int)rank ? qi : qi + 1;
          st_async_f32(dsmem_map(s.P + j, q), pnew, dsmem_map(pbar, q));
        }
        if (nobar && rank == 0) st_async_f32(dsmem_map(s.P + j, 0), pnew, dsmem_map(pbar, 0));
      }
      if (blockIdx.x == 0 && threadIdx.x == kSlice) {
        const double l = (double)dsum * kPackUnfix;
        loss_run = (ks != 0 ? loss_run : 0.0) + l;
        a.epoch_loss[ep] = (ks == a.steps_per_epoch - 1) ? __ddiv_rn(loss_run, (double)a.n) : loss_run;
      }
    }
    if (!packed) {
      __syncthreads();
      mark(s, 14);
      // ---- 3/4. arrival on slice `rank`, then wait for every cluster's (and every GPU's) contribution ----
      // Thread 0 arrives and polls (per-thread polling floods the counters' L2 lines: +0.6 us).  Release
      // at gpu/sys scope is cumulative over the CTA's adds, which the barrier above orders before it.
      if (threadIdx.x == 0) {
        int t_out = 0;
        if (dp) asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        else asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        const unsigned int want = (unsigned int)((seq + 1) * ncl * (uint64_t)world);
        unsigned int v;
        const long long t0 = clock64();
        for (;;) {
          if (dp) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
          else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
          if ((int)(v - want) >= 0) break;
          if (dp && clock64() - t0 > a.dp_timeout_cycles) {  // a peer never arrived: fail, do not hang
            atomicExch(a.dp_error, 1u);
            t_out = 1;
            break;
          }
          __nanosleep(32);
        }
        loss_rx[kCluster] = t_out;  // (slot past the losses) broadcast through the barrier below
      }
      __syncthreads();
      const int to = (int)loss_rx[kCluster];
      if (to) return;
      mark(s, 11);
      if (threadIdx.x < kSlice) {
        const long long t = (long long)(dp ? ld_sys_u64(acc + b * kPStride + j) : __ldcg(acc + b * kPStride + j));
        if (j < kNParam) {
          const float gsum = (float)((double)t * kUnfix);
          if (a.grad_out) {  // data-parallel shard: the shard's gradient sum goes to the allreduce
            if (cid == 0) a.grad_out[j] = gsum;
          } else {
            s.P[j] = fsub(s.P[j], fmul(a.rate, __fdiv_rn(gsum, (float)m_global)));
            if (cid == 0) __stcg(a.params + j, s.P[j]);
          }
        }
        if (dp_early) {  // fused DP: push the updated parameter into the 7 peers right away (as single-GPU)
          const float v = s.P[j];
          uint64_t* const pb = rank == 0 ? &xbar[1] : &xbar[2];
#pragma unroll
          for (int qi = 0; qi < kCluster - 1; ++qi) {
            const int q = qi < (int)rank ? qi : qi + 1;
            st_async_f32(dsmem_map(s.P + j, q), v, dsmem_map(pb, q));
          }
        }
      }
      if (blockIdx.x == 0 && threadIdx.x == kSlice) {
        const double l = (double)(long long)(dp ? ld_sys_u64(lacc + b) : __ldcg(lacc + b)) * kUnfix;
        if (a.grad_out) {
          a.loss_out[0] = l;
        } else {  // running epoch sum kept in a register: no dependent L2 read on CTA 0's critical path
          loss_run = (ks != 0 ? loss_run : 0.0) + l;
          a.epoch_loss[ep] = (ks == a.steps_per_epoch - 1) ? __ddiv_rn(loss_run, (double)a.n) : loss_run;
        }
      }
    }
    const bool pushed = (packed && TLB_PUSH_EARLY) || dp_early;
    if (!pushed) __syncthreads();
    mark(s, 12);
    // ---- 5. push the updated slice into the other CTAs of the cluster (unless pushed early above) ----
    // slice 0 goes to the peers' xbar[1], slices 1-7 to their xbar[2]
    uint64_t* const pbar = rank == 0 ? &xbar[1] : &xbar[2];
    for (int i = threadIdx.x; !pushed && i < (kCluster - 1) * kSlice4; i += blockDim.x) {
      const int qi = i / kSlice4, q = qi < (int)rank ? qi : qi + 1;
      const int o = (int)rank * kSlice + 4 * (i - qi * kSlice4);
      st_async_v4(dsmem_map(s.P + o, q), *reinterpret_cast<const float4*>(s.P + o), dsmem_map(pbar, q));
    }
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&xbar[1], (rank == 0 && !nobar) ? 0u : (uint32_t)(kSlice * sizeof(float)));
      mbar_arrive_expect_tx(&xbar[2], (uint32_t)((rank == 0 ? kCluster - 1 : kCluster - 2) * kSlice * sizeof(float)));
    }
    if (!dp) {
      mbar_wait_cluster_guarded(&xbar[1], parity, a.dp_timeout_cycles, a.dp_error);  // slice 0 (1-7: after conv1)
    } else if (dp_pend) {  // fused DP: slice 0 now (all threads agree on a timeout), slices 1-7 after conv1
      if (__syncthreads_or(!mbar_wait_cluster_for(&xbar[1], parity, a.dp_timeout_cycles))) {
        if (threadIdx.x == 0) atomicExch(a.dp_error, 1u);
        return;
      }
    } else if (__syncthreads_or(!mbar_wait_cluster_for(&xbar[1], parity, a.dp_timeout_cycles) ||
                                !mbar_wait_cluster_for(&xbar[2], parity, a.dp_timeout_cycles))) {
      if (threadIdx.x == 0) atomicExch(a.dp_error, 1u);
      return;
    }
    mark(s, 15);
    mark(s, 13);
  }
  if (!dp) {
    if (a.step_end > a.step_begin)
      mbar_wait_cluster_guarded(&xbar[2], (uint32_t)((a.step_end - a.step_begin - 1) & 1), a.dp_timeout_cycles, a.dp_error);
    cluster_sync_all();  // no CTA leaves while a peer's DSMEM traffic may still target it
  } else if (dp_pend && a.step_end > a.step_begin) {
    // fused DP: the last step's slices 1-7 have landed before this CTA leaves (bounded: a CTA that gave up
    // on a peer returned earlier, so no unbounded cluster barrier here)
    mbar_wait_cluster_guarded(&xbar[2], (uint32_t)((a.step_end - a.step_begin - 1) & 1), a.dp_timeout_cycles, a.dp_error);
  }
}

// ------------------------------------------------------------------------------------------------
// Per-example forward(+backward) cells: net::forward / net::backward / net::loss for n images.
// ------------------------------------------------------------------------------------------------
template <bool EXACT>
__global__ void __launch_bounds__(kThreads, 1) cells_kernel(CellArgs a) {
  const Smem s = carve_smem(tlb_smem);
  smem_setup(s);
  int64_t lo, hi;
  static_chunk(a.n, gridDim.x, blockIdx.x, lo, hi);
  load_params<EXACT>(s, a.params);
  if (threadIdx.x == 0 && lo < hi) issue_image(s, 0, a.images + lo * kImg);
  __syncthreads();
  uint32_t k = 0;
  for (int64_t e = lo; e < hi; ++e, ++k) {
    const int buf = k & 1;
    mbar_wait(&s.bar[buf], (k >> 1) & 1);
    if (threadIdx.x == 0 && e + 1 < hi) issue_image(s, buf ^ 1, a.images + (e + 1) * kImg);
    const float* y = a.targets ? a.targets + e * 10 : nullptr;
    const int label = a.labels ? __ldg(a.labels + e) : -1;
    const bool has_target = y != nullptr || a.labels != nullptr;
    if (a.acts_in) {
      // net::backward(cache, p, y): activations come from the caller's ActCache (network.cpp:145-169)
      const float* src = a.acts_in + e * kNAct;
      for (int i = threadIdx.x; i < kNAct; i += blockDim.x) {
        const float v = src[i];
        if (i < kS1) s.c1[(i / 576) * kC1Plane + i % 576] = v;
        else if (i < kC2) s.s1[i - kS1] = v;
        else if (i < kS2) s.c2[i - kC2] = v;
        else if (i < kOut) s.s2[i - kS2] = v;
        else s.out[i - kOut] = v;
      }
      if constexpr (EXACT) build_shifted(s, s.img + buf * kImg, threadIdx.x, blockDim.x);
      __syncthreads();
      if (threadIdx.x < 10) {
        const float o = s.out[threadIdx.x];
        s.dz[threadIdx.x] = fmul(fmul(fsub(o, target_of(threadIdx.x, label, y)), o), fsub(1.0f, o));
      }
      __syncthreads();
    } else {
      forward_image<EXACT>(s, s.img + buf * kImg, label, y, a.cells != nullptr);
    }
    if (a.acts) {
      float* dst = a.acts + e * kNAct;
      for (int i = threadIdx.x; i < kNAct; i += blockDim.x) {
        float v;
        if (i < kS1) v = s.c1[(i / 576) * kC1Plane + i % 576];
        else if (i < kC2) v = s.s1[i - kS1];
        else if (i < kS2) v = s.c2[i - kC2];
        else if (i < kOut) v = s.s2[i - kS2];
        else v = s.out[i - kOut];
        dst[i] = v;
      }
    }
    if (threadIdx.x < 10 && a.yhat) a.yhat[e * 10 + threadIdx.x] = s.out[threadIdx.x];
    if (threadIdx.x == 0 && a.losses && has_target) a.losses[e] = example_loss(s, label, y);
    __syncthreads();
    if (a.cells) {
      backward_image<EXACT, false>(s, s.img + buf * kImg, a.cells + e * kPStride);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Forward + predict (+ correct count): net::evaluate (network.cpp:263-280).
// ------------------------------------------------------------------------------------------------
template <bool EXACT>
__global__ void __launch_bounds__(kThreads, 1) eval_kernel(EvalArgs a) {
  const Smem s = carve_smem(tlb_smem);
  smem_setup(s);
  int64_t lo, hi;
  static_chunk(a.n, gridDim.x, blockIdx.x, lo, hi);
  load_params<EXACT>(s, a.params);
  if (threadIdx.x == 0 && lo < hi) issue_image(s, 0, a.images + lo * kImg);
  __syncthreads();
  unsigned long long correct = 0;
  uint32_t k = 0;
  for (int64_t e = lo; e < hi; ++e, ++k) {
    const int buf = k & 1;
    mbar_wait(&s.bar[buf], (k >> 1) & 1);
    if (threadIdx.x == 0 && e + 1 < hi) issue_image(s, buf ^ 1, a.images + (e + 1) * kImg);
    forward_image<EXACT>(s, s.img + buf * kImg, -1, nullptr, false);
    if (threadIdx.x < 10 && a.yhat) a.yhat[e * 10 + threadIdx.x] = s.out[threadIdx.x];
    if (threadIdx.x == 0) {
      int best = 0;  // net::predict (network.cpp:253-261): strict >, lowest index wins ties
#pragma unroll
      for (int i = 1; i < 10; ++i)
        if (s.out[i] > s.out[best]) best = i;
      if (a.pred) a.pred[e] = best;
      if (a.labels) correct += (best == __ldg(a.labels + e));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && a.correct && correct) atomicAdd(a.correct, correct);
}

// net::sgd_step (network.cpp:171-180): w - rate * (g / (float)m), elementwise.
__global__ void sgd_kernel(const float* params, const float* grad, float rate, float m, float* out, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[j] = fsub(params[j], fmul(rate, __fdiv_rn(grad[j], m)));
}

// ------------------------------------------------------------------------------------------------
// Host launchers
// ------------------------------------------------------------------------------------------------
size_t smem_bytes() { return kSmemBytes; }
int threads_per_cta() { return kThreads; }

// Dynamic shared memory actually used by a kernel: the prefix (fast), prefix + EXACT tail, or all.
template <class K>
static cudaError_t prep(K kernel, int* occ, int threads, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kernel, threads, smem);
}

cudaError_t train_occupancy(bool exact, int threads, int* occ) {
  return exact ? prep(train_kernel<true>, occ, threads, kSmemExactBytes)
               : prep(train_kernel<false>, occ, threads, kSmemFastBytes);
}

// 256-thread CTAs (two per SM: the stages loop over their lanes) or 512 (one per SM).
cudaError_t launch_train(bool exact, const TrainArgs& a, int grid, int threads, cudaStream_t st) {
  if (a.md_n > 1) {  // multi-GPU: the devices' kernels meet at md_bar (zeroed by the host beforehand);
    // plain launches, grids sized by the host so every device's CTAs are co-resident (bounded waits)
    if (exact) train_kernel<true><<<grid, threads, kSmemExactBytes, st>>>(a);
    else train_kernel<false><<<grid, threads, kSmemFastBytes, st>>>(a);
    return cudaGetLastError();
  }
  cudaError_t e = cudaMemsetAsync(a.barrier, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return e;
  void* args[] = {const_cast<TrainArgs*>(&a)};
  const void* fn = exact ? (const void*)train_kernel<true> : (const void*)train_kernel<false>;
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads), args, exact ? kSmemExactBytes : kSmemFastBytes,
                                     st);
}

cudaError_t cluster_train_capacity(int* max_clusters) {
  *max_clusters = 0;
  cudaError_t e = cudaFuncSetAttribute(train_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  if (e != cudaSuccess) return e;
  if (kCluster > 8) {
    e = cudaFuncSetAttribute(train_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCluster);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(max_clusters, train_cluster_kernel, &cfg);
}

int cluster_size() { return kCluster; }
size_t cluster_work_bytes() { return kAccWords * sizeof(unsigned long long); }
// Fused-DP symmetric workspace per rank: [3][kPStride] u64 accumulators | [3] u64 loss | pad |
// [kCluster] u32 slice counters | u32 watchdog flag.
// (the watchdog flag sits at dp_workspace_bytes() - 32 = right after the slice counters: parallel.FusedDPStep)
size_t dp_workspace_bytes() { return kAccWords * sizeof(unsigned long long) + 8 + 4 * kCluster + 32; }
size_t dp_counter_offset() { return kAccWords * sizeof(unsigned long long) + 8; }

// Grid = clusters * 8 CTAs, all co-resident (clusters <= cluster_train_capacity): the kernel's grid
// barrier needs co-residency, which the cooperative attribute also asserts where the driver allows it.
cudaError_t launch_train_cluster(const TrainArgs& a, int clusters, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  if (a.dp_world == 0) {  // single GPU: fresh accumulators per launch (fused DP: the caller's seq_base)
    e = cudaMemsetAsync(a.barrier, 0, kCluster * sizeof(unsigned int), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.work, 0, kAccWords * sizeof(unsigned long long), st);
  }
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * kCluster);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  // Default: the cooperative attribute, so the driver asserts that every cluster is co-resident (the
  // kernel's cross-cluster waits need it; a co-tenant holding SMs fails the launch instead of starving a
  // cluster).  TLB_CLUSTER_COOP=0 launches plainly (profilers that cannot replay cooperative launches);
  // a driver that rejects the attribute combination falls back to the plain launch once.  Either way
  // every cross-CTA wait is bounded (mbar_wait_cluster_guarded / the packed-word polls).
  static const bool want_coop = [] {
    const char* e = getenv("TLB_CLUSTER_COOP");
    return !(e && e[0] == '0');
  }();
  static bool coop_ok = true;
  if (want_coop && coop_ok) {
    cfg.numAttrs = 2;
    const cudaError_t le = cudaLaunchKernelEx(&cfg, train_cluster_kernel, a);
    if (le != cudaErrorInvalidValue && le != cudaErrorNotSupported && le != cudaErrorInvalidConfiguration)
      return le;
    (void)cudaGetLastError();
    coop_ok = false;
  }
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, train_cluster_kernel, a);
}

cudaError_t launch_cells(bool exact, const CellArgs& a, int grid, cudaStream_t st) {
  int occ = 0;
  cudaError_t e = exact ? prep(cells_kernel<true>, &occ, kThreads, kSmemExactBytes)
                        : prep(cells_kernel<false>, &occ, kThreads, kSmemFastBytes);
  if (e != cudaSuccess) return e;
  if (exact) cells_kernel<true><<<grid, kThreads, kSmemExactBytes, st>>>(a);
  else cells_kernel<false><<<grid, kThreads, kSmemFastBytes, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_eval(bool exact, const EvalArgs& a, int grid, int threads, cudaStream_t st) {
  int occ = 0;
  cudaError_t e = eval_occupancy(exact, threads, &occ);
  if (e != cudaSuccess) return e;
  if (exact) eval_kernel<true><<<grid, threads, kSmemExactBytes, st>>>(a);
  else eval_kernel<false><<<grid, threads, kSmemFastBytes, st>>>(a);
  return cudaGetLastError();
}

cudaError_t eval_occupancy(bool exact, int threads, int* occ) {
  return exact ? prep(eval_kernel<true>, occ, threads, kSmemExactBytes)
               : prep(eval_kernel<false>, occ, threads, kSmemFastBytes);
}

cudaError_t launch_sgd(const float* params, const float* grad, float rate, int64_t m, float* out, int n,
                       cudaStream_t st) {
  sgd_kernel<<<(n + 255) / 256, 256, 0, st>>>(params, grad, rate, (float)m, out, n);
  return cudaGetLastError();
}

}  // namespace tlb
