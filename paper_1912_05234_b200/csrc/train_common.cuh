// train_common.cuh -- step / group / shard bookkeeping shared by the persistent train kernels
// (zhang_kernels.cu, batch_train.cu): the epoch's SGD groups (mnist::batches, mnist.cpp:169-185), the
// examples of a group this launch owns (whole group, a DP shard, or this rank's static_chunk), the
// per-CTA job iteration of the image prefetch ring, and the overlapped-ingestion ready flags.
#pragma once

#include "tlb_common.cuh"
#include "tlb_launch.h"

namespace tlb {

// ------------------------------------------------------------------------------------------------
// Job iteration over (step, example) pairs owned by one CTA, used for the image prefetch ring.
// ------------------------------------------------------------------------------------------------
struct Job {
  int64_t step, e, hi;
};

// Size of SGD group ks (0 <= ks < steps_per_epoch) of the epoch.
__device__ __forceinline__ int64_t group_size_k(const TrainArgs& a, int64_t ks) {
  const int64_t rem = a.n - ks * a.batch;
  return rem < a.batch ? rem : a.batch;
}
__device__ __forceinline__ int64_t group_size(const TrainArgs& a, int64_t st) {
  return group_size_k(a, umod(st, a.steps_per_epoch));
}

// Examples of group ks handled by this launch: the whole group, the DP shard of it given by the
// caller (grad_out mode), or this rank's static_chunk of it (fused data parallelism).
__device__ __forceinline__ void local_range_k(const TrainArgs& a, int64_t ks, int64_t& lo, int64_t& hi) {
  const int64_t m = group_size_k(a, ks);
  if (a.dp_world > 0) {
    static_chunk(m, a.dp_world, a.dp_rank, lo, hi);
  } else if (a.grad_out) {
    lo = a.shard_lo < m ? a.shard_lo : m;
    hi = a.shard_hi < m ? a.shard_hi : m;
    if (hi < lo) hi = lo;
  } else {
    lo = 0;
    hi = m;
  }
}
__device__ __forceinline__ int64_t local_size(const TrainArgs& a, int64_t st) {
  int64_t lo, hi;
  local_range_k(a, umod(st, a.steps_per_epoch), lo, hi);
  return hi - lo;
}
__device__ __forceinline__ int64_t local_offset(const TrainArgs& a, int64_t st) {
  int64_t lo, hi;
  local_range_k(a, umod(st, a.steps_per_epoch), lo, hi);
  return lo;
}

__device__ __forceinline__ bool first_job(const TrainArgs& a, int64_t from, Job& j) {
  for (int64_t st = from; st < a.step_end; ++st) {
    int64_t lo, hi;
    static_chunk(local_size(a, st), gridDim.x, blockIdx.x, lo, hi);
    if (lo < hi) {
      j = Job{st, lo, hi};
      return true;
    }
  }
  return false;
}

__device__ __forceinline__ bool next_job(const TrainArgs& a, Job& j) {
  if (j.e + 1 < j.hi) {
    ++j.e;
    return true;
  }
  return first_job(a, j.step + 1, j);
}

// Dataset index of the launch-local example e of step st (whole-dataset or shard layout).
__device__ __forceinline__ int64_t example_index(const TrainArgs& a, int64_t st, int64_t e) {
  const int64_t ks = umod(st, a.steps_per_epoch);
  return a.local_stride > 0 ? ks * a.local_stride + e : ks * a.batch + local_offset(a, st) + e;
}

__device__ __forceinline__ int64_t job_index(const TrainArgs& a, const Job& j) { return example_index(a, j.step, j.e); }

__device__ __forceinline__ const float* job_image(const TrainArgs& a, const Job& j) {
  return a.images + job_index(a, j) * kImg;
}

// Overlapped ingestion: wait (thread 0) until the copy stream has landed the chunk holding this job's
// image.  The flag is written by a stream memory operation after the chunk's copy completes.
__device__ __forceinline__ void wait_ready_at(const TrainArgs& a, int64_t step, int64_t index) {
  if (!a.ready || step >= a.ready_step_end) return;
  int64_t k;
  // g = step's group in its epoch: steps < ready_step_end lie within one epoch of step_begin, so no
  // division (the issuer computes this on every job; the divisions had cost ~0.3 us per batch-100 step)
  int64_t g = step - a.step_begin + a.ready_g0;
  if (g >= a.steps_per_epoch) g -= a.steps_per_epoch;
  if (a.chunk > 0) {
    k = udiv(index, a.chunk);
  } else if (a.chunk < 0) {  // ramp (see TrainArgs::chunk): groups 0 | 1 | 2-3 | ... | C/2..C-1, then C each
    const int64_t C = -a.chunk;
    if (g < C) k = g == 0 ? 0 : 64 - __clzll((long long)g);
    else k = a.chunk_shift + 1 + ((g - C) >> a.chunk_shift);
  } else {  // geometric (see TrainArgs::chunk): groups 0, 1, then [2^e, 2^e + 2^(e-1)), [.., 2^(e+1))
    if (g < 2) {
      k = g;
    } else {
      const int e = 63 - __clzll((long long)g);
      k = 2 * e + (int)((g - (1ll << e)) >= (1ll << (e - 1)));
    }
  }
  const unsigned int* f = a.ready + k;
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  const long long t0 = clock64();
  while ((int)(v - a.ready_token) < 0) {
    if (clock64() - t0 > 20000000000LL) {  // ~10 s: record the stuck chunk, fail the call, do not hang
      if (atomicCAS(a.ready_err, 0u, 1u) == 0u) {
        a.ready_err[1] = (unsigned int)k;
        a.ready_err[2] = v;
      }
      break;
    }
    __nanosleep(256);
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");  // the TMA read below follows the flag
}

__device__ __forceinline__ void wait_ready(const TrainArgs& a, const Job& j) { wait_ready_at(a, j.step, job_index(a, j)); }

// Byte ingestion: does step st take its images as pixel bytes (TrainArgs::pixels)?
__device__ __forceinline__ bool step_bytes(const TrainArgs& a, int64_t st) {
  return a.pixels != nullptr && st < a.ready_step_end;
}

// nimg images of pixel bytes in shared memory -> fp32 (pixel / 255.0f, IEEE division: bit-identical to
// mnist::load_images / synth::make_set) into shared `img` and back to global `wb` (the launch's later
// epochs read the fp32 copy).  Threads t of T; the caller publishes with a CTA barrier.
__device__ __forceinline__ void convert_pixels(const uint8_t* px, float* img, float* wb, int nimg, int t, int T) {
  for (int q = t; q < nimg * (kImg / 4); q += T) {
    const uint32_t w = reinterpret_cast<const uint32_t*>(px)[q];
    const float4 v = make_float4(__fdiv_rn((float)(w & 0xffu), 255.0f), __fdiv_rn((float)((w >> 8) & 0xffu), 255.0f),
                                 __fdiv_rn((float)((w >> 16) & 0xffu), 255.0f), __fdiv_rn((float)(w >> 24), 255.0f));
    reinterpret_cast<float4*>(img)[q] = v;
    if (wb) __stcg(reinterpret_cast<float4*>(wb) + q, v);  // nullptr: a one-epoch call, no later reader
  }
}

}  // namespace tlb
