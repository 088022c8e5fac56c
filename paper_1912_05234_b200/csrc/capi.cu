// capi.cu -- implementation of the C ABI declared in include/tloom_b200.h.
//
// Owns the per-context device workspaces and maps the reference API (tloom::nn / tloom::net,
// proj/include/tloom/{nn,network}.hpp) onto the sm_100a kernels.  Argument checks reproduce the
// reference's error conditions and messages (nn.cpp:37-94, network.cpp:209-214, mnist.cpp:169-170).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tlb_capi_internal.h"
#include "tlb_launch.h"
#include "tloom_b200.h"
#include "wide_kernels.cuh"

namespace tlb {

namespace {
thread_local std::string g_last_error;
}

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace tlb

using tlb::fail;

#define TLB_CUDA(expr)                                                                           \
  do {                                                                                           \
    const cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                       \
      return fail(TLB_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                                    #expr);                                                      \
  } while (0)

#define TLB_TRY(expr)           \
  do {                          \
    const int rc_ = (expr);     \
    if (rc_ != TLB_OK) return rc_; \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Per-context result block (device, mirrored in the pinned host block of a host call): the error words,
// the parameters and up to kOutEpochs epoch losses, so tlb_train's results return in ONE D2H copy (four
// small copies had cost 16-20 us per call after the kernel).
constexpr size_t kOutParamOff = 8 * sizeof(unsigned int);
constexpr size_t kOutLossOff = kOutParamOff + TLB_PSTRIDE * sizeof(float);
constexpr int32_t kOutEpochs = 1024;
constexpr size_t kOutBytes = kOutLossOff + kOutEpochs * sizeof(double);
static_assert(kOutLossOff % 8 == 0, "fp64 losses");

struct HostBuf {  // pinned host memory (async H2D/D2H staging of small per-call blocks)
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes, 4096);
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

struct tlb_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  int mode = TLB_MODE_EXACT;
  int grid_override = 0;
  unsigned long long* trace = nullptr;  // device buffer for per-stage clock stamps (profiling)
  // CTAs per SM of the flat train / forward kernels, [mode: 0 fast, 1 exact][CTA size: 0 = 256, 1 = 512]
  int occ_train[2][2] = {{0, 0}, {0, 0}};
  int occ_eval[2][2] = {{0, 0}, {0, 0}};
  // CTA size of the flat kernels: 0 = automatic (256 = two independent CTAs per SM once the work exceeds
  // one item per SM -- their barrier stalls overlap, +26-30% measured; 512 for small launches, where the
  // per-item latency decides), else forced (tlb_ctx_set_threads / TLB_FAST_THREADS).
  int threads_override = 0;
  int max_clusters = 0;    // co-resident 8-CTA clusters of train_cluster_kernel (0 = unavailable)
  bool use_cluster = true;
  int64_t shard_stride = 0;  // DP shard layout of the images/labels passed to the shard / fused-DP entry points
  int batched = -1;  // batched fast train kernel: -1 auto (TLB_BATCHED or the group-size rule), 0 off, 1 on
  bool one_epoch_call = false;  // tlb_train* of a single epoch: byte-ingested images need no fp32 write-back
  DevBuf work, losses, loss_part, barrier;  // persistent-train workspaces
  DevBuf eval_claim;                         // batched inference: round counter
  DevBuf outblk;  // [dev_err 4 | ready_err 4 words | params | epoch losses]: one D2H per host call (kOut*)
  DevBuf stage[8];                 // host-API staging buffers
  // Overlapped ingestion for tlb_train: the dataset is copied chunk by chunk on `copy_stream` while
  // the train kernel runs; a stream memory operation raises ready[k] to the call's token after
  // chunk k lands (the kernel polls it before the image's TMA load).
  cudaStream_t copy_stream = nullptr;
  cudaStream_t copy_stream2 = nullptr;  // second copy stream (TLB_INGEST_STREAMS=2): odd chunks from chunk 3
  cudaEvent_t copy_gate = nullptr;
  DevBuf ready;
  DevBuf ready_err;  // [3] u32 ingestion watchdog words (flag, chunk, observed value)
  // [4] u32 device failure words of the train kernels: [0] a bounded cross-CTA wait gave up (abort word),
  // [1] a fixed-point gradient sum was out of range.  Read and cleared by tlb_train / tlb_synchronize.
  DevBuf dev_err;
  HostBuf pin;       // tlb_train: pinned params / losses / watchdog words
  // Pageable sources (e.g. a C++ MnistSet's std::vector): host worker threads copy each chunk into a
  // pinned bounce slot, the slot's DMA + ready flag follow on the copy stream (see ingest_pageable).
  HostBuf bounce;
  std::vector<cudaEvent_t> bounce_ev;
  unsigned int ready_token = 0;
  DevBuf synth_snaps;  // device synthetic corpus: mt19937_64 state snapshots per segment
  // Widened-network workspaces (capacity `wide_cap` images) and the last group's arguments.
  DevBuf wide[12];
  int64_t wide_cap = 0;
  tlb::wide::StepArgs wide_last{};
  // In-process multi-GPU (tlb_ctx_create_multi): the contexts of devices[1..] (this one is devices[0]);
  // each keeps its shard of the data, its parameter copy and its rows in md_* (see train_multi).
  std::vector<tlb_ctx*> peers;
  DevBuf md_img, md_lab, md_u8, md_p, md_loss, md_work, md_losses, md_lpart, md_bar;
};

namespace {

bool exact(const tlb_ctx* c) { return c->mode == TLB_MODE_EXACT; }

int set_device(tlb_ctx* c) {
  TLB_CUDA(cudaSetDevice(c->device));
  return TLB_OK;
}

std::string shape_str(const int64_t* s, int r) {
  std::string out = "[";
  for (int i = 0; i < r; ++i) {
    if (i) out += ',';
    out += std::to_string(s[i]);
  }
  return out + "]";
}

int check_rank(int r, const char* who) {
  if (r < 0 || r > 8)
    return fail(TLB_ERR_SHAPE, std::string(who) + ": rank " + std::to_string(r) + " exceeds maximum 8");
  return TLB_OK;
}

int64_t count_of(const int64_t* s, int r) {
  int64_t c = 1;
  for (int a = 0; a < r; ++a) c *= s[a];
  return c;
}

// conv_result_shape (nn.cpp:37-49)
int conv_shape(const int64_t* in, int ir, const int64_t* k, int kr, int64_t* out) {
  if (ir != kr)
    return fail(TLB_ERR_SHAPE, "conv: input rank " + std::to_string(ir) + " and kernel rank " +
                                   std::to_string(kr) + " differ");
  for (int a = 0; a < ir; ++a) {
    if (k[a] > in[a])
      return fail(TLB_ERR_SHAPE, "conv: kernel shape " + shape_str(k, kr) + " exceeds input shape " +
                                     shape_str(in, ir) + " on axis " + std::to_string(a));
    out[a] = in[a] - k[a] + 1;
  }
  return TLB_OK;
}

// mconv_result_shape (nn.cpp:51-60)
int mconv_shape(const int64_t* in, int ir, const int64_t* k, int kr, const int64_t* b, int br, int64_t* out,
                int* orank) {
  if (br != 1) return fail(TLB_ERR_SHAPE, "mconv: bias shape " + shape_str(b, br) + " is not rank 1");
  if (kr != ir + 1)
    return fail(TLB_ERR_SHAPE, "mconv: kernel stack rank " + std::to_string(kr) + " must be input rank + 1 = " +
                                   std::to_string(ir + 1));
  if (kr < 1 || k[0] != b[0])
    return fail(TLB_ERR_SHAPE, "mconv: " + std::to_string(kr < 1 ? 0 : k[0]) + " kernels but " +
                                   std::to_string(b[0]) + " biases");
  if (1 + ir > 8) return fail(TLB_ERR_SHAPE, "Shape::concat: combined rank exceeds maximum");
  out[0] = b[0];
  TLB_TRY(conv_shape(in, ir, k + 1, kr - 1, out + 1));
  *orank = ir + 1;
  return TLB_OK;
}

// avgpool_result_shape (nn.cpp:62-77)
int avgpool_shape(const int64_t* s, int r, int64_t* out) {
  if (r < 2) return fail(TLB_ERR_SHAPE, "avgpool: rank " + std::to_string(r) + " input, need rank >= 2");
  for (int a = 0; a < r; ++a) {
    if (a >= r - 2) {
      if (s[a] % 2 != 0)
        return fail(TLB_ERR_SHAPE, "avgpool: axis " + std::to_string(a) + " extent " + std::to_string(s[a]) +
                                       " is not even");
      out[a] = s[a] / 2;
    } else {
      out[a] = s[a];
    }
  }
  return TLB_OK;
}

// backavgpool_result_shape (nn.cpp:79-86)
int backavgpool_shape(const int64_t* s, int r, int64_t* out) {
  if (r < 2)
    return fail(TLB_ERR_SHAPE, "backavgpool: rank " + std::to_string(r) + " input, need rank >= 2");
  for (int a = 0; a < r; ++a) out[a] = a >= r - 2 ? s[a] * 2 : s[a];
  return TLB_OK;
}

// backin_result_shape (nn.cpp:88-94)
int backin_shape(const int64_t* d, int dr, const int64_t* k, int kr, const int64_t* in, int ir, int64_t* out) {
  int64_t expected[8];
  TLB_TRY(conv_shape(in, ir, k, kr, expected));
  bool same = dr == ir;
  for (int a = 0; same && a < dr; ++a) same = d[a] == expected[a];
  if (!same)
    return fail(TLB_ERR_SHAPE, "backin: error shape " + shape_str(d, dr) + " does not match shape(in)" +
                                   " - shape(k) + 1 = " + shape_str(expected, ir));
  for (int a = 0; a < ir; ++a) out[a] = in[a];
  return TLB_OK;
}

// Staging: copy host arrays into a context staging slot.
template <class T>
int stage_in(tlb_ctx* c, int slot, const T* host, size_t count, T** dev) {
  TLB_CUDA(c->stage[slot].ensure(std::max<size_t>(count, 1) * sizeof(T)));
  *dev = static_cast<T*>(c->stage[slot].p);
  if (count) TLB_CUDA(cudaMemcpyAsync(*dev, host, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  return TLB_OK;
}

template <class T>
int stage_out(tlb_ctx* c, int slot, size_t count, T** dev) {
  TLB_CUDA(c->stage[slot].ensure(std::max<size_t>(count, 1) * sizeof(T)));
  *dev = static_cast<T*>(c->stage[slot].p);
  return TLB_OK;
}

template <class T>
int fetch(tlb_ctx* c, T* host, const T* dev, size_t count) {
  if (count) TLB_CUDA(cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  TLB_CUDA(cudaStreamSynchronize(c->stream));
  return TLB_OK;
}

int pick_threads(const tlb_ctx* c, int64_t items) {
  if (c->threads_override) return c->threads_override;
  return items > c->sm_count ? 256 : 512;
}

// Batched fast kernel from this many local examples per group (TLB_BATCHED=0 never, =1 always).
bool use_batched(const tlb_ctx* c, int64_t m_local) {
  static const int mode = [] {
    const char* e = getenv("TLB_BATCHED");
    return e ? atoi(e) : -1;
  }();
  const int want = c->batched >= 0 ? c->batched : mode;
  if (want == 0) return false;
  if (want == 1) return true;
  return m_local >= 4 * (int64_t)c->sm_count;
}

int train_grid(tlb_ctx* c, int64_t m_max, int threads) {
  const int occ = c->occ_train[exact(c) ? 1 : 0][threads == 256 ? 0 : 1];
  const int coop = std::max(1, occ * c->sm_count);
  if (c->grid_override > 0) return std::min(c->grid_override, coop);
  const int64_t want = std::max<int64_t>(c->sm_count, std::min<int64_t>(m_max, coop));
  return (int)std::min<int64_t>(want, coop);
}

int plain_grid(tlb_ctx* c, int64_t n, int threads = 512) {
  const int occ = c->occ_eval[exact(c) ? 1 : 0][threads == 256 ? 0 : 1];
  const int64_t cap = (int64_t)std::max(1, occ) * c->sm_count;
  return (int)std::max<int64_t>(1, std::min<int64_t>(n, cap));
}

// cuStreamWriteValue32 through the runtime's driver entry point (no link-time libcuda dependency).
using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValue32Fn write_value32() {
  static WriteValue32Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<WriteValue32Fn>(p);
  }();
  return fn;
}

// First SGD group of ramp chunk k (TrainArgs::chunk = -C): 0, 1, 2, 4, ..., C, 2C, 3C, ...
int64_t ramp_chunk_start(int64_t k, int64_t C) {
  if (k == 0) return 0;
  int64_t lg = 0;
  while (((int64_t)1 << lg) < C) ++lg;  // C is a power of two
  if (k <= lg) return (int64_t)1 << (k - 1);
  return C * (k - lg);
}

// First SGD group of geometric ingestion chunk k (TrainArgs::chunk == 0; the kernel's wait_ready
// inverts it): 0, 1, 2, 3, 4, 6, 8, 12, 16, 24, ...
int64_t geo_chunk_start(int64_t k) {
  if (k < 2) return k;
  const int64_t e = k / 2;
  return ((int64_t)1 << e) + (k % 2) * ((int64_t)1 << (e - 1));
}

// Upload n images on the copy stream, raising ready[k] to `token` after chunk k lands: chunk > 0 =
// fixed chunks of `chunk` images; chunk == 0 = geometric chunks of SGD groups (groups 0 and 1, then
// the halves of each [2^e, 2^(e+1))), see TrainArgs::chunk.  The copy stream first waits for all earlier work on the
// context stream (buffer reuse).
// Host pixel source of the ingestion: fp32 images (mnist::MnistSet) or the raw bytes they are made from
// (IDX payload / synth::make_digits), converted on the device by pixel / 255.0f (mnist.cpp:57, synth.cpp:158).
struct HostImages {
  const float* f32 = nullptr;
  const uint8_t* u8 = nullptr;
  uint8_t* d_u8 = nullptr;  // device byte staging (u8 source)
};

int ingest_images(tlb_ctx* c, const HostImages& host, float* dev, int64_t n, int64_t chunk, int64_t batch,
                  unsigned int token) {
  TLB_CUDA(cudaStreamWaitEvent(c->copy_stream, c->copy_gate, 0));  // recorded by the caller
  static const bool two = [] {
    const char* e = std::getenv("TLB_INGEST_STREAMS");
    return e && std::atoi(e) == 2;
  }();
  if (two) TLB_CUDA(cudaStreamWaitEvent(c->copy_stream2, c->copy_gate, 0));
  unsigned int* flags = static_cast<unsigned int*>(c->ready.p);
  for (int64_t k = 0, lo = 0; lo < n; ++k) {
    const int64_t hi = chunk > 0 ? lo + chunk
                       : chunk < 0 ? ramp_chunk_start(k + 1, -chunk) * batch : geo_chunk_start(k + 1) * batch;
    const int64_t cnt = std::min(hi, n) - lo;
    // (two streams: the first chunks stay on one stream so the first step's data is not slowed)
    cudaStream_t cs = (two && k >= 3 && (k & 1)) ? c->copy_stream2 : c->copy_stream;
    if (host.u8)  // bytes: the train kernel converts them (TrainArgs::pixels)
      TLB_CUDA(cudaMemcpyAsync(host.d_u8 + lo * 784, host.u8 + lo * 784, (size_t)cnt * 784, cudaMemcpyHostToDevice, cs));
    else
      TLB_CUDA(cudaMemcpyAsync(dev + lo * 784, host.f32 + lo * 784, (size_t)cnt * 784 * sizeof(float),
                               cudaMemcpyHostToDevice, cs));
    const CUresult r = write_value32()(reinterpret_cast<CUstream>(cs),
                                       reinterpret_cast<CUdeviceptr>(flags + k), token, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(TLB_ERR_CUDA, "cuStreamWriteValue32 failed: " + std::to_string((int)r));
    lo += cnt;
  }
  return TLB_OK;
}

// Pageable source (the memory a C++ caller's MnistSet lives in): the driver would stage a pageable
// cudaMemcpyAsync synchronously through its own bounce buffers, one chunk at a time, ahead of the
// kernel.  Instead W host threads copy the chunks into pinned bounce slots (worker w takes chunks
// k = w, w + W, ... into its own ring of kBounceRing slots) and each slot's DMA + ready flag follow on
// the copy stream, so the host copies, the DMA and the running train kernel overlap.  A slot is reused
// once its previous DMA completed (event).  Called after the kernel launch, like the pinned path.
constexpr int kBounceRing = 2;
struct PageablePlan {
  std::vector<int64_t> lo_of;  // chunk k covers images [lo_of[k], lo_of[k + 1])
  size_t elem = 0, slot = 0;
  int workers = 1;
};
// The chunk plan (the same ramp the kernel's ready flags follow), the slot size and the worker count;
// allocates the bounce slots and their events.  Runs BEFORE the kernel launch: growing pinned memory
// (cudaFreeHost) synchronises the device, which would deadlock against a kernel waiting for the chunks.
int plan_pageable(tlb_ctx* c, bool u8, int64_t n, int64_t chunk, int64_t batch, PageablePlan* pl) {
  pl->elem = u8 ? 784 : 784 * sizeof(float);
  pl->lo_of.clear();
  for (int64_t k = 0, lo = 0; lo < n; ++k) {
    pl->lo_of.push_back(lo);
    const int64_t hi = chunk > 0 ? lo + chunk
                       : chunk < 0 ? ramp_chunk_start(k + 1, -chunk) * batch : geo_chunk_start(k + 1) * batch;
    lo = std::min(hi, n);
  }
  pl->lo_of.push_back(n);
  const int64_t nk = (int64_t)pl->lo_of.size() - 1;
  size_t slot = 0;
  for (int64_t k = 0; k < nk; ++k) slot = std::max(slot, (size_t)(pl->lo_of[k + 1] - pl->lo_of[k]) * pl->elem);
  pl->slot = (slot + 4095) / 4096 * 4096;
  // host copy threads: 4 measured best on the GPU VMs (1: 4.6, 2: 5.7, 4: 6.0, 8: 4.4 M img/s through
  // tloom::net::train at batch 100; profiles/r2/cpp_e2e_threads_r2i.txt); TLB_INGEST_THREADS overrides
  static const int env_w = [] {
    const char* e = std::getenv("TLB_INGEST_THREADS");
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  pl->workers = (int)std::max<int64_t>(1, std::min<int64_t>(nk, env_w ? env_w : std::min(4, std::max(1, hw / 2))));
  TLB_CUDA(c->bounce.ensure((size_t)pl->workers * kBounceRing * pl->slot));
  while (c->bounce_ev.size() < (size_t)pl->workers * kBounceRing) {
    cudaEvent_t ev;
    TLB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    c->bounce_ev.push_back(ev);
  }
  return TLB_OK;
}

int ingest_pageable(tlb_ctx* c, const HostImages& host, float* dev, const PageablePlan& pl, unsigned int token) {
  TLB_CUDA(cudaStreamWaitEvent(c->copy_stream, c->copy_gate, 0));  // recorded by the caller
  const std::vector<int64_t>& lo_of = pl.lo_of;
  const int64_t nk = (int64_t)lo_of.size() - 1;
  const size_t elem = pl.elem, slot = pl.slot;
  const int W = pl.workers;
  unsigned int* flags = static_cast<unsigned int*>(c->ready.p);
  uint8_t* const base = static_cast<uint8_t*>(c->bounce.p);
  const uint8_t* const src = host.u8 ? host.u8 : reinterpret_cast<const uint8_t*>(host.f32);
  uint8_t* const dst = host.u8 ? host.d_u8 : reinterpret_cast<uint8_t*>(dev);
  std::vector<int> status(W, TLB_OK);
  std::vector<std::string> why(W);
  auto worker = [&](int w) {
    cudaSetDevice(c->device);
    for (int64_t k = w, j = 0; k < nk; k += W, ++j) {
      const int s = w * kBounceRing + (int)(j % kBounceRing);
      uint8_t* b = base + (size_t)s * slot;
      cudaError_t e = j >= kBounceRing ? cudaEventSynchronize(c->bounce_ev[s]) : cudaSuccess;
      const size_t off = (size_t)lo_of[k] * elem, bytes = (size_t)(lo_of[k + 1] - lo_of[k]) * elem;
      if (e == cudaSuccess) {
        std::memcpy(b, src + off, bytes);
        e = cudaMemcpyAsync(dst + off, b, bytes, cudaMemcpyHostToDevice, c->copy_stream);
      }
      if (e == cudaSuccess) e = cudaEventRecord(c->bounce_ev[s], c->copy_stream);
      if (e != cudaSuccess) {
        status[w] = TLB_ERR_CUDA;
        why[w] = std::string("pageable ingestion: ") + cudaGetErrorString(e);
        return;  // the kernel's ready-flag watchdog fails the call
      }
      const CUresult r = write_value32()(reinterpret_cast<CUstream>(c->copy_stream),
                                         reinterpret_cast<CUdeviceptr>(flags + k), token, CU_STREAM_WRITE_VALUE_DEFAULT);
      if (r != CUDA_SUCCESS) {
        status[w] = TLB_ERR_CUDA;
        why[w] = "cuStreamWriteValue32 failed: " + std::to_string((int)r);
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < W; ++w) pool.emplace_back(worker, w);
  worker(0);
  for (auto& t : pool) t.join();
  for (int w = 0; w < W; ++w)
    if (status[w] != TLB_OK) return fail(status[w], why[w]);
  return TLB_OK;
}

// Number of ingestion chunks for n images (see ingest_images).
int64_t ingest_chunks(int64_t n, int64_t chunk, int64_t batch) {
  if (chunk > 0) return (n + chunk - 1) / chunk;
  const int64_t groups = (n + batch - 1) / batch;
  int64_t k = 0;
  while ((chunk < 0 ? ramp_chunk_start(k + 1, -chunk) : geo_chunk_start(k + 1)) < groups) ++k;
  return k + 1;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

constexpr double kWaitLimitSeconds = 2.0;  // bound of the single-GPU cross-CTA waits

// Device failure words (tlb_ctx::dev_err) -> status; clears them.  `words` = the host copy.
int device_status(tlb_ctx* c, const unsigned int* words) {
  if (!words[0] && !words[1]) return TLB_OK;
  cudaMemsetAsync(c->dev_err.p, 0, 4 * sizeof(unsigned int), c->stream);
  cudaStreamSynchronize(c->stream);
  if (words[1])
    return fail(TLB_ERR_VALUE, "train (fast mode): a gradient sum left the fixed-point range of the clustered "
                               "exchange (|sum| >= 2^18 / clusters; unnormalised inputs or a diverging run) -- the "
                               "result is invalid; use exact mode or normalised data");
  return fail(TLB_ERR_CUDA, "train: a cross-CTA wait of the clustered kernel timed out (" +
                                std::to_string(kWaitLimitSeconds) + " s: SMs held by another process?)");
}

struct DpArgs {
  int world, rank;
  void* const* peer_ws;  // world pointers: every rank's symmetric workspace (tlb_dp_workspace_bytes)
  uint64_t seq_base;
  long long timeout_cycles;
};

int check_train_args(int64_t n, int32_t epochs, float rate, int64_t batch) {
  // network.cpp:211-214 then mnist::batches (mnist.cpp:170)
  if (n == 0) return fail(TLB_ERR_ERROR, "train: empty dataset");
  if (epochs < 0) return fail(TLB_ERR_ERROR, "train: negative epoch count");
  if (!(rate > 0.0f)) return fail(TLB_ERR_ERROR, "train: rate must be > 0");
  if (batch < 1) return fail(TLB_ERR_ERROR, "batches: size must be >= 1, got " + std::to_string(batch));
  if (n < 0) return fail(TLB_ERR_ARG, "train: negative dataset size");
  return TLB_OK;
}

// Enqueue epochs [epoch_begin, epoch_begin + epochs) on device buffers.
int enqueue_train(tlb_ctx* c, const float* d_images, const int32_t* d_labels, int64_t n, float* d_params,
                  float rate, int32_t epoch_begin, int32_t epochs, int64_t batch, double* d_epoch_loss,
                  int64_t shard_lo = 0, int64_t shard_hi = 0, int64_t group = -1, float* grad_out = nullptr,
                  double* loss_out = nullptr, const unsigned int* ready = nullptr, unsigned int token = 0,
                  int64_t chunk = 1, const DpArgs* dp = nullptr, const uint8_t* pixels = nullptr) {
  const int64_t spe = (n + batch - 1) / batch;
  const int64_t m_max = std::min<int64_t>(batch, n);
  const int64_t m_local = grad_out ? std::max<int64_t>(0, std::min(shard_hi, m_max) - shard_lo) : m_max;
  // Clustered fast kernel: one example per CTA per step, every CTA co-resident.
  const int csz = tlb::cluster_size();
  int clusters = (int)((std::max<int64_t>(m_local, 1) + csz - 1) / csz);
  if (dp) {  // every rank launches the same grid: size it for the largest static_chunk
    const int64_t block = (m_max + dp->world - 1) / dp->world;
    clusters = (int)((std::max<int64_t>(block, 1) + csz - 1) / csz);
  }
  const bool clustered = !exact(c) && c->use_cluster && c->grid_override == 0 && c->max_clusters > 0 &&
                         clusters <= c->max_clusters;
  // Large groups (configs[3]): the batched fast kernel (NI images per CTA round, batch_train.cu).
  const bool batched = !exact(c) && !clustered && !dp && c->grid_override == 0 && use_batched(c, m_local);
  const int threads = pick_threads(c, m_local);
  const int grid = clustered ? clusters * csz
                   : batched ? tlb::batch_train_grid(c->sm_count, std::max<int64_t>(m_local, 1))
                             : train_grid(c, std::max<int64_t>(m_local, 1), threads);
  if (grid <= 0) return fail(TLB_ERR_CUDA, "train: batched kernel configuration failed");
  const int64_t rows = exact(c) ? std::max<int64_t>(m_local, 1) : grid;
  TLB_CUDA(c->work.ensure(clustered ? tlb::cluster_work_bytes()
                                     : (size_t)rows * TLB_PSTRIDE * sizeof(float) +
                                           (batched ? tlb::kBatchWorkExtraBytes : 0)));
  TLB_CUDA(c->losses.ensure((size_t)std::max<int64_t>(m_local, 1) * sizeof(float)));
  TLB_CUDA(c->barrier.ensure(tlb::cluster_size() * sizeof(unsigned int)));
  TLB_CUDA(c->loss_part.ensure((size_t)(clustered ? 2 * clusters : grid) * sizeof(double)));
  tlb::TrainArgs a{};
  a.images = d_images;
  a.labels = d_labels;
  a.n = n;
  a.batch = batch;
  a.rate = rate;
  a.steps_per_epoch = spe;
  if (group >= 0) {
    a.step_begin = group;
    a.step_end = group + 1;
  } else {
    a.step_begin = (int64_t)epoch_begin * spe;
    a.step_end = (int64_t)(epoch_begin + epochs) * spe;
  }
  a.params = d_params;
  a.work = static_cast<float*>(c->work.p);
  a.losses = static_cast<float*>(c->losses.p);
  a.loss_part = static_cast<double*>(c->loss_part.p);
  a.epoch_loss = d_epoch_loss;
  a.barrier = static_cast<unsigned int*>(c->barrier.p);
  a.shard_lo = shard_lo;
  a.shard_hi = shard_hi;
  a.grad_out = grad_out;
  a.loss_out = loss_out;
  a.trace = c->trace;
  a.ready = ready;
  a.ready_err = static_cast<unsigned int*>(c->ready_err.p);
  a.ready_token = token;
  a.chunk = chunk;
  a.ready_step_end = a.step_begin + spe;  // only the call's first epoch can outrun the copies
  a.ready_g0 = a.step_begin % spe;        // the ramp's chunk of a group without divisions on the device
  a.chunk_shift = 0;
  if (chunk < 0)
    while ((int64_t)1 << (a.chunk_shift + 1) <= -chunk) ++a.chunk_shift;
  a.dp_error = static_cast<unsigned int*>(c->dev_err.p);        // single GPU: abort word of the bounded waits
  a.fix_err = static_cast<unsigned int*>(c->dev_err.p) + 1;
  a.dp_timeout_cycles = (long long)(kWaitLimitSeconds * 2.0e9);  // ~2 GHz SM clock
  a.local_stride = (dp || grad_out) ? c->shard_stride : 0;
  a.pixels = ready ? pixels : nullptr;  // bytes only while the ingestion flags are live (the first epoch)
  a.images_wb = c->one_epoch_call ? nullptr : const_cast<float*>(d_images);
  if (clustered) {
    if (dp) {  // fused data parallelism: slice s lives on rank s % world (peer memory)
      a.dp_world = dp->world;
      a.dp_rank = dp->rank;
      for (int sl = 0; sl < tlb::cluster_size(); ++sl) {
        char* base = static_cast<char*>(dp->peer_ws[sl % dp->world]);
        a.slice_acc[sl] = reinterpret_cast<unsigned long long*>(base);
        a.slice_cnt[sl] = reinterpret_cast<unsigned int*>(base + tlb::dp_counter_offset()) + sl;
      }
      a.loss_acc = reinterpret_cast<unsigned long long*>(static_cast<char*>(dp->peer_ws[0]) + 3 * TLB_PSTRIDE * 8);
      a.seq_base = dp->seq_base;
      a.dp_error = reinterpret_cast<unsigned int*>(static_cast<char*>(dp->peer_ws[dp->rank]) +
                                                   tlb::dp_counter_offset()) + tlb::cluster_size();
      a.dp_timeout_cycles = dp->timeout_cycles;
    } else {
      for (int sl = 0; sl < tlb::cluster_size(); ++sl) {
        a.slice_acc[sl] = static_cast<unsigned long long*>(c->work.p);
        a.slice_cnt[sl] = static_cast<unsigned int*>(c->barrier.p) + sl;
      }
      a.loss_acc = static_cast<unsigned long long*>(c->work.p) + 3 * TLB_PSTRIDE;
    }
  } else if (dp) {
    return fail(TLB_ERR_ARG, "fused data parallelism needs fast mode and groups of <= 8 x co-resident clusters "
                             "per rank");
  }
  if (a.step_end <= a.step_begin) return TLB_OK;
  if (clustered) TLB_CUDA(tlb::launch_train_cluster(a, clusters, c->stream));
  else if (batched) TLB_CUDA(tlb::launch_train_batch(a, c->sm_count, std::max<int64_t>(m_local, 1), c->stream));
  else TLB_CUDA(tlb::launch_train(exact(c), a, grid, threads, c->stream));
  return TLB_OK;
}

}  // namespace

extern "C" {

const char* tlb_last_error(void) { return tlb::g_last_error.c_str(); }

const char* tlb_version(void) { return "tloom-b200 0.1 (sm_100a)"; }

int tlb_ctx_create(int device, tlb_ctx** out) {
  if (!out) return fail(TLB_ERR_ARG, "tlb_ctx_create: null output");
  *out = nullptr;
  int count = 0;
  TLB_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count)
    return fail(TLB_ERR_ARG, "tlb_ctx_create: device " + std::to_string(device) + " out of range (" +
                                 std::to_string(count) + " devices)");
  TLB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  TLB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(TLB_ERR_CUDA, std::string("tlb_ctx_create: device is ") + prop.name + " (sm_" +
                                  std::to_string(prop.major) + std::to_string(prop.minor) +
                                  "); this build targets sm_100a (B200)");
  tlb_ctx* c = new tlb_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  cudaError_t e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
  if (const char* t = getenv("TLB_FAST_THREADS")) c->threads_override = atoi(t) == 256 ? 256 : atoi(t) == 512 ? 512 : 0;
  for (int x = 0; x < 2; ++x)
    for (int t = 0; t < 2; ++t) {
      if (e == cudaSuccess) e = tlb::train_occupancy(x == 1, t ? 512 : 256, &c->occ_train[x][t]);
      if (e == cudaSuccess) e = tlb::eval_occupancy(x == 1, t ? 512 : 256, &c->occ_eval[x][t]);
    }
  if (e != cudaSuccess) {
    delete c;
    return fail(TLB_ERR_CUDA, std::string("tlb_ctx_create: ") + cudaGetErrorString(e));
  }
  if (e == cudaSuccess && tlb::cluster_train_capacity(&c->max_clusters) != cudaSuccess) {
    (void)cudaGetLastError();  // no cluster launch on this device: the flat kernel is used
    c->max_clusters = 0;
  }
  if (e == cudaSuccess) e = c->outblk.ensure(kOutBytes);
  if (e == cudaSuccess) e = cudaMemset(c->outblk.p, 0, kOutBytes);
  if (e == cudaSuccess) {  // views into outblk (never freed on their own)
    c->dev_err.p = c->outblk.p;
    c->ready_err.p = static_cast<char*>(c->outblk.p) + 4 * sizeof(unsigned int);
    c->dev_err.cap = c->ready_err.cap = 4 * sizeof(unsigned int);
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy_stream2, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->copy_gate, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete c;
    return fail(TLB_ERR_CUDA, std::string("tlb_ctx_create: ") + cudaGetErrorString(e));
  }
  c->stream = c->own_stream;
  *out = c;
  return TLB_OK;
}

int tlb_ctx_destroy(tlb_ctx* c) {
  if (!c) return TLB_OK;
  for (tlb_ctx* p : c->peers) tlb_ctx_destroy(p);
  c->peers.clear();
  cudaSetDevice(c->device);
  for (DevBuf* b : {&c->md_img, &c->md_lab, &c->md_u8, &c->md_p, &c->md_loss, &c->md_work, &c->md_losses, &c->md_lpart,
                    &c->md_bar})
    b->release();
  cudaStreamSynchronize(c->stream);
  c->work.release();
  c->losses.release();
  c->loss_part.release();
  c->barrier.release();
  c->eval_claim.release();
  for (auto& s : c->stage) s.release();
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  if (c->copy_stream2) cudaStreamSynchronize(c->copy_stream2);
  c->ready.release();
  c->ready_err.p = c->dev_err.p = nullptr;  // views into outblk
  c->ready_err.cap = c->dev_err.cap = 0;
  c->outblk.release();
  c->pin.release();
  c->bounce.release();
  for (cudaEvent_t ev : c->bounce_ev) cudaEventDestroy(ev);
  for (auto& w : c->wide) w.release();
  c->synth_snaps.release();
  if (c->copy_gate) cudaEventDestroy(c->copy_gate);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->copy_stream2) cudaStreamDestroy(c->copy_stream2);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
  return TLB_OK;
}

int tlb_ctx_set_stream(tlb_ctx* c, void* stream) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  c->stream = static_cast<cudaStream_t>(stream);  // NULL = the legacy default stream, as in CUDA
  return TLB_OK;
}

int tlb_ctx_set_mode(tlb_ctx* c, int mode) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  if (mode != TLB_MODE_EXACT && mode != TLB_MODE_FAST)
    return fail(TLB_ERR_ARG, "tlb_ctx_set_mode: unknown mode " + std::to_string(mode));
  c->mode = mode;
  for (tlb_ctx* p : c->peers) p->mode = mode;
  return TLB_OK;
}

int tlb_ctx_create_multi(const int* devices, int n_devices, tlb_ctx** out) {
  if (!out || !devices) return fail(TLB_ERR_ARG, "tlb_ctx_create_multi: null argument");
  *out = nullptr;
  if (n_devices < 1 || n_devices > 8) return fail(TLB_ERR_ARG, "tlb_ctx_create_multi: 1..8 devices");
  tlb_ctx* c = nullptr;
  TLB_TRY(tlb_ctx_create(devices[0], &c));
  for (int i = 1; i < n_devices; ++i) {
    tlb_ctx* p = nullptr;
    const int rc = tlb_ctx_create(devices[i], &p);
    if (rc != TLB_OK) {
      tlb_ctx_destroy(c);
      return rc;
    }
    c->peers.push_back(p);
  }
  // peer access between distinct devices (the reduction reads every device's rows, writes every copy)
  for (int i = 0; i < n_devices; ++i)
    for (int j = 0; j < n_devices; ++j) {
      if (devices[i] == devices[j]) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, devices[i], devices[j]);
      if (!ok) {
        tlb_ctx_destroy(c);
        return fail(TLB_ERR_CUDA, "tlb_ctx_create_multi: device " + std::to_string(devices[i]) +
                                      " cannot access device " + std::to_string(devices[j]) + " (no P2P)");
      }
      cudaSetDevice(devices[i]);
      const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        tlb_ctx_destroy(c);
        return fail(TLB_ERR_CUDA, std::string("tlb_ctx_create_multi: ") + cudaGetErrorString(e));
      }
      (void)cudaGetLastError();
    }
  cudaSetDevice(devices[0]);
  *out = c;
  return TLB_OK;
}

int tlb_ctx_device_count(const tlb_ctx* c, int* n) {
  if (!c || !n) return fail(TLB_ERR_ARG, "null argument");
  *n = 1 + (int)c->peers.size();
  return TLB_OK;
}

int tlb_ctx_get_mode(const tlb_ctx* c, int* mode) {
  if (!c || !mode) return fail(TLB_ERR_ARG, "null argument");
  *mode = c->mode;
  return TLB_OK;
}

int tlb_ctx_set_grid(tlb_ctx* c, int ctas) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  c->grid_override = std::max(0, ctas);
  return TLB_OK;
}

int tlb_ctx_set_threads(tlb_ctx* c, int threads) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  if (threads != 0 && threads != 256 && threads != 512)
    return fail(TLB_ERR_ARG, "tlb_ctx_set_threads: 0 (automatic), 256 or 512");
  c->threads_override = threads;
  return TLB_OK;
}

int tlb_ctx_set_shard_layout(tlb_ctx* c, int64_t local_stride) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  if (local_stride < 0) return fail(TLB_ERR_ARG, "tlb_ctx_set_shard_layout: negative stride");
  c->shard_stride = local_stride;
  return TLB_OK;
}

int tlb_ctx_set_batched(tlb_ctx* c, int mode) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  if (mode < -1 || mode > 1) return fail(TLB_ERR_ARG, "tlb_ctx_set_batched: -1 (automatic), 0 or 1");
  c->batched = mode;
  return TLB_OK;
}

int tlb_ctx_set_cluster(tlb_ctx* c, int enable) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  c->use_cluster = enable != 0;
  return TLB_OK;
}

int tlb_ctx_set_trace(tlb_ctx* c, void* d_trace) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  c->trace = static_cast<unsigned long long*>(d_trace);
  return TLB_OK;
}

int tlb_ctx_info(const tlb_ctx* c, int* sm, int* occ_train, int* occ_eval, int64_t* smem) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  const int x = c->mode == TLB_MODE_EXACT ? 1 : 0;
  if (sm) *sm = c->sm_count;
  if (occ_train) *occ_train = c->occ_train[x][1];
  if (occ_eval) *occ_eval = c->occ_eval[x][1];
  if (smem) *smem = (int64_t)tlb::smem_bytes();
  return TLB_OK;
}

int tlb_synchronize(tlb_ctx* c) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  TLB_CUDA(cudaSetDevice(c->device));
  TLB_CUDA(cudaStreamSynchronize(c->stream));
  unsigned int words[4] = {0, 0, 0, 0};  // failures of earlier device-API train launches
  TLB_CUDA(cudaMemcpy(words, c->dev_err.p, sizeof(words), cudaMemcpyDeviceToHost));
  return device_status(c, words);
}

// ---- network, host buffers ------------------------------------------------------------------
// TLB_HOST_TRACE=1: per-call host timeline of tlb_train on stderr (developer diagnostics of the e2e path).
struct HostTrace {
  bool on;
  std::chrono::steady_clock::time_point t0;
  std::string log;
  cudaEvent_t ev[4] = {};  // device-side: before the kernel, after it, after the D2H, (spare)
  int nev = 0;
  HostTrace() : on(std::getenv("TLB_HOST_TRACE") != nullptr), t0(std::chrono::steady_clock::now()) {}
  void mark(const char* what) {
    if (!on) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    log += std::string(" ") + what + "=" + std::to_string((int)us);
  }
  void event(cudaStream_t st) {  // device timeline stamp on the stream (trace mode only)
    if (!on || nev >= 4) return;
    cudaEventCreate(&ev[nev]);
    cudaEventRecord(ev[nev++], st);
  }
  ~HostTrace() {
    if (!on) return;
    for (int i = 1; i < nev; ++i) {
      float ms = 0.0f;
      cudaEventSynchronize(ev[i]);
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      log += " dev" + std::to_string(i) + "=" + std::to_string((int)(ms * 1000.0f));
    }
    for (int i = 0; i < nev; ++i) cudaEventDestroy(ev[i]);
    fprintf(stderr, "tlb_train host us:%s\n", log.c_str());
  }
};

// In-process multi-GPU net::train (tlb_ctx_create_multi): device d trains
// static_chunk(m, N, d) of every SGD group (runtime.cpp:138-145) on its shard of the data (shard layout,
// stride ceil(batch / N)); one flat persistent kernel per device, launched together, meets the others at a
// grid barrier over every CTA of every device, and the reduction phase sums ALL devices' rows -- EXACT: the
// per-example rows in example order, so the result is bit-identical to one device (and to the reference)
// for any device count, as the reference is for any worker count; fast: CTA partials in (device, CTA)
// order (deterministic for a given N).  Every device's parameter copy receives the update.
static int train_multi(tlb_ctx* c, HostImages src, const int32_t* labels, int64_t n, float* params, float rate,
                       int32_t epochs, int64_t batch, double* epoch_loss, tlb_epoch_cb on_epoch, void* user) {
  std::vector<tlb_ctx*> dv{c};
  for (tlb_ctx* p : c->peers) dv.push_back(p);
  const int N = (int)dv.size();
  const bool ex = exact(c);
  const int64_t spe = (n + batch - 1) / batch, full = n / batch, last = n - full * batch;
  const int64_t S = (batch + N - 1) / N;  // shard stride
  auto static_chunk = [](int64_t m, int workers, int w, int64_t& lo, int64_t& hi) {  // runtime.cpp:138-145
    const int64_t block = (m + workers - 1) / workers;
    lo = std::min<int64_t>((int64_t)w * block, m);
    hi = std::min<int64_t>(lo + block, m);
  };
  const int threads = 512;
  // co-residency: devices listed more than once (one-GPU tests) share its SMs
  int G = 1 << 30;
  for (int d = 0; d < N; ++d) {
    int share = 0;
    for (int e = 0; e < N; ++e) share += dv[e]->device == dv[d]->device;
    const int occ = std::max(1, dv[d]->occ_train[ex ? 1 : 0][1]);
    G = std::min(G, std::max(1, occ * dv[d]->sm_count / share));
  }
  const int64_t rows = ex ? S : G;
  const size_t elem = src.u8 ? 1 : sizeof(float);
  const void* img_host = src.u8 ? static_cast<const void*>(src.u8) : static_cast<const void*>(src.f32);
  std::vector<float> h_par(TLB_PSTRIDE, 0.0f);
  std::memcpy(h_par.data(), params, TLB_NPARAM * sizeof(float));
  // per-device buffers and the shard upload (one 2-D copy for the full groups, one for the ragged tail)
  for (int d = 0; d < N; ++d) {
    tlb_ctx* x = dv[d];
    TLB_TRY(set_device(x));
    TLB_CUDA(x->md_img.ensure((size_t)spe * S * 784 * sizeof(float)));
    TLB_CUDA(x->md_lab.ensure((size_t)spe * S * sizeof(int32_t)));
    if (src.u8) TLB_CUDA(x->md_u8.ensure((size_t)spe * S * 784));
    TLB_CUDA(x->md_p.ensure(TLB_PSTRIDE * sizeof(float)));
    TLB_CUDA(x->md_loss.ensure((size_t)std::max(epochs, 1) * sizeof(double)));
    TLB_CUDA(x->md_work.ensure((size_t)std::max<int64_t>(rows, 1) * TLB_PSTRIDE * sizeof(float)));
    TLB_CUDA(x->md_losses.ensure((size_t)S * sizeof(float)));
    TLB_CUDA(x->md_lpart.ensure((size_t)G * sizeof(double)));
    void* dst = src.u8 ? x->md_u8.p : x->md_img.p;
    int64_t lo, hi;
    static_chunk(batch, N, d, lo, hi);
    if (full > 0 && hi > lo) {
      TLB_CUDA(cudaMemcpy2DAsync(dst, S * 784 * elem, static_cast<const char*>(img_host) + lo * 784 * elem,
                                 batch * 784 * elem, (hi - lo) * 784 * elem, full, cudaMemcpyHostToDevice, x->stream));
      TLB_CUDA(cudaMemcpy2DAsync(x->md_lab.p, S * sizeof(int32_t), labels + lo, batch * sizeof(int32_t),
                                 (hi - lo) * sizeof(int32_t), full, cudaMemcpyHostToDevice, x->stream));
    }
    if (last > 0) {
      static_chunk(last, N, d, lo, hi);
      if (hi > lo) {
        TLB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + full * S * 784 * elem,
                                 static_cast<const char*>(img_host) + (full * batch + lo) * 784 * elem,
                                 (hi - lo) * 784 * elem, cudaMemcpyHostToDevice, x->stream));
        TLB_CUDA(cudaMemcpyAsync(static_cast<int32_t*>(x->md_lab.p) + full * S, labels + full * batch + lo,
                                 (hi - lo) * sizeof(int32_t), cudaMemcpyHostToDevice, x->stream));
      }
    }
    if (src.u8)
      TLB_CUDA(tlb::launch_pixels_to_f32(static_cast<const uint8_t*>(x->md_u8.p), static_cast<float*>(x->md_img.p),
                                         spe * S * 784, x->stream));
    TLB_CUDA(cudaMemcpyAsync(x->md_p.p, h_par.data(), TLB_PSTRIDE * sizeof(float), cudaMemcpyHostToDevice, x->stream));
    TLB_CUDA(cudaMemsetAsync(x->dev_err.p, 0, 4 * sizeof(unsigned int), x->stream));
  }
  TLB_TRY(set_device(c));
  TLB_CUDA(c->md_bar.ensure(sizeof(unsigned int)));
  auto launch = [&](int32_t e0, int32_t ne) -> int {
    for (tlb_ctx* x : dv) {
      TLB_CUDA(cudaSetDevice(x->device));
      TLB_CUDA(cudaStreamSynchronize(x->stream));
    }
    TLB_TRY(set_device(c));
    TLB_CUDA(cudaMemset(c->md_bar.p, 0, sizeof(unsigned int)));  // the kernels meet on it from step 0
    TLB_CUDA(cudaDeviceSynchronize());
    for (int d = 0; d < N; ++d) {
      tlb_ctx* x = dv[d];
      TLB_TRY(set_device(x));
      tlb::TrainArgs a{};
      a.images = static_cast<const float*>(x->md_img.p);
      a.images_wb = static_cast<float*>(x->md_img.p);
      a.labels = static_cast<const int32_t*>(x->md_lab.p);
      a.n = n;
      a.batch = batch;
      a.rate = rate;
      a.steps_per_epoch = spe;
      a.step_begin = (int64_t)e0 * spe;
      a.step_end = (int64_t)(e0 + ne) * spe;
      a.params = static_cast<float*>(x->md_p.p);
      a.work = static_cast<float*>(x->md_work.p);
      a.losses = static_cast<float*>(x->md_losses.p);
      a.loss_part = static_cast<double*>(x->md_lpart.p);
      a.epoch_loss = static_cast<double*>(x->md_loss.p);
      a.barrier = static_cast<unsigned int*>(c->md_bar.p);
      a.dp_world = N;
      a.dp_rank = d;
      a.local_stride = S;
      a.md_n = N;
      for (int e = 0; e < N; ++e) {
        a.md_work[e] = static_cast<float*>(dv[e]->md_work.p);
        a.md_losses[e] = static_cast<float*>(dv[e]->md_losses.p);
        a.md_loss_part[e] = static_cast<double*>(dv[e]->md_lpart.p);
        a.md_params[e] = static_cast<float*>(dv[e]->md_p.p);
        a.md_epoch_loss[e] = static_cast<double*>(dv[e]->md_loss.p);
      }
      a.md_bar = static_cast<unsigned int*>(c->md_bar.p);
      a.dp_error = static_cast<unsigned int*>(x->dev_err.p);
      a.fix_err = static_cast<unsigned int*>(x->dev_err.p) + 1;
      a.dp_timeout_cycles = (long long)(kWaitLimitSeconds * 2.0e9);
      TLB_CUDA(tlb::launch_train(ex, a, G, threads, x->stream));
    }
    for (tlb_ctx* x : dv) {
      TLB_CUDA(cudaSetDevice(x->device));
      TLB_CUDA(cudaStreamSynchronize(x->stream));
    }
    for (int d = 0; d < N; ++d) {
      unsigned int w[4];
      TLB_CUDA(cudaSetDevice(dv[d]->device));
      TLB_CUDA(cudaMemcpy(w, dv[d]->dev_err.p, sizeof(w), cudaMemcpyDeviceToHost));
      if (w[0] || w[1]) {
        TLB_CUDA(cudaMemset(dv[d]->dev_err.p, 0, sizeof(w)));
        return fail(TLB_ERR_CUDA, "train: device " + std::to_string(dv[d]->device) + " (rank " + std::to_string(d) +
                                      ") timed out at the cross-device grid barrier (another device never arrived)");
      }
    }
    return TLB_OK;
  };
  std::vector<double> losses((size_t)std::max(epochs, 1));
  if (!on_epoch) {
    TLB_TRY(launch(0, epochs));
  } else {
    for (int32_t e = 0; e < epochs; ++e) {
      TLB_TRY(launch(e, 1));
      TLB_TRY(set_device(c));
      TLB_CUDA(cudaMemcpy(&losses[(size_t)e], static_cast<double*>(c->md_loss.p) + e, sizeof(double),
                          cudaMemcpyDeviceToHost));
      on_epoch(e + 1, losses[(size_t)e], user);
    }
  }
  TLB_TRY(set_device(c));
  TLB_CUDA(cudaMemcpy(params, c->md_p.p, TLB_NPARAM * sizeof(float), cudaMemcpyDeviceToHost));
  if (epoch_loss) TLB_CUDA(cudaMemcpy(epoch_loss, c->md_loss.p, epochs * sizeof(double), cudaMemcpyDeviceToHost));
  return TLB_OK;
}

static int train_host(tlb_ctx* c, HostImages src, const int32_t* labels, int64_t n, float* params, float rate,
                      int32_t epochs, int64_t batch, double* epoch_loss, tlb_epoch_cb on_epoch, void* user) {
  const void* images = src.u8 ? static_cast<const void*>(src.u8) : static_cast<const void*>(src.f32);
  HostTrace ht;
  if (!c || !params) return fail(TLB_ERR_ARG, "tlb_train: null argument");
  TLB_TRY(check_train_args(n, epochs, rate, batch));
  if (!images || !labels) return fail(TLB_ERR_ARG, "tlb_train: null dataset");
  for (int64_t i = 0; i < n; ++i)  // mnist::one_hot (mnist.cpp:161-167) of every label
    if (labels[i] < 0 || labels[i] > 9)
      return fail(TLB_ERR_VALUE, "one_hot: label " + std::to_string(labels[i]) + " out of range 0..9");
  TLB_TRY(set_device(c));
  ht.mark("checked");
  if (epochs == 0) return TLB_OK;
  if (!c->peers.empty()) return train_multi(c, src, labels, n, params, rate, epochs, batch, epoch_loss, on_epoch, user);
  float* d_img;
  int32_t* d_lab;
  float* d_p;
  double* d_loss;
  // The dataset streams in on the copy stream while the first epoch already trains on the chunks
  // that have landed; labels/params are tiny and go first.
  // Default: a ramp of whole SGD groups -- 1 | 1 | 2 | 4 ... up to C groups of >= 1 MiB (4 at batch
  // 100), then C groups per chunk: the first step waits for one group only, the next chunks double
  // while the copy gets ahead, and the ~3 us per-chunk copy-engine/driver overhead stays <= 5% on the
  // slowest VM links (pinned H2D measured 18-55 GB/s).  TLB_INGEST_CHUNK=<images> = fixed chunks,
  // 0 = unbounded geometric growth.
  static const int64_t chunk_env = [] {
    const char* e = std::getenv("TLB_INGEST_CHUNK");
    return e ? std::max<int64_t>(0, std::atoll(e)) : (int64_t)-1;
  }();
  const int64_t group_bytes = batch * 784 * (int64_t)sizeof(float);
  int64_t cap = 1;  // ramp cap C: groups per steady chunk, a power of two
  while (cap * group_bytes < (int64_t)(1 << 20)) cap *= 2;
  // Large groups train on the batched kernel, whose CTAs take the group's rounds interleaved while chunks
  // are in flight (round r on CTA r % grid, batch_train.cu): any prefix of a group feeds every CTA, so
  // chunks of batch / 8 images (1k..16k) are consumed as they land -- with whole-group chunks the first
  // group's bytes had to arrive before the last CTA could start (16k: ~0.25 ms of a 1.6 ms call).
  const bool batched_launch = !exact(c) && c->grid_override == 0 && use_batched(c, std::min(batch, n));
  const int64_t chunk = chunk_env >= 0       ? chunk_env
                        : batched_launch ? std::min<int64_t>(16384, std::max<int64_t>(1024, batch / 8))
                                         : -cap;
  const int64_t nchunks = ingest_chunks(n, chunk, batch);
  // Byte source: the chunks of bytes (1/4 of the fp32 volume) stream in like fp32 chunks and the train
  // kernel converts each image where it is trained (a separate conversion kernel could not run beside a
  // persistent train kernel that may hold every SM); without stream memory operations the bytes land and
  // are converted before the kernel.
  const bool overlap = write_value32() != nullptr;
  TLB_TRY(stage_out(c, 0, (size_t)n * 784, &d_img));
  if (src.u8) TLB_TRY(stage_out(c, 4, (size_t)n * 784, &src.d_u8));
  if (overlap) {
    if ((size_t)nchunks * sizeof(unsigned int) > c->ready.cap) {
      TLB_CUDA(cudaStreamSynchronize(c->copy_stream));
      TLB_CUDA(cudaStreamSynchronize(c->copy_stream2));
      TLB_CUDA(c->ready.ensure((size_t)nchunks * sizeof(unsigned int)));
      TLB_CUDA(cudaMemset(c->ready.p, 0, c->ready.cap));
      c->ready_token = 0;
    }
    if (++c->ready_token == 0) {  // wrapped: restart the token sequence from clean flags
      TLB_CUDA(cudaStreamSynchronize(c->copy_stream));
      TLB_CUDA(cudaStreamSynchronize(c->copy_stream2));
      TLB_CUDA(cudaMemset(c->ready.p, 0, c->ready.cap));
      c->ready_token = 1;
    }
    // The copy stream may only overwrite the staging buffer after all earlier work on the context
    // stream: gate it on an event recorded now, before this call's kernel (which waits on the copies).
    TLB_CUDA(cudaEventRecord(c->copy_gate, c->stream));
  } else if (n && src.u8) {  // no stream memory operations: bytes first, converted before the kernel
    TLB_CUDA(cudaMemcpyAsync(src.d_u8, src.u8, (size_t)n * 784, cudaMemcpyHostToDevice, c->stream));
    TLB_CUDA(tlb::launch_pixels_to_f32(src.d_u8, d_img, n * 784, c->stream));
  } else if (n) {
    TLB_CUDA(cudaMemcpyAsync(d_img, src.f32, (size_t)n * 784 * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  }
  const unsigned int* rdy = overlap ? static_cast<const unsigned int*>(c->ready.p) : nullptr;
  TLB_TRY(stage_in(c, 1, labels, (size_t)n, &d_lab));
  // params / losses / watchdog words: the context's result block (one D2H at the end) mirrored by a pinned
  // host block (async copies, one sync); calls of more than kOutEpochs epochs stage params / losses apart
  const bool one_copy = epochs <= kOutEpochs;
  char* const ob = static_cast<char*>(c->outblk.p);
  if (one_copy) {
    d_p = reinterpret_cast<float*>(ob + kOutParamOff);
    d_loss = reinterpret_cast<double*>(ob + kOutLossOff);
  } else {
    TLB_TRY(stage_out(c, 2, TLB_PSTRIDE, &d_p));
    TLB_TRY(stage_out(c, 3, (size_t)epochs, &d_loss));
  }
  TLB_CUDA(cudaMemsetAsync(d_p, 0, TLB_PSTRIDE * sizeof(float), c->stream));
  TLB_CUDA(c->pin.ensure(kOutLossOff + (size_t)epochs * sizeof(double)));
  char* const hb = static_cast<char*>(c->pin.p);
  unsigned int* h_err = reinterpret_cast<unsigned int*>(hb);  // [0..3] dev_err, [4..6] ready_err
  float* h_p = reinterpret_cast<float*>(hb + kOutParamOff);
  double* h_loss = reinterpret_cast<double*>(hb + kOutLossOff);
  std::memcpy(h_p, params, TLB_NPARAM * sizeof(float));
  TLB_CUDA(cudaMemcpyAsync(d_p, h_p, TLB_NPARAM * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  // Launch the kernel first, then enqueue the chunk copies (the host's enqueue calls overlap the running
  // kernel, which polls the ready flags): pinned sources DMA straight from the caller's memory, pageable
  // ones through the pinned bounce slots filled by host worker threads (ingest_pageable).
  // TLB_PAGEABLE_COPIES_FIRST=1 restores the earlier pageable policy (copies enqueued before the kernel).
  ht.mark("staged");
  static const bool pageable_first = [] {
    const char* e = std::getenv("TLB_PAGEABLE_COPIES_FIRST");
    return e && std::atoi(e) == 1;
  }();
  const bool pageable = overlap && !is_pinned(images);
  const bool copies_first = pageable && pageable_first;
  PageablePlan plan;
  if (pageable && !copies_first) TLB_TRY(plan_pageable(c, src.u8 != nullptr, n, chunk, batch, &plan));
  auto ingest = [&]() {
    return pageable && !copies_first ? ingest_pageable(c, src, d_img, plan, c->ready_token)
                                     : ingest_images(c, src, d_img, n, chunk, batch, c->ready_token);
  };
  // a one-epoch call never reads the fp32 images back: byte-ingested images skip the write-back
  c->one_epoch_call = epochs == 1;
  struct ResetFlag {
    tlb_ctx* c;
    ~ResetFlag() { c->one_epoch_call = false; }
  } reset_flag{c};
  if (copies_first) TLB_TRY(ingest_images(c, src, d_img, n, chunk, batch, c->ready_token));
  if (!on_epoch) {
    ht.event(c->stream);
    TLB_TRY(enqueue_train(c, d_img, d_lab, n, d_p, rate, 0, epochs, batch, d_loss, 0, 0, -1, nullptr, nullptr,
                          rdy, c->ready_token, chunk, nullptr, src.d_u8));
    ht.event(c->stream);
    ht.mark("launched");
    if (overlap && !copies_first) TLB_TRY(ingest());
    ht.mark("ingest_enqueued");
  } else {
    for (int32_t e = 0; e < epochs; ++e) {
      TLB_TRY(enqueue_train(c, d_img, d_lab, n, d_p, rate, e, 1, batch, d_loss, 0, 0, -1, nullptr, nullptr,
                            e == 0 ? rdy : nullptr, c->ready_token, chunk, nullptr, src.d_u8));
      if (e == 0 && overlap && !copies_first) TLB_TRY(ingest());
      double mean = 0.0;
      TLB_TRY(fetch(c, &mean, d_loss + e, 1));
      on_epoch(e + 1, mean, user);
    }
  }
  if (one_copy) {  // error words + params (+ losses) in one copy
    TLB_CUDA(cudaMemcpyAsync(hb, ob, kOutLossOff + (epoch_loss ? epochs * sizeof(double) : 0), cudaMemcpyDeviceToHost,
                             c->stream));
  } else {
    TLB_CUDA(cudaMemcpyAsync(h_p, d_p, TLB_NPARAM * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    if (epoch_loss) TLB_CUDA(cudaMemcpyAsync(h_loss, d_loss, epochs * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    TLB_CUDA(cudaMemcpyAsync(h_err, ob, 8 * sizeof(unsigned int), cudaMemcpyDeviceToHost, c->stream));
  }
  ht.event(c->stream);
  ht.mark("d2h_enqueued");
  TLB_CUDA(cudaStreamSynchronize(c->stream));
  ht.mark("stream_synced");
  {
    const unsigned int dev_words[4] = {h_err[0], h_err[1], h_err[2], h_err[3]};
    TLB_TRY(device_status(c, dev_words));  // params stay untouched on a device failure
  }
  std::memcpy(params, h_p, TLB_NPARAM * sizeof(float));
  if (epoch_loss) std::memcpy(epoch_loss, h_loss, epochs * sizeof(double));
  if (overlap) {
    TLB_CUDA(cudaStreamSynchronize(c->copy_stream));  // (the kernel consumed every chunk: already done)
    TLB_CUDA(cudaStreamSynchronize(c->copy_stream2));
    const unsigned int err[3] = {h_err[4], h_err[5], h_err[6]};
    if (err[0]) {
      TLB_CUDA(cudaMemset(c->ready_err.p, 0, sizeof(err)));
      return fail(TLB_ERR_CUDA, "tlb_train: dataset chunk " + std::to_string(err[1]) + " never became ready (flag " +
                                    std::to_string(err[2]) + ", token " + std::to_string(c->ready_token) + ")");
    }
  }
  ht.mark("done");
  return TLB_OK;
}

int tlb_host_register(tlb_ctx* c, const void* ptr, size_t bytes) {
  if (!c || !ptr || bytes == 0) return fail(TLB_ERR_ARG, "tlb_host_register: null argument");
  TLB_TRY(set_device(c));
  const cudaError_t e = cudaHostRegister(const_cast<void*>(ptr), bytes,
                                         cudaHostRegisterPortable | cudaHostRegisterReadOnly);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(TLB_ERR_CUDA, std::string("tlb_host_register: ") + cudaGetErrorString(e));
  }
  return TLB_OK;
}

int tlb_host_unregister(tlb_ctx* c, const void* ptr) {
  if (!c || !ptr) return fail(TLB_ERR_ARG, "tlb_host_unregister: null argument");
  TLB_TRY(set_device(c));
  const cudaError_t e = cudaHostUnregister(const_cast<void*>(ptr));
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(TLB_ERR_CUDA, std::string("tlb_host_unregister: ") + cudaGetErrorString(e));
  }
  return TLB_OK;
}

int tlb_train(tlb_ctx* c, const float* images, const int32_t* labels, int64_t n, float* params, float rate,
              int32_t epochs, int64_t batch, double* epoch_loss, tlb_epoch_cb on_epoch, void* user) {
  if (c && params && !images && n > 0) return fail(TLB_ERR_ARG, "tlb_train: null dataset");
  HostImages src;
  src.f32 = images;
  return train_host(c, src, labels, n, params, rate, epochs, batch, epoch_loss, on_epoch, user);
}

int tlb_train_u8(tlb_ctx* c, const uint8_t* pixels, const int32_t* labels, int64_t n, float* params, float rate,
                 int32_t epochs, int64_t batch, double* epoch_loss, tlb_epoch_cb on_epoch, void* user) {
  if (c && params && !pixels && n > 0) return fail(TLB_ERR_ARG, "tlb_train_u8: null dataset");
  HostImages src;
  src.u8 = pixels;
  return train_host(c, src, labels, n, params, rate, epochs, batch, epoch_loss, on_epoch, user);
}

int tlb_train_idx(tlb_ctx* c, const uint8_t* image_file, size_t image_bytes, const uint8_t* label_file,
                  size_t label_bytes, float* params, float rate, int32_t epochs, int64_t batch, double* epoch_loss,
                  tlb_epoch_cb on_epoch, void* user) {
  if (!c || !params || !image_file || !label_file) return fail(TLB_ERR_ARG, "tlb_train_idx: null argument");
  int64_t idim[3], ldim[3];
  size_t ioff = 0, loff = 0;
  TLB_TRY(tlb_idx_parse(image_file, image_bytes, 0, idim, &ioff));
  TLB_TRY(tlb_idx_parse(label_file, label_bytes, 1, ldim, &loff));
  if (idim[1] != 28 || idim[2] != 28)  // mnist::MnistSet geometry (mnist.hpp:14-19)
    return fail(TLB_ERR_FORMAT, "dataset: images have shape [" + std::to_string(idim[0]) + "," +
                                    std::to_string(idim[1]) + "," + std::to_string(idim[2]) + "], expected [n,28,28]");
  if (idim[0] != ldim[0])
    return fail(TLB_ERR_FORMAT, "dataset: " + std::to_string(idim[0]) + " images but " + std::to_string(ldim[0]) +
                                    " labels");
  std::vector<int32_t> labels((size_t)ldim[0]);
  for (int64_t i = 0; i < ldim[0]; ++i) {
    labels[(size_t)i] = label_file[loff + (size_t)i];
    if (labels[(size_t)i] > 9)
      return fail(TLB_ERR_VALUE, "idx: label " + std::to_string(labels[(size_t)i]) + " at offset " +
                                     std::to_string(loff + (size_t)i) + " out of range 0..9");
  }
  return tlb_train_u8(c, image_file + ioff, labels.data(), idim[0], params, rate, epochs, batch, epoch_loss, on_epoch,
                      user);
}

static int run_cells(tlb_ctx* c, const float* images, const int32_t* labels, const float* targets, int64_t n,
                     const float* params, float* cells, float* acts, float* yhat, const float* acts_in = nullptr,
                     float* grads_only = nullptr) {
  if (!c || !params || (n > 0 && !images)) return fail(TLB_ERR_ARG, "null argument");
  if (n < 0) return fail(TLB_ERR_ARG, "negative count");
  if (n == 0) return TLB_OK;
  TLB_TRY(set_device(c));
  float *d_img, *d_p, *d_cells = nullptr, *d_acts = nullptr, *d_yhat = nullptr, *d_tg = nullptr;
  int32_t* d_lab = nullptr;
  TLB_TRY(stage_in(c, 0, images, (size_t)n * 784, &d_img));
  TLB_TRY(stage_out(c, 2, TLB_PSTRIDE, &d_p));
  TLB_CUDA(cudaMemsetAsync(d_p, 0, TLB_PSTRIDE * sizeof(float), c->stream));
  TLB_CUDA(cudaMemcpyAsync(d_p, params, TLB_NPARAM * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  if (targets) TLB_TRY(stage_in(c, 1, targets, (size_t)n * 10, &d_tg));
  else if (labels) TLB_TRY(stage_in(c, 1, labels, (size_t)n, &d_lab));
  // slot 3: cells rows [n][3904] (loss rides in column 3898); slot 4: acts; slot 5: yhat
  if (cells || grads_only) TLB_TRY(stage_out(c, 3, (size_t)n * TLB_PSTRIDE, &d_cells));
  float* d_acts_in = nullptr;
  if (acts_in) TLB_TRY(stage_in(c, 6, acts_in, (size_t)n * TLB_NACT, &d_acts_in));
  if (acts) TLB_TRY(stage_out(c, 4, (size_t)n * TLB_NACT, &d_acts));
  if (yhat || cells) TLB_TRY(stage_out(c, 5, (size_t)n * 11, &d_yhat));
  tlb::CellArgs a{};
  a.images = d_img;
  a.labels = d_lab;
  a.targets = d_tg;
  a.n = n;
  a.params = d_p;
  a.cells = d_cells;
  a.losses = d_yhat ? d_yhat + n * 10 : nullptr;
  a.acts = d_acts;
  a.yhat = d_yhat;
  a.acts_in = d_acts_in;
  TLB_CUDA(tlb::launch_cells(exact(c), a, plain_grid(c, n), c->stream));
  if (grads_only)
    TLB_CUDA(cudaMemcpy2DAsync(grads_only, TLB_NPARAM * sizeof(float), d_cells, TLB_PSTRIDE * sizeof(float),
                               TLB_NPARAM * sizeof(float), (size_t)n, cudaMemcpyDeviceToHost, c->stream));
  if (cells) {
    // rows of 3904 -> host cells of 3899 (3898 grads + loss)
    TLB_CUDA(cudaMemcpy2DAsync(cells, TLB_CELL * sizeof(float), d_cells, TLB_PSTRIDE * sizeof(float),
                               TLB_NPARAM * sizeof(float), (size_t)n, cudaMemcpyDeviceToHost, c->stream));
    TLB_CUDA(cudaMemcpy2DAsync(cells + TLB_NPARAM, TLB_CELL * sizeof(float), d_yhat + n * 10, sizeof(float),
                               sizeof(float), (size_t)n, cudaMemcpyDeviceToHost, c->stream));
  }
  if (acts) TLB_CUDA(cudaMemcpyAsync(acts, d_acts, (size_t)n * TLB_NACT * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  if (yhat) TLB_CUDA(cudaMemcpyAsync(yhat, d_yhat, (size_t)n * 10 * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  TLB_CUDA(cudaStreamSynchronize(c->stream));
  return TLB_OK;
}

int tlb_forward(tlb_ctx* c, const float* images, int64_t n, const float* params, float* yhat, float* acts) {
  return run_cells(c, images, nullptr, nullptr, n, params, nullptr, acts, yhat);
}

int tlb_forward_backward(tlb_ctx* c, const float* images, const int32_t* labels, const float* targets, int64_t n,
                         const float* params, float* cells, float* acts) {
  if (!targets && !labels) return fail(TLB_ERR_ARG, "tlb_forward_backward: need labels or targets");
  if (!cells) return fail(TLB_ERR_ARG, "tlb_forward_backward: null cells");
  if (!targets)
    for (int64_t i = 0; i < n; ++i)
      if (labels[i] < 0 || labels[i] > 9)
        return fail(TLB_ERR_VALUE, "one_hot: label " + std::to_string(labels[i]) + " out of range 0..9");
  return run_cells(c, images, labels, targets, n, params, cells, acts, nullptr);
}

int tlb_backward(tlb_ctx* c, const float* images, const float* acts, const float* targets, int64_t n,
                 const float* params, float* grads) {
  if (!acts || !targets || !grads) return fail(TLB_ERR_ARG, "tlb_backward: null argument");
  return run_cells(c, images, nullptr, targets, n, params, nullptr, nullptr, nullptr, acts, grads);
}

int tlb_loss(tlb_ctx* c, const float* yhat, const float* y, int64_t n, float* out) {
  if (!c || !yhat || !y || !out) return fail(TLB_ERR_ARG, "tlb_loss: null argument");
  if (n <= 0) return TLB_OK;
  TLB_TRY(set_device(c));
  float *d_h, *d_y, *d_o;
  TLB_TRY(stage_in(c, 0, yhat, (size_t)n * 10, &d_h));
  TLB_TRY(stage_in(c, 1, y, (size_t)n * 10, &d_y));
  TLB_TRY(stage_out(c, 2, (size_t)n, &d_o));
  TLB_CUDA(tlb::nn_loss(d_h, d_y, n, d_o, c->stream));
  return fetch(c, out, d_o, (size_t)n);
}

int tlb_evaluate(tlb_ctx* c, const float* images, const int32_t* labels, int64_t n, const float* params,
                 int32_t* pred, int64_t* correct) {
  if (!c || !params) return fail(TLB_ERR_ARG, "tlb_evaluate: null argument");
  if (n == 0) return fail(TLB_ERR_ERROR, "evaluate: empty dataset");
  if (n < 0 || !images) return fail(TLB_ERR_ARG, "tlb_evaluate: bad dataset");
  TLB_TRY(set_device(c));
  float *d_img, *d_p;
  int32_t *d_lab = nullptr, *d_pred = nullptr;
  unsigned long long* d_cnt;
  TLB_TRY(stage_in(c, 0, images, (size_t)n * 784, &d_img));
  if (labels) TLB_TRY(stage_in(c, 1, labels, (size_t)n, &d_lab));
  TLB_TRY(stage_out(c, 2, TLB_PSTRIDE, &d_p));
  TLB_CUDA(cudaMemsetAsync(d_p, 0, TLB_PSTRIDE * sizeof(float), c->stream));
  TLB_CUDA(cudaMemcpyAsync(d_p, params, TLB_NPARAM * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  if (pred) TLB_TRY(stage_out(c, 3, (size_t)n, &d_pred));
  TLB_TRY(stage_out(c, 4, 1, &d_cnt));
  TLB_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), c->stream));
  TLB_TRY(tlb_evaluate_device(c, d_img, d_lab, n, d_p, d_pred, d_cnt));
  if (pred) TLB_CUDA(cudaMemcpyAsync(pred, d_pred, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  unsigned long long cnt = 0;
  TLB_TRY(fetch(c, &cnt, d_cnt, 1));
  if (correct) *correct = (int64_t)cnt;
  return TLB_OK;
}

int tlb_sgd_step(tlb_ctx* c, const float* params, const float* grads, float rate, int64_t batch, float* out) {
  if (!c || !params || !grads || !out) return fail(TLB_ERR_ARG, "tlb_sgd_step: null argument");
  if (batch < 1) return fail(TLB_ERR_ERROR, "sgd_step: batch must be >= 1");
  TLB_TRY(set_device(c));
  float *d_p, *d_g, *d_o;
  TLB_TRY(stage_in(c, 0, params, TLB_NPARAM, &d_p));
  TLB_TRY(stage_in(c, 1, grads, TLB_NPARAM, &d_g));
  TLB_TRY(stage_out(c, 2, TLB_NPARAM, &d_o));
  TLB_CUDA(tlb::launch_sgd(d_p, d_g, rate, batch, d_o, TLB_NPARAM, c->stream));
  return fetch(c, out, d_o, TLB_NPARAM);
}

// ---- network, device buffers ----------------------------------------------------------------
int tlb_train_device(tlb_ctx* c, const float* d_images, const int32_t* d_labels, int64_t n, float* d_params,
                     float rate, int32_t epoch_begin, int32_t epochs, int64_t batch, double* d_epoch_loss) {
  if (!c || !d_params || !d_epoch_loss) return fail(TLB_ERR_ARG, "tlb_train_device: null argument");
  TLB_TRY(check_train_args(n, epochs, rate, batch));
  if (epoch_begin < 0) return fail(TLB_ERR_ARG, "tlb_train_device: negative epoch_begin");
  TLB_TRY(set_device(c));
  return enqueue_train(c, d_images, d_labels, n, d_params, rate, epoch_begin, epochs, batch, d_epoch_loss);
}

int tlb_train_shard_device(tlb_ctx* c, const float* d_images, const int32_t* d_labels, int64_t n, int64_t batch,
                           int64_t group, int64_t shard_lo, int64_t shard_hi, const float* d_params,
                           float* d_grad_sum, double* d_loss_sum) {
  if (!c || !d_params || !d_grad_sum || !d_loss_sum) return fail(TLB_ERR_ARG, "tlb_train_shard_device: null argument");
  TLB_TRY(check_train_args(n, 1, 1.0f, batch));
  const int64_t spe = (n + batch - 1) / batch;
  if (group < 0 || group >= spe) return fail(TLB_ERR_ARG, "tlb_train_shard_device: group out of range");
  if (shard_lo < 0 || shard_hi < shard_lo) return fail(TLB_ERR_ARG, "tlb_train_shard_device: bad shard");
  TLB_TRY(set_device(c));
  return enqueue_train(c, d_images, d_labels, n, const_cast<float*>(d_params), 1.0f, 0, 1, batch, nullptr, shard_lo,
                       shard_hi, group, d_grad_sum, d_loss_sum);
}

size_t tlb_dp_workspace_bytes(void) { return tlb::dp_workspace_bytes(); }

int tlb_train_dp_device(tlb_ctx* c, const float* d_images, const int32_t* d_labels, int64_t n, float* d_params,
                        float rate, int32_t epoch_begin, int32_t epochs, int64_t batch, double* d_epoch_loss, int world,
                        int rank, void* const* peer_ws, uint64_t seq_base, double timeout_s) {
  if (!c || !d_params || !d_epoch_loss || !peer_ws) return fail(TLB_ERR_ARG, "tlb_train_dp_device: null argument");
  TLB_TRY(check_train_args(n, epochs, rate, batch));
  if (world < 1 || world > 8 || rank < 0 || rank >= world)
    return fail(TLB_ERR_ARG, "tlb_train_dp_device: world must be 1..8 and 0 <= rank < world");
  for (int r = 0; r < world; ++r)
    if (!peer_ws[r]) return fail(TLB_ERR_ARG, "tlb_train_dp_device: null peer workspace");
  if (exact(c)) return fail(TLB_ERR_ARG, "tlb_train_dp_device: fused data parallelism runs in fast mode");
  TLB_TRY(set_device(c));
  const DpArgs dp{world, rank, peer_ws, seq_base, (long long)(timeout_s * 2.0e9)};
  return enqueue_train(c, d_images, d_labels, n, d_params, rate, epoch_begin, epochs, batch, d_epoch_loss, 0, 0, -1,
                       nullptr, nullptr, nullptr, 0, 1, &dp);
}

int tlb_apply_sgd_device(tlb_ctx* c, float* d_params, const float* d_grad_sum, float rate, int64_t m) {
  if (!c || !d_params || !d_grad_sum) return fail(TLB_ERR_ARG, "tlb_apply_sgd_device: null argument");
  if (m < 1) return fail(TLB_ERR_ERROR, "sgd_step: batch must be >= 1");
  TLB_TRY(set_device(c));
  TLB_CUDA(tlb::launch_sgd(d_params, d_grad_sum, rate, m, d_params, TLB_NPARAM, c->stream));
  return TLB_OK;
}

int tlb_evaluate_device(tlb_ctx* c, const float* d_images, const int32_t* d_labels, int64_t n, const float* d_params,
                        int32_t* d_pred, unsigned long long* d_correct) {
  if (!c || !d_params) return fail(TLB_ERR_ARG, "tlb_evaluate_device: null argument");
  if (n <= 0) return TLB_OK;
  TLB_TRY(set_device(c));
  tlb::EvalArgs a{d_images, d_labels, n, d_params, d_pred, nullptr, d_correct, nullptr};
  if (!exact(c) && c->grid_override == 0 && c->threads_override == 0) {  // batched forward-only kernel
    TLB_CUDA(c->eval_claim.ensure(sizeof(unsigned long long)));
    a.claim = static_cast<unsigned long long*>(c->eval_claim.p);
    TLB_CUDA(tlb::launch_infer(a, c->sm_count, c->stream));
    return TLB_OK;
  }
  const int threads = pick_threads(c, n);
  TLB_CUDA(tlb::launch_eval(exact(c), a, plain_grid(c, n, threads), threads, c->stream));
  return TLB_OK;
}

// ---- generic ops ----------------------------------------------------------------------------
int tlb_nn_conv_shape(const int64_t* in, int ir, const int64_t* k, int kr, int64_t* out, int* orank) {
  TLB_TRY(check_rank(ir, "conv"));
  TLB_TRY(check_rank(kr, "conv"));
  TLB_TRY(conv_shape(in, ir, k, kr, out));
  if (orank) *orank = ir;
  return TLB_OK;
}

int tlb_nn_mconv_shape(const int64_t* in, int ir, const int64_t* k, int kr, const int64_t* b, int br, int64_t* out,
                       int* orank) {
  TLB_TRY(check_rank(ir, "mconv"));
  TLB_TRY(check_rank(kr, "mconv"));
  int r = 0;
  TLB_TRY(mconv_shape(in, ir, k, kr, b, br, out, &r));
  if (orank) *orank = r;
  return TLB_OK;
}

int tlb_nn_avgpool_shape(const int64_t* s, int r, int64_t* out, int* orank) {
  TLB_TRY(check_rank(r, "avgpool"));
  TLB_TRY(avgpool_shape(s, r, out));
  if (orank) *orank = r;
  return TLB_OK;
}

int tlb_nn_backavgpool_shape(const int64_t* s, int r, int64_t* out, int* orank) {
  TLB_TRY(check_rank(r, "backavgpool"));
  TLB_TRY(backavgpool_shape(s, r, out));
  if (orank) *orank = r;
  return TLB_OK;
}

int tlb_nn_backin_shape(const int64_t* d, int dr, const int64_t* k, int kr, const int64_t* in, int ir, int64_t* out,
                        int* orank) {
  TLB_TRY(check_rank(dr, "backin"));
  TLB_TRY(backin_shape(d, dr, k, kr, in, ir, out));
  if (orank) *orank = ir;
  return TLB_OK;
}

static int run_conv(tlb_ctx* c, const float* in, const int64_t* is, int r, const float* k, const int64_t* ks,
                    const float* b, int64_t nk, float* out) {
  TLB_TRY(set_device(c));
  int64_t os[8];
  for (int a = 0; a < r; ++a) os[a] = is[a] - ks[a] + 1;
  const int64_t nout = count_of(os, r) * nk;
  float *d_in, *d_k, *d_b = nullptr, *d_o;
  TLB_TRY(stage_in(c, 0, in, (size_t)count_of(is, r), &d_in));
  TLB_TRY(stage_in(c, 1, k, (size_t)(count_of(ks, r) * nk), &d_k));
  if (b) TLB_TRY(stage_in(c, 2, b, (size_t)nk, &d_b));
  TLB_TRY(stage_out(c, 3, (size_t)nout, &d_o));
  TLB_CUDA(tlb::nn_conv(d_in, is, d_k, ks, r, d_b, nk, d_o, c->stream));
  return fetch(c, out, d_o, (size_t)nout);
}

int tlb_nn_conv(tlb_ctx* c, const float* in, const int64_t* is, int ir, const float* k, const int64_t* ks, int kr,
                float* out) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  int64_t os[8];
  int orank;
  TLB_TRY(tlb_nn_conv_shape(is, ir, ks, kr, os, &orank));
  return run_conv(c, in, is, ir, k, ks, nullptr, 1, out);
}

int tlb_nn_mconv(tlb_ctx* c, const float* in, const int64_t* is, int ir, const float* k, const int64_t* ks, int kr,
                 const float* b, const int64_t* bs, int br, float* out) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  int64_t os[8];
  int orank;
  TLB_TRY(tlb_nn_mconv_shape(is, ir, ks, kr, bs, br, os, &orank));
  return run_conv(c, in, is, ir, k, ks + 1, b, ks[0], out);
}

int tlb_nn_sigmoid(tlb_ctx* c, const float* x, int64_t n, float* out) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  TLB_TRY(set_device(c));
  float *d_x, *d_o;
  TLB_TRY(stage_in(c, 0, x, (size_t)n, &d_x));
  TLB_TRY(stage_out(c, 1, (size_t)n, &d_o));
  TLB_CUDA(tlb::nn_sigmoid(d_x, n, d_o, c->stream));
  return fetch(c, out, d_o, (size_t)n);
}

int tlb_nn_backsigmoid(tlb_ctx* c, const float* d, const float* o, int64_t n, float* out) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  TLB_TRY(set_device(c));
  float *d_d, *d_op, *d_o;
  TLB_TRY(stage_in(c, 0, d, (size_t)n, &d_d));
  TLB_TRY(stage_in(c, 1, o, (size_t)n, &d_op));
  TLB_TRY(stage_out(c, 2, (size_t)n, &d_o));
  TLB_CUDA(tlb::nn_backsigmoid(d_d, d_op, n, d_o, c->stream));
  return fetch(c, out, d_o, (size_t)n);
}

int tlb_nn_avgpool(tlb_ctx* c, const float* in, const int64_t* s, int r, float* out) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  int64_t os[8];
  int orank;
  TLB_TRY(tlb_nn_avgpool_shape(s, r, os, &orank));
  TLB_TRY(set_device(c));
  float *d_in, *d_o;
  const int64_t nout = count_of(os, r);
  TLB_TRY(stage_in(c, 0, in, (size_t)count_of(s, r), &d_in));
  TLB_TRY(stage_out(c, 1, (size_t)nout, &d_o));
  TLB_CUDA(tlb::nn_avgpool(d_in, s, r, d_o, c->stream));
  return fetch(c, out, d_o, (size_t)nout);
}

int tlb_nn_backavgpool(tlb_ctx* c, const float* d, const int64_t* s, int r, float* out) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  int64_t os[8];
  int orank;
  TLB_TRY(tlb_nn_backavgpool_shape(s, r, os, &orank));
  TLB_TRY(set_device(c));
  float *d_d, *d_o;
  const int64_t nout = count_of(os, r);
  TLB_TRY(stage_in(c, 0, d, (size_t)count_of(s, r), &d_d));
  TLB_TRY(stage_out(c, 1, (size_t)nout, &d_o));
  TLB_CUDA(tlb::nn_backavgpool(d_d, s, r, d_o, c->stream));
  return fetch(c, out, d_o, (size_t)nout);
}

int tlb_nn_backweights(tlb_ctx* c, const float* d, const int64_t* ds, int dr, const float* in, const int64_t* is,
                       int ir, float* out) {
  // backweights(d_out, in) = conv(in, d_out) (nn.cpp:160)
  return tlb_nn_conv(c, in, is, ir, d, ds, dr, out);
}

int tlb_nn_backbias(tlb_ctx* c, const float* d, int64_t n, float* out) {
  if (!c || !out) return fail(TLB_ERR_ARG, "null argument");
  TLB_TRY(set_device(c));
  float *d_d, *d_o;
  TLB_TRY(stage_in(c, 0, d, (size_t)n, &d_d));
  TLB_TRY(stage_out(c, 1, 1, &d_o));
  TLB_CUDA(tlb::nn_sum_all(d_d, n, d_o, c->stream));
  return fetch(c, out, d_o, 1);
}

int tlb_nn_backin(tlb_ctx* c, const float* d, const int64_t* ds, int dr, const float* k, const int64_t* ks, int kr,
                  const int64_t* is, int ir, float* out) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  int64_t os[8];
  int orank;
  TLB_TRY(tlb_nn_backin_shape(ds, dr, ks, kr, is, ir, os, &orank));
  TLB_TRY(set_device(c));
  float *d_d, *d_k, *d_o;
  const int64_t nout = count_of(is, ir);
  TLB_TRY(stage_in(c, 0, d, (size_t)count_of(ds, dr), &d_d));
  TLB_TRY(stage_in(c, 1, k, (size_t)count_of(ks, kr), &d_k));
  TLB_TRY(stage_out(c, 2, (size_t)nout, &d_o));
  TLB_CUDA(tlb::nn_backin(d_d, ds, d_k, ks, ir, d_o, c->stream));
  return fetch(c, out, d_o, (size_t)nout);
}

// ---- device synthetic corpus (synth.cpp:117-161) ---------------------------------------------------------
static int synth_device(tlb_ctx* c, int64_t n, uint64_t seed, uint8_t* px, float* im, int32_t* lab) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  if (n < 0) return fail(TLB_ERR_ERROR, "make_digits: negative count");
  if (n > 0 && !px && !im && !lab) return TLB_OK;
  TLB_TRY(set_device(c));
  if (n == 0) return TLB_OK;
  TLB_CUDA(c->synth_snaps.ensure(tlb::synth::snapshot_bytes(n)));
  TLB_CUDA(tlb::synth::make_digits(n, seed, static_cast<uint64_t*>(c->synth_snaps.p), px, im, lab, c->stream));
  return TLB_OK;
}

int tlb_synth_make_digits_device(tlb_ctx* c, int64_t n, uint64_t seed, uint8_t* d_pixels, int32_t* d_labels) {
  return synth_device(c, n, seed, d_pixels, nullptr, d_labels);
}

int tlb_synth_make_set_device(tlb_ctx* c, int64_t n, uint64_t seed, float* d_images, int32_t* d_labels) {
  return synth_device(c, n, seed, nullptr, d_images, d_labels);
}

int tlb_pixels_to_images_device(tlb_ctx* c, const uint8_t* d_pixels, int64_t count, float* d_images) {
  if (!c || (count > 0 && (!d_pixels || !d_images))) return fail(TLB_ERR_ARG, "tlb_pixels_to_images_device: null argument");
  if (count < 0) return fail(TLB_ERR_ARG, "tlb_pixels_to_images_device: negative count");
  TLB_TRY(set_device(c));
  TLB_CUDA(tlb::launch_pixels_to_f32(d_pixels, d_images, count, c->stream));
  return TLB_OK;
}

// ---- widened CNN (BASELINE configs[4]) -------------------------------------------------------------------
namespace {
namespace W = tlb::wide;

int wide_ws(tlb_ctx* c, int64_t m, W::StepArgs& a) {
  if (m > c->wide_cap) {
    const size_t f = sizeof(float);
    const size_t sizes[12] = {(size_t)m * W::kC1N * W::kC1W * W::kC1W * f, (size_t)m * W::kC1N * W::kS1Pos * f,
                              (size_t)m * W::kC2N * W::kC2Pos * f,        (size_t)m * W::kS2Len * f,
                              (size_t)m * W::kClasses * f,                (size_t)m * f,
                              (size_t)m * W::kC2N * W::kDzPlane * f,      (size_t)42 * W::kGk2Rows * W::kC2N * f,
                              (size_t)m * W::kC1N * 26 * f,               (size_t)(W::kNParam + 64) * f,
                              (size_t)m * W::kC2N * W::kC2Pos * f,        W::kBImgBytes};
    for (int i = 0; i < 12; ++i) {
      c->wide[i].release();
      TLB_CUDA(c->wide[i].ensure(sizes[i]));
    }
    TLB_CUDA(cudaMemset(c->wide[6].p, 0, sizes[6]));  // dz2's zero border (interior rewritten per group)
    c->wide_cap = m;
  }
  a.c1 = static_cast<float*>(c->wide[0].p);
  a.s1 = static_cast<float*>(c->wide[1].p);
  a.c2 = static_cast<float*>(c->wide[2].p);
  a.s2 = static_cast<float*>(c->wide[3].p);
  a.dz = static_cast<float*>(c->wide[4].p);
  a.loss = static_cast<float*>(c->wide[5].p);
  a.dz2 = static_cast<float*>(c->wide[6].p);
  a.part = static_cast<float*>(c->wide[7].p);
  a.part1 = static_cast<float*>(c->wide[8].p);
  a.grad = static_cast<float*>(c->wide[9].p);
  a.dz2t = static_cast<float*>(c->wide[10].p);
  a.bimg = static_cast<float*>(c->wide[11].p);
  return TLB_OK;
}

int check_engine(int engine) {
  if (engine != TLB_WIDE_FP32 && engine != TLB_WIDE_TC)
    return fail(TLB_ERR_ARG, "unknown GEMM engine " + std::to_string(engine));
  return TLB_OK;
}

int wide_enqueue(tlb_ctx* c, const float* d_images, const int32_t* d_labels, int64_t n, float* d_params, float rate,
                 int32_t epoch_begin, int32_t epochs, int64_t batch, double* d_epoch_loss, int engine) {
  const int64_t spe = (n + batch - 1) / batch;
  W::StepArgs a{};
  TLB_TRY(wide_ws(c, std::min(batch, n), a));
  a.params = d_params;
  a.rate = rate;
  a.tensor = engine == TLB_WIDE_TC;
  a.n_total = (double)n;
  for (int32_t e = epoch_begin; e < epoch_begin + epochs; ++e)
    for (int64_t s = 0; s < spe; ++s) {
      const int64_t lo = s * batch;
      a.m = std::min(batch, n - lo);
      a.images = d_images + lo * W::kImgW * W::kImgW;
      a.labels = d_labels + lo;
      a.epoch_loss = d_epoch_loss ? d_epoch_loss + e : nullptr;
      a.first = s == 0;
      a.last = s == spe - 1;
      TLB_CUDA(W::step(a, c->stream));
      c->wide_last = a;
    }
  return TLB_OK;
}
}  // namespace

int tlb_wide_train_device(tlb_ctx* c, const float* d_images, const int32_t* d_labels, int64_t n, float* d_params,
                          float rate, int32_t epoch_begin, int32_t epochs, int64_t batch, double* d_epoch_loss,
                          int engine) {
  if (!c || !d_params || !d_images || !d_labels) return fail(TLB_ERR_ARG, "tlb_wide_train_device: null argument");
  TLB_TRY(check_train_args(n, epochs, rate, batch));
  TLB_TRY(check_engine(engine));
  TLB_TRY(set_device(c));
  return wide_enqueue(c, d_images, d_labels, n, d_params, rate, epoch_begin, epochs, batch, d_epoch_loss, engine);
}

int tlb_wide_train(tlb_ctx* c, const float* images, const int32_t* labels, int64_t n, float* params, float rate,
                   int32_t epochs, int64_t batch, double* epoch_loss, int engine) {
  if (!c || !params) return fail(TLB_ERR_ARG, "tlb_wide_train: null argument");
  TLB_TRY(check_train_args(n, epochs, rate, batch));
  TLB_TRY(check_engine(engine));
  if (!images || !labels) return fail(TLB_ERR_ARG, "tlb_wide_train: null dataset");
  for (int64_t i = 0; i < n; ++i)
    if (labels[i] < 0 || labels[i] > 9)
      return fail(TLB_ERR_VALUE, "one_hot: label " + std::to_string(labels[i]) + " out of range 0..9");
  TLB_TRY(set_device(c));
  if (epochs == 0) return TLB_OK;
  float *d_img, *d_p;
  int32_t* d_lab;
  double* d_loss;
  TLB_TRY(stage_in(c, 0, images, (size_t)n * W::kImgW * W::kImgW, &d_img));
  TLB_TRY(stage_in(c, 1, labels, (size_t)n, &d_lab));
  TLB_TRY(stage_in(c, 2, params, (size_t)W::kNParam, &d_p));
  TLB_TRY(stage_out(c, 3, (size_t)epochs, &d_loss));
  TLB_TRY(wide_enqueue(c, d_img, d_lab, n, d_p, rate, 0, epochs, batch, d_loss, engine));
  TLB_CUDA(cudaMemcpyAsync(params, d_p, W::kNParam * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  if (epoch_loss) TLB_CUDA(cudaMemcpyAsync(epoch_loss, d_loss, epochs * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  TLB_CUDA(cudaStreamSynchronize(c->stream));
  return TLB_OK;
}

int tlb_wide_forward(tlb_ctx* c, const float* images, int64_t n, const float* params, float* yhat, int engine) {
  if (!c || !params || !yhat || (n > 0 && !images)) return fail(TLB_ERR_ARG, "tlb_wide_forward: null argument");
  if (n < 0) return fail(TLB_ERR_ARG, "negative count");
  TLB_TRY(check_engine(engine));
  if (n == 0) return TLB_OK;
  TLB_TRY(set_device(c));
  float *d_img, *d_p, *d_y;
  TLB_TRY(stage_in(c, 0, images, (size_t)n * W::kImgW * W::kImgW, &d_img));
  TLB_TRY(stage_in(c, 2, params, (size_t)W::kNParam, &d_p));
  TLB_TRY(stage_out(c, 3, (size_t)n * W::kClasses, &d_y));
  const int64_t chunk = 256;
  W::StepArgs a{};
  TLB_TRY(wide_ws(c, std::min(chunk, n), a));
  a.params = d_p;
  a.tensor = engine == TLB_WIDE_TC;
  for (int64_t lo = 0; lo < n; lo += chunk) {
    a.m = std::min(chunk, n - lo);
    a.images = d_img + lo * W::kImgW * W::kImgW;
    TLB_CUDA(W::forward(a, d_y + lo * W::kClasses, c->stream));
  }
  return fetch(c, yhat, d_y, (size_t)n * W::kClasses);
}

int tlb_wide_gemm_device(tlb_ctx* c, int which, int engine) {
  if (!c) return fail(TLB_ERR_ARG, "null context");
  TLB_TRY(check_engine(engine));
  if (which < 0 || which > 2) return fail(TLB_ERR_ARG, "tlb_wide_gemm_device: which must be 0, 1 or 2");
  if (c->wide_last.m <= 0) return fail(TLB_ERR_ERROR, "tlb_wide_gemm_device: no widened group trained yet");
  TLB_TRY(set_device(c));
  TLB_CUDA(W::gemm_only(which, engine == TLB_WIDE_TC, c->wide_last, c->stream));
  return TLB_OK;
}

int tlb_expf_range(tlb_ctx* c, uint32_t start_bits, int64_t n, float* out) {
  if (!c || !out) return fail(TLB_ERR_ARG, "null argument");
  TLB_TRY(set_device(c));
  float* d_o;
  TLB_TRY(stage_out(c, 0, (size_t)n, &d_o));
  TLB_CUDA(tlb::nn_expf_range(start_bits, n, d_o, c->stream));
  return fetch(c, out, d_o, (size_t)n);
}

}  // extern "C"
