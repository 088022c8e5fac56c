// tlb_launch.h -- internal kernel argument blocks and launchers (not part of the public C ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace tlb {

struct TrainArgs {
  const float* images;    // [n][784] fp32, device
  const int32_t* labels;  // [n]
  int64_t n;
  int64_t batch;
  float rate;
  int64_t step_begin, step_end;  // absolute step range (epoch * steps_per_epoch + group)
  int64_t steps_per_epoch;
  float* params;        // [3904] in/out
  float* work;          // EXACT: [min(batch,n)][3904] example rows; fast: [grid][3904] CTA partials
  float* losses;        // EXACT: [min(batch,n)] per-example loss of the current group
  double* loss_part;    // fast: [grid] per-CTA fp64 loss partials
  double* epoch_loss;   // [epochs] running fp64 sum -> mean (network.cpp:239, 245)
  unsigned int* barrier;
  // Data-parallel shard mode (grad_out != nullptr): only examples [shard_lo, shard_hi) of each
  // group are processed and, instead of the SGD update, their fixed-order gradient sum goes to
  // grad_out[3898] and the fp64 loss sum to loss_out[0] (for the NCCL allreduce).
  int64_t shard_lo, shard_hi;
  float* grad_out;
  double* loss_out;
  unsigned long long* trace;  // optional [steps][16] clock64 stamps of CTA 0 (tlb_ctx_set_trace)
  // Overlapped ingestion (tlb_train on host buffers): images arrive in chunks on a copy stream;
  // ready[k] >= ready_token once chunk k is resident.  chunk > 0: chunk k = images [k*chunk, (k+1)*chunk);
  // chunk == 0: geometric chunks of whole SGD groups -- groups 0 and 1, then each [2^e, 2^(e+1)) in two
  // halves (chunk 2e, 2e + 1) -- 14 copies for a 100-group epoch; chunk k lands before group 1.5x its
  // start is reached whenever H2D >= 1.5 x (group bytes / group time), ~29 GB/s at batch 100.
  // Steps < ready_step_end poll the flag before the image's TMA load; nullptr = every image resident.
  const unsigned int* ready;
  unsigned int ready_token;
  int64_t chunk;  // (chunk < 0: ramp of -chunk = C groups, a power of two: chunks of groups 0 | 1 | 2-3 |
                  //  4-7 | ... up to C, then C groups each -- the first step waits for one group only)
  int64_t ready_step_end;
  int64_t ready_g0;  // group (within its epoch) of step_begin
  int chunk_shift;   // ramp: log2 C
  unsigned int* ready_err;  // [3] diagnostic words: set when a ready flag never arrives (then the kernel
                            // proceeds and the host call fails instead of hanging)
  // Fused data parallelism over NVLink peer memory (clustered kernel, dp_world > 0): rank dp_rank of
  // dp_world trains static_chunk(group, dp_world, dp_rank) of every global group; slice s of the
  // fixed-point gradient accumulator and its arrival counter live on rank s % dp_world, the loss
  // accumulator on rank 0 (symmetric buffers, peer pointers).  seq_base = steps run on these buffers
  // since they were zeroed (triple-buffer phase and counter targets continue across launches).
  int dp_world, dp_rank;
  unsigned long long* slice_acc[16];  // [3][3904] u64 accumulator holding slice s (local or peer)
  unsigned int* slice_cnt[16];        // arrival counter of slice s (cluster_size() entries used)
  unsigned long long* loss_acc;      // [3] u64 loss accumulators
  uint64_t seq_base;
  unsigned int* dp_error;            // set when a peer wait times out (the kernel then exits); single GPU:
                                     // the abort word of the guarded cluster waits (mbar_wait_cluster_guarded)
  long long dp_timeout_cycles;       // bound of every cross-CTA / cross-GPU wait
  unsigned int* fix_err;             // set when a cluster's gradient sum left the fixed-point range (clamped)
  // Shard layout (DP shard / fused DP modes, tlb_ctx_set_shard_layout): 0 = `images`/`labels` hold the whole
  // dataset (example e of group g at g * batch + e); > 0 = they hold only this rank's shards, the shard of
  // group g starting at g * local_stride (the local example e of it at g * local_stride + e).
  int64_t local_stride;
  // Byte ingestion (tlb_train_u8 / tlb_train_idx): during the steps < ready_step_end the images arrive as
  // pixel bytes in `pixels` (chunked, ready flags as above); the CTA that trains an image loads its 784
  // bytes, converts them in shared memory (pixel / 255.0f, mnist.cpp:57) and writes the fp32 image back to
  // images_wb (== images) for the later epochs of the launch.  nullptr = fp32 images throughout.
  const uint8_t* pixels;
  float* images_wb;
  // In-process multi-GPU (tlb_ctx_create_multi): md_n > 1 devices run the flat train kernel at once, device
  // dp_rank on static_chunk(m, md_n, dp_rank) of every group (dp_world = md_n, shard layout).  Phase 2 spans
  // every device: global CTA (dp_rank * grid + cta) reduces its parameter slice over ALL devices' rows in
  // example order (EXACT: bit-identical to one device) or (device, CTA) order (fast), reading peers' rows
  // through their pointers, and writes the update into every device's parameter copy; the grid barrier
  // counts every CTA of every device on md_bar (device 0).  md_n == 0: single device.
  int md_n;
  float* md_work[8];
  float* md_losses[8];
  double* md_loss_part[8];
  float* md_params[8];
  double* md_epoch_loss[8];
  unsigned int* md_bar;
  // Batched kernel with two CTAs per SM (batch_train.cu): the CTA that reaches the SM's slot counter first
  // is scheduled ahead of its partner; it trains this share of the SM's examples (set at launch).
  float pair_share;
};

struct CellArgs {
  const float* images;
  const int32_t* labels;  // one-hot targets from labels (mnist::one_hot) when targets == nullptr
  const float* targets;   // [n][10] dense targets or nullptr
  int64_t n;
  const float* params;
  float* cells;   // [n][3904] gradient rows (nullptr: forward only)
  float* losses;  // [n] or nullptr
  float* acts;    // [n][5290] c1,s1,c2,s2,out or nullptr
  const float* acts_in;  // backward from cached activations (net::backward) instead of a forward pass
  float* yhat;    // [n][10] or nullptr
};

struct EvalArgs {
  const float* images;
  const int32_t* labels;  // nullable
  int64_t n;
  const float* params;
  int32_t* pred;   // nullable
  float* yhat;     // nullable
  unsigned long long* correct;  // nullable
  // Batched inference: rounds are claimed from this counter (zeroed at launch) so co-resident CTAs share
  // the work however the schedulers favour them; nullptr = static per-CTA chunks.
  unsigned long long* claim;
};

size_t smem_bytes();
int threads_per_cta();
cudaError_t train_occupancy(bool exact, int threads, int* occ);
cudaError_t eval_occupancy(bool exact, int threads, int* occ);
cudaError_t launch_train(bool exact, const TrainArgs& a, int grid, int threads, cudaStream_t st);
cudaError_t cluster_train_capacity(int* max_clusters);
int cluster_size();
size_t cluster_work_bytes();
size_t dp_workspace_bytes();
size_t dp_counter_offset();
cudaError_t launch_train_cluster(const TrainArgs& a, int clusters, cudaStream_t st);
cudaError_t launch_cells(bool exact, const CellArgs& a, int grid, cudaStream_t st);
cudaError_t launch_eval(bool exact, const EvalArgs& a, int grid, int threads, cudaStream_t st);
// Fast-mode batched train kernel for large groups (batch_train.cu): NI images per CTA round.
int batch_train_grid(int sm_count, int64_t m_max);
// The batched kernel's work buffer: [grid][3904] partial rows + this many bytes (SM-pair mapping scratch).
constexpr size_t kBatchWorkExtraBytes = 8192;
constexpr int kPairMaxGrid = 1024;
cudaError_t launch_train_batch(const TrainArgs& a, int sm_count, int64_t m_max, cudaStream_t st);
// Fast-mode batched inference (infer_kernels.cu): forward + argmax + correct count over n images.
cudaError_t launch_infer(const EvalArgs& a, int sm_count, cudaStream_t st);
cudaError_t launch_sgd(const float* params, const float* grad, float rate, int64_t m, float* out, int n,
                       cudaStream_t st);

// Generic rank-polymorphic nn ops (nn_ops.cu).  Shapes are host arrays (rank <= 8).
cudaError_t nn_conv(const float* in, const int64_t* is, const float* k, const int64_t* ks, int r,
                    const float* bias, int64_t nk, float* out, cudaStream_t st);
cudaError_t nn_sigmoid(const float* x, int64_t n, float* out, cudaStream_t st);
cudaError_t nn_backsigmoid(const float* d, const float* o, int64_t n, float* out, cudaStream_t st);
cudaError_t nn_avgpool(const float* in, const int64_t* s, int r, float* out, cudaStream_t st);
cudaError_t nn_backavgpool(const float* d, const int64_t* s, int r, float* out, cudaStream_t st);
cudaError_t nn_backin(const float* d, const int64_t* ds, const float* k, const int64_t* ks, int r, float* out,
                      cudaStream_t st);
cudaError_t nn_loss(const float* yhat, const float* y, int64_t n, float* out, cudaStream_t st);
cudaError_t nn_sum_all(const float* x, int64_t n, float* out, cudaStream_t st);
cudaError_t nn_expf(const float* x, int64_t n, float* out, cudaStream_t st);
cudaError_t nn_expf_range(uint32_t start_bits, int64_t n, float* out, cudaStream_t st);

// Pixel bytes -> fp32 images, pixel / 255.0f (mnist.cpp:57): the device half of the byte ingestion.
cudaError_t launch_pixels_to_f32(const uint8_t* src, float* dst, int64_t count, cudaStream_t st);

// Device synthetic corpus (synth_device.cu)
namespace synth {
size_t snapshot_bytes(int64_t n);
cudaError_t make_digits(int64_t n, uint64_t seed, uint64_t* snaps, uint8_t* pixels, float* images, int32_t* labels,
                        cudaStream_t st);
}  // namespace synth

}  // namespace tlb
