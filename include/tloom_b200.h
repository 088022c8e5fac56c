/*
 * tloom_b200.h -- C ABI of the B200-native tensorloom hot path (libtloom_b200.so).
 *
 * This is the drop-in boundary for the reference's training path.  The reference
 * exposes it as the C++ headers proj/include/tloom/{nn,network,mnist}.hpp; our C++ mirror of those
 * headers (include/tloom/ *.hpp, same names and exceptions) and any FFI binding (ctypes, cgo, JNI)
 * sit on top of these entry points.  Plain pointers and sizes only; no torch or C++ types.
 *
 * Conventions
 *  - Every call returns TLB_OK (0) or an error code; tlb_last_error() returns the message of the
 *    calling thread's last failure.  Codes map 1:1 onto the reference's exception taxonomy
 *    (proj/include/tloom/errors.hpp:9-31) so the C++ layer rethrows the same types and messages.
 *  - "Host" entry points take host buffers, stage them to HBM, run, copy results back and return
 *    after device completion (the reference's synchronous semantics).  "_device" entry points take
 *    device pointers and enqueue on the context stream without synchronising.
 *  - Parameters / gradients are flat fp32 in write_flat order k1,b1,k2,b2,fc,b
 *    (proj/src/network.cpp:186-193), TLB_NPARAM = 3898 floats.  Device-side parameter buffers are
 *    padded to TLB_PSTRIDE = 3904 floats.
 *  - Images are [n][28][28] fp32 in [0,1] (mnist::MnistSet, proj/include/tloom/mnist.hpp:14-19),
 *    labels int32 0..9.
 *  - Mode TLB_MODE_EXACT (default) reproduces the reference bit for bit (same per-element summation
 *    order, no FMA, glibc expf restatement, example-order batch reduction).  TLB_MODE_FAST uses FFMA
 *    and per-CTA partial sums (deterministic; within 1e-4 relative of the reference).
 */
#ifndef TLOOM_B200_H
#define TLOOM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLB_OK 0
#define TLB_ERR_ERROR 1  /* tloom::Error       */
#define TLB_ERR_SHAPE 2  /* tloom::ShapeError  */
#define TLB_ERR_BOUNDS 3 /* tloom::BoundsError */
#define TLB_ERR_FORMAT 4 /* tloom::FormatError */
#define TLB_ERR_VALUE 5  /* tloom::ValueError  */
#define TLB_ERR_CUDA 10
#define TLB_ERR_NCCL 11
#define TLB_ERR_ARG 12

#define TLB_MODE_EXACT 0
#define TLB_MODE_FAST 1

#define TLB_NPARAM 3898
#define TLB_PSTRIDE 3904
#define TLB_NACT 5290 /* c1[6,24,24] s1[6,12,12] c2[12,1,8,8] s2[12,1,4,4] out[10,1,1,1,1] */
#define TLB_CELL 3899 /* gradient row + loss, network.cpp:218 */

typedef struct tlb_ctx tlb_ctx;
/* on_epoch(epoch, mean_loss) of net::train (network.hpp:79-80, network.cpp:246-248). */
typedef void (*tlb_epoch_cb)(int epoch, double mean_loss, void* user);

const char* tlb_last_error(void);
const char* tlb_version(void);

/* ---- context: device, stream, mode, workspaces ------------------------------------------------ */
int tlb_ctx_create(int device, tlb_ctx** out);
int tlb_ctx_destroy(tlb_ctx* ctx);
/* A context over several local GPUs in one process: tlb_train / tlb_train_u8 /
 * tlb_train_idx split every SGD group over the devices with the reference's static_chunk rule
 * (runtime.cpp:138-145) -- each device keeps its shard of the data -- and reduce the gradient over all of
 * them at every step through peer memory (one persistent kernel per device).  EXACT mode: bit-identical to
 * one device and to the reference, for any device count (as the reference is for any worker count); fast
 * mode: deterministic for a given count, within the 1e-4 tolerance.  A device may be listed more than once
 * (the kernels then share it).  Other entry points run on devices[0]. */
int tlb_ctx_create_multi(const int* devices, int n_devices, tlb_ctx** out);
int tlb_ctx_device_count(const tlb_ctx* ctx, int* n_devices);
/* Enqueue on a caller-owned cudaStream_t (NULL = the legacy default stream).  A new context uses
 * its own non-blocking stream. */
int tlb_ctx_set_stream(tlb_ctx* ctx, void* cuda_stream);
int tlb_ctx_set_mode(tlb_ctx* ctx, int mode);
int tlb_ctx_get_mode(const tlb_ctx* ctx, int* mode);
/* CTAs of the persistent train kernel (0 = auto); clamped to the co-resident maximum. */
int tlb_ctx_set_grid(tlb_ctx* ctx, int ctas);
/* Profiling hook: device buffer of [steps][16] uint64 clock64 stamps written by CTA 0 of the
 * persistent train kernel at each stage boundary (NULL disables; see bench.py --trace). */
int tlb_ctx_set_trace(tlb_ctx* ctx, void* d_trace);
/* Fast mode, groups of <= 8 x (co-resident clusters) examples: 1 (default) runs the clustered train
 * kernel (DSMEM gradient pre-reduction, one grid barrier per step); 0 forces the flat kernel. */
int tlb_ctx_set_cluster(tlb_ctx* ctx, int enable);
/* Fast mode, groups the clustered kernel does not take: -1 (default) runs the batched train kernel (NI
 * images per CTA round, batch_train.cu) from 4 x SM-count examples per group (env TLB_BATCHED=0/1
 * overrides), 0 the one-image-per-CTA flat kernel, 1 the batched kernel for every such group. */
int tlb_ctx_set_batched(tlb_ctx* ctx, int mode);
/* Data layout of the images/labels given to tlb_train_shard_device / tlb_train_dp_device: 0 (default) = the
 * whole dataset (every rank holds every group); > 0 = only this rank's shards, the shard of SGD group g
 * (static_chunk of the group, runtime.cpp:138-145) starting at example g * local_stride -- each rank then
 * uploads and keeps 1/world of the corpus. */
int tlb_ctx_set_shard_layout(tlb_ctx* ctx, int64_t local_stride);
/* CTA size of the flat train / forward kernels: 0 = automatic (default: 256 = two independent CTAs per SM
 * whose barrier stalls overlap once a launch has more than one item per SM, else 512), or forced 256 / 512.
 * Env TLB_FAST_THREADS. */
int tlb_ctx_set_threads(tlb_ctx* ctx, int threads);
int tlb_ctx_info(const tlb_ctx* ctx, int* sm_count, int* train_ctas_per_sm, int* eval_ctas_per_sm,
                 int64_t* smem_bytes_per_cta);
/* Waits for the context stream and reports device-side failures of earlier device-API launches (a bounded
 * cross-CTA wait that gave up: TLB_ERR_CUDA; a fast-mode fixed-point gradient overflow: TLB_ERR_VALUE),
 * clearing them.  tlb_train performs the same check before it returns. */
int tlb_synchronize(tlb_ctx* ctx);

/* ---- host-side helpers of the reference API --------------------------------------------------- */
/* net::init_params (network.cpp:56-79). */
int tlb_init_params(uint64_t seed, float* params_out /* TLB_NPARAM */);
/* synth::make_digits / make_set (synth.cpp:117-161): n 28x28 glyph images + labels. */
int tlb_synth_make_digits(int64_t n, uint64_t seed, uint8_t* pixels_out, int32_t* labels_out);
/* synth::make_digits / synth::make_set (synth.cpp:117-161) generated on the device into device buffers,
 * byte-identical to the host versions for every (n, seed): the mt19937_64 stream is rebuilt by a serial
 * twist chain that snapshots the state per image segment, then all segments synthesise in parallel.
 * Either output may be NULL.  Enqueued on the context stream. */
int tlb_synth_make_digits_device(tlb_ctx* ctx, int64_t n, uint64_t seed, uint8_t* d_pixels, int32_t* d_labels);
int tlb_synth_make_set_device(tlb_ctx* ctx, int64_t n, uint64_t seed, float* d_images, int32_t* d_labels);
int tlb_synth_make_set(int64_t n, uint64_t seed, float* images_out, int32_t* labels_out);
/* Device half of the byte ingestion: d_images[i] = d_pixels[i] / 255.0f for `count` bytes (mnist.cpp:57),
 * on the context stream. */
int tlb_pixels_to_images_device(tlb_ctx* ctx, const uint8_t* d_pixels, int64_t count, float* d_images);
/* mnist::make_set invariants (mnist.cpp:126-154): pixels in [0,1], labels in 0..9 (ValueError). */
int tlb_validate_set(const float* images, const int32_t* labels, int64_t n);

/* ---- host memory -------------------------------------------------------------------------------- */
/* Page-lock (and unlock) a caller-owned host range for the direct-DMA ingestion path of tlb_train /
 * tlb_evaluate (no reference counterpart: the C++ mirror keeps its last training set registered across
 * net::train calls, tloom/network.hpp).  Returns TLB_ERR_CUDA if the range cannot be registered (e.g. it
 * overlaps a registered range); the call then simply takes the pageable path. */
int tlb_host_register(tlb_ctx* ctx, const void* ptr, size_t bytes);
int tlb_host_unregister(tlb_ctx* ctx, const void* ptr);

/* ---- network, host buffers (replaces tloom::net, network.hpp:59-86) --------------------------- */
/* net::train (network.cpp:209-251): params updated in place; epoch_loss[epochs] = mean losses.
 * Errors as the reference: n==0, epochs<0, !(rate>0) -> TLB_ERR_ERROR; batch<1 -> TLB_ERR_ERROR. */
int tlb_train(tlb_ctx* ctx, const float* images, const int32_t* labels, int64_t n, float* params,
              float rate, int32_t epochs, int64_t batch, double* epoch_loss, tlb_epoch_cb on_epoch,
              void* user);
/* net::forward (network.cpp:81-95) for n images: yhat [n][10]; acts [n][TLB_NACT] (nullable). */
/* net::train on the raw pixel bytes the fp32 images are made from (the IDX payload, mnist.cpp:41-61, or
 * synth::make_digits, synth.cpp:117-153): the bytes cross the host link (1/4 of the fp32 volume) and are
 * converted on the device as pixel / 255.0f -- bit-identical to mnist::load_images / synth::make_set, so the
 * result equals tlb_train on the converted images bit for bit. */
int tlb_train_u8(tlb_ctx* ctx, const uint8_t* pixels /* n x 784 */, const int32_t* labels, int64_t n, float* params,
                 float rate, int32_t epochs, int64_t batch, double* epoch_loss_out, tlb_epoch_cb on_epoch, void* user);
/* net::train straight from the bytes of an IDX image file and an IDX label file (mnist::load_images /
 * load_labels + make_set): headers validated with the reference's FormatError / ValueError messages, the
 * image payload ingested as bytes (tlb_train_u8). */
int tlb_train_idx(tlb_ctx* ctx, const uint8_t* image_file, size_t image_bytes, const uint8_t* label_file,
                  size_t label_bytes, float* params, float rate, int32_t epochs, int64_t batch,
                  double* epoch_loss_out, tlb_epoch_cb on_epoch, void* user);
/* IDX header check (no device): kind 0 = images (magic 2051: count, rows, cols), 1 = labels (magic 2049:
 * count); dims_out[3] (unused dims 1), *payload_offset = first payload byte.  TLB_ERR_FORMAT with the
 * reference's message on a bad magic, truncated header/payload or trailing bytes (mnist.cpp:14-61). */
int tlb_idx_parse(const uint8_t* bytes, size_t len, int kind, int64_t* dims_out, size_t* payload_offset);
int tlb_forward(tlb_ctx* ctx, const float* images, int64_t n, const float* params, float* yhat,
                float* acts);
/* forward + net::backward + net::loss per example: cells [n][TLB_CELL] (3898 grads + loss).
 * Targets: dense [n][10] (nullable) else one_hot(labels). */
int tlb_forward_backward(tlb_ctx* ctx, const float* images, const int32_t* labels,
                         const float* targets, int64_t n, const float* params, float* cells,
                         float* acts);
/* net::backward (network.cpp:145-169) from cached activations acts [n][TLB_NACT] (as returned by
 * tlb_forward) and dense targets [n][10]: grads [n][TLB_NPARAM]. */
int tlb_backward(tlb_ctx* ctx, const float* images, const float* acts, const float* targets, int64_t n,
                 const float* params, float* grads);
/* net::loss (network.cpp:97-109) for n rows: out[r] = 0.5f * sum_i (y[r][i] - yhat[r][i])^2. */
int tlb_loss(tlb_ctx* ctx, const float* yhat, const float* y, int64_t n, float* out);
/* net::predict / net::evaluate (network.cpp:253-280): pred [n] (nullable), correct count. */
int tlb_evaluate(tlb_ctx* ctx, const float* images, const int32_t* labels, int64_t n,
                 const float* params, int32_t* pred, int64_t* correct);
/* net::sgd_step (network.cpp:171-180): out = p - rate * (g / (float)batch). */
int tlb_sgd_step(tlb_ctx* ctx, const float* params, const float* grads, float rate, int64_t batch,
                 float* out);

/* ---- network, device-resident buffers (async on the context stream) --------------------------- */
/* Runs epochs [epoch_begin, epoch_begin+epochs) of net::train in one persistent kernel launch.
 * d_params: [TLB_PSTRIDE]; d_epoch_loss: indexed by absolute epoch. */
int tlb_train_device(tlb_ctx* ctx, const float* d_images, const int32_t* d_labels, int64_t n,
                     float* d_params, float rate, int32_t epoch_begin, int32_t epochs, int64_t batch,
                     double* d_epoch_loss);
/* One data-parallel shard of one SGD group: group `group` (examples [group*batch, ...) of the
 * dataset, network.cpp:225-234) restricted to its examples [shard_lo, shard_hi).
 * d_grad_sum[0..3897] = fixed-order sum of the shard's gradient rows; d_loss_sum[0] = fp64 sum of
 * its per-example losses.  Feed both to an allreduce, then tlb_apply_sgd_device. */
int tlb_train_shard_device(tlb_ctx* ctx, const float* d_images, const int32_t* d_labels, int64_t n,
                           int64_t batch, int64_t group, int64_t shard_lo, int64_t shard_hi,
                           const float* d_params, float* d_grad_sum, double* d_loss_sum);
/* sgd_step on device buffers (post-allreduce): d_params -= rate * (d_grad_sum / m). */
/* Fused data parallelism over NVLink (one call per rank, no NCCL on the data path): rank `rank` of
 * `world` (<= 8) trains static_chunk(group, world, rank) of every global group of `batch` examples in ONE
 * persistent clustered launch; the 2^-40 fixed-point gradient accumulator of slice s (of 8) and its
 * arrival counter live in rank (s % world)'s workspace and every rank adds into it over peer memory
 * (system-scope `red`), then applies the identical sgd_step with the global group size.  peer_ws holds
 * every rank's workspace pointer (tlb_dp_workspace_bytes each, zeroed before the first call, e.g. a
 * torch symmetric-memory buffer); seq_base = SGD steps run on these workspaces since they were zeroed.
 * A peer wait longer than timeout_s sets the watchdog word (u32 at byte offset
 * tlb_dp_workspace_bytes() - 32 of this rank's workspace) and ends the kernel instead of hanging. */
size_t tlb_dp_workspace_bytes(void);
int tlb_train_dp_device(tlb_ctx* ctx, const float* d_images, const int32_t* d_labels, int64_t n, float* d_params,
                        float rate, int32_t epoch_begin, int32_t epochs, int64_t batch, double* d_epoch_loss,
                        int world, int rank, void* const* peer_ws, uint64_t seq_base, double timeout_s);
int tlb_apply_sgd_device(tlb_ctx* ctx, float* d_params, const float* d_grad_sum, float rate,
                         int64_t m);
int tlb_evaluate_device(tlb_ctx* ctx, const float* d_images, const int32_t* d_labels, int64_t n,
                        const float* d_params, int32_t* d_pred, unsigned long long* d_correct);

/* ---- generic layer ops, host buffers (replaces tloom::nn, nn.hpp:12-58) ------------------------
 * Shapes are int64 extent arrays, rank <= 8, row-major.  Shape preconditions are checked with the
 * reference's ShapeError messages before any data is touched. */
int tlb_nn_conv(tlb_ctx* ctx, const float* in, const int64_t* in_shape, int in_rank, const float* k,
                const int64_t* k_shape, int k_rank, float* out);
int tlb_nn_mconv(tlb_ctx* ctx, const float* in, const int64_t* in_shape, int in_rank, const float* k,
                 const int64_t* k_shape, int k_rank, const float* b, const int64_t* b_shape,
                 int b_rank, float* out);
int tlb_nn_sigmoid(tlb_ctx* ctx, const float* x, int64_t n, float* out);
int tlb_nn_backsigmoid(tlb_ctx* ctx, const float* d, const float* o, int64_t n, float* out);
int tlb_nn_avgpool(tlb_ctx* ctx, const float* in, const int64_t* shape, int rank, float* out);
int tlb_nn_backavgpool(tlb_ctx* ctx, const float* d, const int64_t* shape, int rank, float* out);
int tlb_nn_backweights(tlb_ctx* ctx, const float* d, const int64_t* d_shape, int d_rank,
                       const float* in, const int64_t* in_shape, int in_rank, float* out);
int tlb_nn_backbias(tlb_ctx* ctx, const float* d, int64_t n, float* out);
int tlb_nn_backin(tlb_ctx* ctx, const float* d, const int64_t* d_shape, int d_rank, const float* k,
                  const int64_t* k_shape, int k_rank, const int64_t* in_shape, int in_rank,
                  float* out);
/* Result-shape functions (nn.hpp:12-32); out_shape must hold 8 extents. */
int tlb_nn_conv_shape(const int64_t* in_shape, int in_rank, const int64_t* k_shape, int k_rank,
                      int64_t* out_shape, int* out_rank);
int tlb_nn_mconv_shape(const int64_t* in_shape, int in_rank, const int64_t* k_shape, int k_rank,
                       const int64_t* b_shape, int b_rank, int64_t* out_shape, int* out_rank);
int tlb_nn_avgpool_shape(const int64_t* shape, int rank, int64_t* out_shape, int* out_rank);
int tlb_nn_backavgpool_shape(const int64_t* shape, int rank, int64_t* out_shape, int* out_rank);
int tlb_nn_backin_shape(const int64_t* d_shape, int d_rank, const int64_t* k_shape, int k_rank,
                        const int64_t* in_shape, int in_rank, int64_t* out_shape, int* out_rank);

/* ---- Widened CNN (BASELINE.json configs[4]): conv1 32@5x5 -> sigmoid -> avgpool -> conv2 64@32x5x5 ->
 * sigmoid -> avgpool -> FC 10 from [64,1,13,13], 64x64 inputs, 160,266 parameters in write_flat order
 * (k1 [32,5,5], b1 [32], k2 [64,32,5,5], b2 [64], fc [10,64,1,13,13], b [10]).  Same group semantics
 * as tlb_train (network.cpp:209-251: per-example gradients summed over the group, sgd_step) built from
 * the shape-polymorphic nn:: operators (nn.cpp:96-217); the reference has no widened net::train, the
 * oracle is the composition of its operators (oracle/widened.py).  engine selects the GEMM engine of
 * the three conv2 contractions: TLB_WIDE_FP32 (register-tiled FFMA on the CUDA cores) or
 * TLB_WIDE_TC (tcgen05 tensor cores, 3xTF32 split = fp32-level accuracy).  Deterministic, within the
 * 1e-4 relative tolerance of the reference composition (not bitwise). */
#define TLB_WIDE_NPARAM 160266
#define TLB_WIDE_IMG 4096 /* 64 x 64 */
#define TLB_WIDE_FP32 0
#define TLB_WIDE_TC 1
/* init_params rule (network.cpp:56-79) with the widened fans: k1 (25, 3600), k2 (800, 676), fc (10816, 1). */
int tlb_wide_init_params(uint64_t seed, float* params_out);
/* n synthetic 64x64 inputs: synth::make_digits(n, seed) glyphs centred at offset 18, / 255.0f. */
int tlb_wide_make_set(int64_t n, uint64_t seed, float* images_out, int32_t* labels_out);
int tlb_wide_train(tlb_ctx* ctx, const float* images, const int32_t* labels, int64_t n, float* params, float rate,
                   int32_t epochs, int64_t batch, double* epoch_loss, int engine);
int tlb_wide_train_device(tlb_ctx* ctx, const float* d_images, const int32_t* d_labels, int64_t n, float* d_params,
                          float rate, int32_t epoch_begin, int32_t epochs, int64_t batch, double* d_epoch_loss,
                          int engine);
/* Forward only (inference): yhat [n][10]. */
int tlb_wide_forward(tlb_ctx* ctx, const float* images, int64_t n, const float* params, float* yhat, int engine);
/* Benchmark hook: re-run one conv2 contraction (0 forward, 1 weight gradient, 2 backin) of the last
 * trained group on the context's workspaces with the given engine. */
int tlb_wide_gemm_device(tlb_ctx* ctx, int which, int engine);

/* Test hook: device glibc-expf restatement over float bit patterns [start, start+n). */
int tlb_expf_range(tlb_ctx* ctx, uint32_t start_bits, int64_t n, float* out);

#ifdef __cplusplus
}
#endif
#endif /* TLOOM_B200_H */
