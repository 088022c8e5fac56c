/*
 * tloom_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference (`tensorloom`, /root/reference/proj) hot path:
 * the Zhang MNIST CNN forward / backward / loss / batch reduction / SGD step
 * (proj/src/network.cpp:81-251, kernels proj/src/nn.cpp:96-217), the generic
 * rank-polymorphic nn ops (nn.cpp:37-217), init_params (network.cpp:56-79), the
 * synthetic digit corpus (proj/src/synth.cpp:117-161) and glibc 2.39 `expf`.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library, and only as the checker -- never as the product path.
 *
 * Parity pinning: every function here is checked against the reference library
 * itself (oracle/_ref, built from /root/reference sources by oracle/Makefile) and
 * against golden vectors dumped from it (tests/golden/, see
 * tests/golden/make_golden.py).  Arithmetic is plain IEEE fp32 with no FMA
 * contraction (built with -ffp-contract=off, no -march), which is exactly how the
 * reference's Release build computes (CMakeLists.txt:8-24: -O3, no -march).
 */
#ifndef TLOOM_ORACLE_H
#define TLOOM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Flat parameter layout = write_flat order (network.cpp:186-193). */
#define ORC_K1 0
#define ORC_B1 150
#define ORC_K2 156
#define ORC_B2 1956
#define ORC_FC 1968
#define ORC_B 3888
#define ORC_NPARAM 3898
/* Per-image activation layout: c1[6,24,24] s1[6,12,12] c2[12,8,8] s2[12,4,4] out[10]. */
#define ORC_C1 0
#define ORC_S1 3456
#define ORC_C2 4320
#define ORC_S2 5088
#define ORC_OUT 5280
#define ORC_NACT 5290

/* --- PRNG + data ------------------------------------------------------------ */
void orc_init_params(uint64_t seed, float* params /*3898*/);
void orc_make_digits(int64_t n, uint64_t seed, uint8_t* pixels /*n*784*/, int32_t* labels);
void orc_make_set(int64_t n, uint64_t seed, float* images /*n*784*/, int32_t* labels);

/* --- scalar math ------------------------------------------------------------- */
float orc_expf(float x);          /* the host libm expf the reference calls (std::exp(float)) */
float orc_expf_port(float x);     /* restated glibc 2.39 expf algorithm (FMA variant) */
float orc_sigmoid(float x);       /* 1.0f / (1.0f + expf(-x)), nn.cpp:127-129 */
/* Exhaustive check of orc_expf_port vs libm expf over float bit patterns in
 * [lo_bits, hi_bits] (inclusive, both same sign); returns the mismatch count.  */
int64_t orc_expf_port_mismatches(uint32_t lo_bits, uint32_t hi_bits, int threads);
/* Compare device outputs `got[i]` for inputs with bit pattern (start + i) against libm. */
int64_t orc_expf_compare(uint32_t start_bits, int64_t count, const float* got, int threads,
                         uint32_t* first_bad_bits);

/* --- network (fixed Zhang shapes) -------------------------------------------- */
void orc_forward(const float* image, const float* params, float* act /*5290*/);
float orc_loss(const float* yhat, const float* y);
void orc_backward(const float* image, const float* act, const float* params, const float* y,
                  float* grad /*3898*/);
/* One example's train cell: grads[0..3897] + loss at [3898] (network.cpp:228-234). */
void orc_example_cell(const float* image, const float* params, int32_t label, float* cell);
/* net::train (network.cpp:209-251).  params is updated in place.  Returns 0, or a
 * negative code for the reference's argument errors (-1 empty, -2 epochs<0,
 * -3 rate<=0, -4 batch<1). */
int orc_train(const float* images, const int32_t* labels, int64_t n, float* params, float rate,
              int epochs, int64_t batch, double* epoch_loss, int threads);
/* One batch group [start, start+m): per-example cells reduced in example order,
 * then sgd_step.  loss_sum accumulates in double (network.cpp:236-244). */
void orc_train_group(const float* images, const int32_t* labels, int64_t start, int64_t m,
                     float* params, float rate, double* loss_sum, int threads);
int orc_predict(const float* yhat);
int64_t orc_evaluate(const float* params, const float* images, const int32_t* labels, int64_t n,
                     int32_t* pred, int threads);

/* --- generic rank-polymorphic nn ops (row-major, rank <= 8) ------------------ */
void orc_conv(const float* in, const int64_t* in_shape, int in_rank, const float* k,
              const int64_t* k_shape, float* out);
void orc_mconv(const float* in, const int64_t* in_shape, int in_rank, const float* k,
               const int64_t* k_shape /* rank in_rank+1 */, const float* b, float* out);
void orc_avgpool(const float* in, const int64_t* shape, int rank, float* out);
void orc_backavgpool(const float* d, const int64_t* shape, int rank, float* out);
void orc_backin(const float* d, const int64_t* d_shape, const float* k, const int64_t* k_shape,
                int rank, float* out /* shape = d_shape + k_shape - 1 */);
float orc_sum_all(const float* x, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
