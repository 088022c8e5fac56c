// tloom/network.hpp -- the Zhang digit CNN and its training driver, on the B200 (sm_100a).
//
// Drop-in for proj/include/tloom/network.hpp:12-93.  forward / backward / train / evaluate run the
// fused shared-memory kernels through the C ABI (tloom_b200.h):
//   train    -> tlb_train: one persistent cooperative kernel per call (or per epoch with on_epoch),
//               per-example forward+backward in shared memory, example-order batch reduction,
//               sgd_step; bitwise identical to the reference in the default EXACT mode.
//   forward  -> tlb_forward (activations returned as the ActCache)
//   backward -> tlb_backward (gradients from the cached activations)
//   evaluate -> tlb_evaluate (forward + argmax + correct count)
// Set TLOOM_B200_MODE=fast for the FFMA / per-CTA-partial variant (within 1e-4 of the reference).
#pragma once

#include <cstdint>
#include <filesystem>
#include <functional>
#include <utility>
#include <vector>

#include "tloom/mnist.hpp"
#include "tloom/tensor.hpp"

namespace tloom::net {

struct Params {
  Tensor k1;  // [6,5,5]
  Tensor b1;  // [6]
  Tensor k2;  // [12,6,5,5]
  Tensor b2;  // [12]
  Tensor fc;  // [10,12,1,4,4]
  Tensor b;   // [10]

  void validate() const;  // ShapeError unless every tensor has its signature shape
  static Params zeros();
};

struct Grads {
  Tensor k1, b1, k2, b2, fc, b;
};

struct ActCache {
  Tensor input;  // [28,28]
  Tensor c1;     // [6,24,24]
  Tensor s1;     // [6,12,12]
  Tensor c2;     // [12,1,8,8]
  Tensor s2;     // [12,1,4,4]
  Tensor out;    // [10,1,1,1,1]
};

struct Hyper {
  float rate = 0.05f;
  int epochs = 10;
  std::int64_t batch = 100;
  std::uint64_t seed = 42;
};

struct TrainResult {
  Params params;
  std::vector<double> epoch_mean_loss;
};

Params init_params(std::uint64_t seed);
std::pair<Tensor, ActCache> forward(const Tensor& image, const Params& p);
float loss(const Tensor& yhat, const Tensor& y);
Grads backward(const ActCache& cache, const Params& p, const Tensor& y);
Params sgd_step(const Params& p, const Grads& acc, float rate, std::int64_t batch);
TrainResult train(const Params& p, const mnist::MnistSet& data, const Hyper& h,
                  const std::function<void(int, double)>& on_epoch = {});
int predict(const Tensor& yhat);
double evaluate(const Params& p, const mnist::MnistSet& data);
void save_params(const std::filesystem::path& path, const Params& p);
Params load_params(const std::filesystem::path& path);

}  // namespace tloom::net
