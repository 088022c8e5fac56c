// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library (tensorloom), compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/libtloom_ref.so.
// It lets the pytest suite and bench.py's reference arm call the reference's own
// public API (tloom::net / tloom::nn / tloom::synth) through ctypes.  Nothing in
// the product links this.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "tloom/errors.hpp"
#include "tloom/mnist.hpp"
#include "tloom/network.hpp"
#include "tloom/nn.hpp"
#include "tloom/runtime.hpp"
#include "tloom/synth.hpp"
#include "tloom/tensor.hpp"

using namespace tloom;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const BoundsError*>(&e)) return 3;
  if (dynamic_cast<const ShapeError*>(&e)) return 2;
  if (dynamic_cast<const ValueError*>(&e)) return 5;
  if (dynamic_cast<const FormatError*>(&e)) return 4;
  if (dynamic_cast<const Error*>(&e)) return 1;
  return 9;
}

Shape shape_from(const int64_t* s, int r) { return Shape(std::span<const std::int64_t>(s, r)); }

Tensor tensor_from(const float* p, const int64_t* s, int r) {
  const Shape sh = shape_from(s, r);
  return Tensor(sh, std::vector<float>(p, p + sh.count()));
}

net::Params params_from(const float* p) {
  const int64_t n[6] = {150, 6, 1800, 12, 1920, 10};
  net::Params q = net::Params::zeros();
  Tensor* parts[6] = {&q.k1, &q.b1, &q.k2, &q.b2, &q.fc, &q.b};
  for (int i = 0; i < 6; ++i) {
    *parts[i] = Tensor(parts[i]->shape(), std::vector<float>(p, p + n[i]));
    p += n[i];
  }
  return q;
}

void params_to(const net::Params& q, float* out) {
  const Tensor* parts[6] = {&q.k1, &q.b1, &q.k2, &q.b2, &q.fc, &q.b};
  for (const Tensor* t : parts) {
    const auto d = t->data();
    std::memcpy(out, d.data(), d.size() * sizeof(float));
    out += d.size();
  }
}

void copy_out(const Tensor& t, float* out) {
  const auto d = t.data();
  std::memcpy(out, d.data(), d.size() * sizeof(float));
}

mnist::MnistSet set_from(const float* images, const int32_t* labels, int64_t n) {
  return mnist::make_set(Tensor(Shape{n, 28, 28}, std::vector<float>(images, images + n * 784)),
                         std::vector<int>(labels, labels + n));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_set_workers(int workers) {
  try {
    runtime::set_global_config({workers, 4096});
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_init_params(uint64_t seed, float* out) { params_to(net::init_params(seed), out); }

// TLM1 checkpoint round trip through the reference's own codec (network.cpp:282-362).
int ref_save_params(const char* path, const float* params) {
  try {
    net::save_params(path, params_from(params));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_load_params(const char* path, float* out) {
  try {
    params_to(net::load_params(path), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// mnist::load_set of IDX files (mnist.cpp:126-154) -> images [n][784], labels [n]; returns n.
int64_t ref_load_set(const char* images_path, const char* labels_path, int64_t limit, float* images, int32_t* labels) {
  try {
    const mnist::MnistSet s = mnist::load_set(images_path, labels_path, limit);
    if (images) copy_out(s.images, images);
    if (labels)
      for (int64_t i = 0; i < s.size(); ++i) labels[i] = s.labels[static_cast<std::size_t>(i)];
    return s.size();
  } catch (const std::exception& e) {
    return -fail(e);
  }
}

void ref_make_digits(int64_t n, uint64_t seed, uint8_t* px, int32_t* labels) {
  const synth::Corpus c = synth::make_digits(n, seed);
  std::memcpy(px, c.pixels.data(), c.pixels.size());
  for (int64_t i = 0; i < n; ++i) labels[i] = c.labels[static_cast<std::size_t>(i)];
}

void ref_make_set(int64_t n, uint64_t seed, float* images, int32_t* labels) {
  const mnist::MnistSet s = synth::make_set(n, seed);
  copy_out(s.images, images);
  for (int64_t i = 0; i < n; ++i) labels[i] = s.labels[static_cast<std::size_t>(i)];
}

// net::forward on one image; act = c1,s1,c2,s2,out flattened (5290 floats).
int ref_forward(const float* image, const float* params, float* act) {
  try {
    const auto [yhat, cache] = net::forward(Tensor(Shape{28, 28}, std::vector<float>(image, image + 784)),
                                            params_from(params));
    copy_out(cache.c1, act);
    copy_out(cache.s1, act + 3456);
    copy_out(cache.c2, act + 4320);
    copy_out(cache.s2, act + 5088);
    copy_out(cache.out, act + 5280);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// forward + backward + loss for one example with a dense target y[10].
int ref_forward_backward(const float* image, const float* params, const float* y, float* cell) {
  try {
    const net::Params p = params_from(params);
    const Tensor yt(Shape{10}, std::vector<float>(y, y + 10));
    const auto [yhat, cache] =
        net::forward(Tensor(Shape{28, 28}, std::vector<float>(image, image + 784)), p);
    const net::Grads g = net::backward(cache, p, yt);
    net::Params as_p{g.k1, g.b1, g.k2, g.b2, g.fc, g.b};
    params_to(as_p, cell);
    cell[3898] = net::loss(yhat, yt);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_train(const float* images, const int32_t* labels, int64_t n, float* params, float rate,
              int epochs, int64_t batch, double* epoch_loss) {
  try {
    net::Hyper h;
    h.rate = rate;
    h.epochs = epochs;
    h.batch = batch;
    const net::TrainResult r = net::train(params_from(params), set_from(images, labels, n), h);
    params_to(r.params, params);
    for (std::size_t e = 0; e < r.epoch_mean_loss.size(); ++e) epoch_loss[e] = r.epoch_mean_loss[e];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_evaluate(const float* params, const float* images, const int32_t* labels, int64_t n,
                 int32_t* pred, double* accuracy) {
  try {
    const net::Params p = params_from(params);
    const mnist::MnistSet s = set_from(images, labels, n);
    if (pred)
      for (int64_t i = 0; i < n; ++i)
        pred[i] = net::predict(net::forward(s.images.select(Index{i}), p).first);
    *accuracy = net::evaluate(p, s);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Generic ops.  Shapes are passed as (ptr, rank); outputs must be pre-sized.
int ref_conv(const float* in, const int64_t* is, int ir, const float* k, const int64_t* ks, int kr,
             float* out) {
  try {
    copy_out(nn::conv(tensor_from(in, is, ir), tensor_from(k, ks, kr)), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_mconv(const float* in, const int64_t* is, int ir, const float* k, const int64_t* ks, int kr,
              const float* b, const int64_t* bs, int br, float* out) {
  try {
    copy_out(nn::mconv(tensor_from(in, is, ir), tensor_from(k, ks, kr), tensor_from(b, bs, br)), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_sigmoid(const float* in, const int64_t* s, int r, float* out) {
  try {
    copy_out(nn::sigmoid(tensor_from(in, s, r)), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_avgpool(const float* in, const int64_t* s, int r, float* out) {
  try {
    copy_out(nn::avgpool(tensor_from(in, s, r)), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_backavgpool(const float* d, const int64_t* s, int r, float* out) {
  try {
    copy_out(nn::backavgpool(tensor_from(d, s, r)), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_backin(const float* d, const int64_t* ds, const float* k, const int64_t* ks,
               const int64_t* ins, int r, float* out) {
  try {
    copy_out(nn::backin(tensor_from(d, ds, r), tensor_from(k, ks, r), Tensor::zeros(shape_from(ins, r))),
             out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_backweights(const float* d, const int64_t* ds, const float* in, const int64_t* ins, int r,
                    float* out) {
  try {
    copy_out(nn::backweights(tensor_from(d, ds, r), tensor_from(in, ins, r)), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_backsigmoid(const float* d, const float* o, const int64_t* s, int r, float* out) {
  try {
    copy_out(nn::backsigmoid(tensor_from(d, s, r), tensor_from(o, s, r)), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

float ref_backbias(const float* d, const int64_t* s, int r) {
  return nn::backbias(tensor_from(d, s, r));
}

}  // extern "C"
