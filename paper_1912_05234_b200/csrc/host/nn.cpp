// nn.cpp -- tloom::nn (include/tloom/nn.hpp) over the C ABI: shape checks with the reference's
// messages (nn.cpp:37-94 of the reference), then the sm_100a op kernels (tlb_nn_*).
#include "tloom/nn.hpp"

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "device.hpp"
#include "tloom_b200.h"

namespace tloom {

namespace detail {

namespace {
std::mutex g_mutex;
tlb_ctx* g_ctx = nullptr;
}  // namespace

void raise(int status) {
  if (status == TLB_OK) return;
  const std::string msg = tlb_last_error();
  switch (status) {
    case TLB_ERR_SHAPE: throw ShapeError(msg);
    case TLB_ERR_BOUNDS: throw BoundsError(msg);
    case TLB_ERR_FORMAT: throw FormatError(msg);
    case TLB_ERR_VALUE: throw ValueError(msg);
    default: throw Error(msg);
  }
}

void check(int status) { raise(status); }

DeviceLock device() {
  std::unique_lock<std::mutex> lk(g_mutex);
  if (!g_ctx) {
    // TLOOM_B200_DEVICES=0,1,2,3: one context over several GPUs (net::train splits every group over them);
    // else TLOOM_B200_DEVICE (default 0)
    if (const char* list = std::getenv("TLOOM_B200_DEVICES")) {
      std::vector<int> devs;
      for (const char* p = list; *p;) {
        char* end = nullptr;
        devs.push_back(static_cast<int>(std::strtol(p, &end, 10)));
        p = (*end == ',') ? end + 1 : end;
        if (end == p && *p) break;
      }
      check(tlb_ctx_create_multi(devs.data(), static_cast<int>(devs.size()), &g_ctx));
    } else {
      const char* dev = std::getenv("TLOOM_B200_DEVICE");
      check(tlb_ctx_create(dev ? std::atoi(dev) : 0, &g_ctx));
    }
    const char* mode = std::getenv("TLOOM_B200_MODE");
    if (mode && std::strcmp(mode, "fast") == 0) check(tlb_ctx_set_mode(g_ctx, TLB_MODE_FAST));
  }
  return DeviceLock{std::move(lk), g_ctx};
}

}  // namespace detail

namespace nn {

namespace {

struct Dims {
  std::int64_t e[8] = {};
  int r = 0;
  explicit Dims(const Shape& s) : r(s.rank()) {
    for (int a = 0; a < r; ++a) e[a] = s[a];
  }
};

Shape shape_of_dims(const std::int64_t* e, int r) { return Shape(std::span<const std::int64_t>(e, r)); }

}  // namespace

Shape conv_result_shape(const Shape& in, const Shape& k) {
  const Dims a(in), b(k);
  std::int64_t out[8];
  int r = 0;
  detail::check(tlb_nn_conv_shape(a.e, a.r, b.e, b.r, out, &r));
  return shape_of_dims(out, r);
}

Shape mconv_result_shape(const Shape& in, const Shape& k, const Shape& b) {
  const Dims x(in), y(k), z(b);
  std::int64_t out[8];
  int r = 0;
  detail::check(tlb_nn_mconv_shape(x.e, x.r, y.e, y.r, z.e, z.r, out, &r));
  return shape_of_dims(out, r);
}

Shape avgpool_result_shape(const Shape& in) {
  const Dims x(in);
  std::int64_t out[8];
  int r = 0;
  detail::check(tlb_nn_avgpool_shape(x.e, x.r, out, &r));
  return shape_of_dims(out, r);
}

Shape backavgpool_result_shape(const Shape& in) {
  const Dims x(in);
  std::int64_t out[8];
  int r = 0;
  detail::check(tlb_nn_backavgpool_shape(x.e, x.r, out, &r));
  return shape_of_dims(out, r);
}

Shape backin_result_shape(const Shape& d_out, const Shape& k, const Shape& in) {
  const Dims a(d_out), b(k), c(in);
  std::int64_t out[8];
  int r = 0;
  detail::check(tlb_nn_backin_shape(a.e, a.r, b.e, b.r, c.e, c.r, out, &r));
  return shape_of_dims(out, r);
}

Tensor conv(const Tensor& in, const Tensor& k) {
  const Shape os = conv_result_shape(in.shape(), k.shape());
  std::vector<float> out(static_cast<std::size_t>(os.count()));
  const Dims a(in.shape()), b(k.shape());
  auto dev = detail::device();
  detail::check(tlb_nn_conv(dev.ctx, in.data().data(), a.e, a.r, k.data().data(), b.e, b.r, out.data()));
  return Tensor(os, std::move(out));
}

Tensor mconv(const Tensor& in, const Tensor& k, const Tensor& b) {
  const Shape os = mconv_result_shape(in.shape(), k.shape(), b.shape());
  std::vector<float> out(static_cast<std::size_t>(os.count()));
  const Dims x(in.shape()), y(k.shape()), z(b.shape());
  auto dev = detail::device();
  detail::check(tlb_nn_mconv(dev.ctx, in.data().data(), x.e, x.r, k.data().data(), y.e, y.r, b.data().data(), z.e,
                             z.r, out.data()));
  return Tensor(os, std::move(out));
}

Tensor sigmoid(const Tensor& t) {
  std::vector<float> out(static_cast<std::size_t>(t.count()));
  auto dev = detail::device();
  detail::check(tlb_nn_sigmoid(dev.ctx, t.data().data(), t.count(), out.data()));
  return Tensor(t.shape(), std::move(out));
}

Tensor backsigmoid(const Tensor& d_out, const Tensor& out) {
  if (d_out.shape() != out.shape())
    throw ShapeError("map_binary: shapes " + d_out.shape().str() + " and " + out.shape().str() + " differ");
  std::vector<float> r(static_cast<std::size_t>(d_out.count()));
  auto dev = detail::device();
  detail::check(tlb_nn_backsigmoid(dev.ctx, d_out.data().data(), out.data().data(), d_out.count(), r.data()));
  return Tensor(d_out.shape(), std::move(r));
}

Tensor avgpool(const Tensor& t) {
  const Shape os = avgpool_result_shape(t.shape());
  std::vector<float> out(static_cast<std::size_t>(os.count()));
  const Dims a(t.shape());
  auto dev = detail::device();
  detail::check(tlb_nn_avgpool(dev.ctx, t.data().data(), a.e, a.r, out.data()));
  return Tensor(os, std::move(out));
}

Tensor backavgpool(const Tensor& d_out) {
  const Shape os = backavgpool_result_shape(d_out.shape());
  std::vector<float> out(static_cast<std::size_t>(os.count()));
  const Dims a(d_out.shape());
  auto dev = detail::device();
  detail::check(tlb_nn_backavgpool(dev.ctx, d_out.data().data(), a.e, a.r, out.data()));
  return Tensor(os, std::move(out));
}

Tensor backweights(const Tensor& d_out, const Tensor& in) { return conv(in, d_out); }

float backbias(const Tensor& d_out) {
  float out = 0.0f;
  auto dev = detail::device();
  detail::check(tlb_nn_backbias(dev.ctx, d_out.data().data(), d_out.count(), &out));
  return out;
}

Tensor backin(const Tensor& d_out, const Tensor& k, const Tensor& in) {
  const Shape os = backin_result_shape(d_out.shape(), k.shape(), in.shape());
  std::vector<float> out(static_cast<std::size_t>(os.count()));
  const Dims a(d_out.shape()), b(k.shape()), c(in.shape());
  auto dev = detail::device();
  detail::check(tlb_nn_backin(dev.ctx, d_out.data().data(), a.e, a.r, k.data().data(), b.e, b.r, c.e, c.r,
                              out.data()));
  return Tensor(os, std::move(out));
}

}  // namespace nn
}  // namespace tloom
