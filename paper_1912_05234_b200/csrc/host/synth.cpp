// synth.cpp -- tloom::synth (include/tloom/synth.hpp) over tlb_synth_make_digits (host_data.cpp).
#include "tloom/synth.hpp"

#include "device.hpp"
#include "tloom_b200.h"

namespace tloom::synth {

Corpus make_digits(std::int64_t n, std::uint64_t seed) {
  if (n < 0) throw Error("make_digits: negative count");
  Corpus c;
  c.pixels.resize(static_cast<std::size_t>(n) * 784);
  std::vector<std::int32_t> lab(static_cast<std::size_t>(n));
  detail::check(tlb_synth_make_digits(n, seed, c.pixels.data(), lab.data()));
  c.labels.assign(lab.begin(), lab.end());
  return c;
}

mnist::MnistSet make_set(std::int64_t n, std::uint64_t seed) {
  Corpus c = make_digits(n, seed);
  std::vector<float> px(c.pixels.size());
  for (std::size_t i = 0; i < px.size(); ++i) px[i] = static_cast<float>(c.pixels[i]) / 255.0f;
  return mnist::make_set(Tensor(Shape{n, 28, 28}, std::move(px)), std::move(c.labels));
}

}  // namespace tloom::synth
