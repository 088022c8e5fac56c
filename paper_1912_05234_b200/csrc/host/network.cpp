// network.cpp -- tloom::net (include/tloom/network.hpp) over the C ABI.
//
// Parameter tensors travel as one flat fp32 buffer in write_flat order (reference network.cpp:186-193);
// train / forward / backward / loss / sgd_step / evaluate run on the B200 (tlb_* entry points).
// Argument checks and messages follow the reference (network.cpp:27-49, 83-85, 98-101, 211-214).
#include "tloom/network.hpp"

#include <algorithm>
#include <bit>
#include <cstring>
#include <fstream>
#include <iterator>

#include "device.hpp"
#include "tloom_b200.h"

namespace tloom::net {

namespace {

const Shape kK1{6, 5, 5}, kB1{6}, kK2{12, 6, 5, 5}, kB2{12}, kFc{10, 12, 1, 4, 4}, kB{10}, kImage{28, 28};

void expect(const Tensor& t, const Shape& s, const char* name) {
  if (t.shape() != s)
    throw ShapeError(std::string("params: ") + name + " has shape " + t.shape().str() + ", expected " + s.str());
}

std::vector<float> flat(const Params& p) {
  std::vector<float> v;
  v.reserve(TLB_NPARAM);
  for (const Tensor* t : {&p.k1, &p.b1, &p.k2, &p.b2, &p.fc, &p.b}) v.insert(v.end(), t->data().begin(), t->data().end());
  return v;
}

template <class T>
T unflat(const float* v) {
  const Shape* shapes[6] = {&kK1, &kB1, &kK2, &kB2, &kFc, &kB};
  Tensor parts[6];
  for (int i = 0; i < 6; ++i) {
    const auto n = static_cast<std::size_t>(shapes[i]->count());
    parts[i] = Tensor(*shapes[i], std::vector<float>(v, v + n));
    v += n;
  }
  return T{parts[0], parts[1], parts[2], parts[3], parts[4], parts[5]};
}

}  // namespace

void Params::validate() const {
  expect(k1, kK1, "k1");
  expect(b1, kB1, "b1");
  expect(k2, kK2, "k2");
  expect(b2, kB2, "b2");
  expect(fc, kFc, "fc");
  expect(b, kB, "b");
}

Params Params::zeros() {
  return Params{Tensor::zeros(kK1), Tensor::zeros(kB1), Tensor::zeros(kK2),
                Tensor::zeros(kB2), Tensor::zeros(kFc), Tensor::zeros(kB)};
}

Params init_params(std::uint64_t seed) {
  std::vector<float> v(TLB_NPARAM);
  detail::check(tlb_init_params(seed, v.data()));
  return unflat<Params>(v.data());
}

std::pair<Tensor, ActCache> forward(const Tensor& image, const Params& p) {
  p.validate();
  if (image.shape() != kImage)
    throw ShapeError("forward: image has shape " + image.shape().str() + ", expected " + kImage.str());
  const std::vector<float> w = flat(p);
  std::vector<float> yhat(10), act(TLB_NACT);
  {
    auto dev = detail::device();
    detail::check(tlb_forward(dev.ctx, image.data().data(), 1, w.data(), yhat.data(), act.data()));
  }
  ActCache c;
  c.input = image;
  const float* a = act.data();
  c.c1 = Tensor(Shape{6, 24, 24}, std::vector<float>(a, a + 3456));
  c.s1 = Tensor(Shape{6, 12, 12}, std::vector<float>(a + 3456, a + 4320));
  c.c2 = Tensor(Shape{12, 1, 8, 8}, std::vector<float>(a + 4320, a + 5088));
  c.s2 = Tensor(Shape{12, 1, 4, 4}, std::vector<float>(a + 5088, a + 5280));
  c.out = Tensor(Shape{10, 1, 1, 1, 1}, std::vector<float>(a + 5280, a + 5290));
  return {c.out.reshape(Shape{10}), c};
}

float loss(const Tensor& yhat, const Tensor& y) {
  if (yhat.shape() != Shape{10} || y.shape() != Shape{10})
    throw ShapeError("loss: shapes " + yhat.shape().str() + " and " + y.shape().str() + ", expected [10] and [10]");
  float out = 0.0f;
  auto dev = detail::device();
  detail::check(tlb_loss(dev.ctx, yhat.data().data(), y.data().data(), 1, &out));
  return out;
}

Grads backward(const ActCache& cache, const Params& p, const Tensor& y) {
  p.validate();
  if (y.shape() != Shape{10})
    throw ShapeError("ew_map2: shapes [10] and " + y.shape().str() + " differ");
  std::vector<float> act;
  act.reserve(TLB_NACT);
  for (const Tensor* t : {&cache.c1, &cache.s1, &cache.c2, &cache.s2, &cache.out})
    act.insert(act.end(), t->data().begin(), t->data().end());
  if (act.size() != TLB_NACT || cache.input.count() != 784)
    throw ShapeError("backward: activation cache does not match the network signature");
  const std::vector<float> w = flat(p);
  std::vector<float> g(TLB_NPARAM);
  {
    auto dev = detail::device();
    detail::check(tlb_backward(dev.ctx, cache.input.data().data(), act.data(), y.data().data(), 1, w.data(), g.data()));
  }
  return unflat<Grads>(g.data());
}

Params sgd_step(const Params& p, const Grads& acc, float rate, std::int64_t batch) {
  if (batch < 1) throw Error("sgd_step: batch must be >= 1");
  const std::vector<float> w = flat(p);
  std::vector<float> g;
  g.reserve(TLB_NPARAM);
  for (const Tensor* t : {&acc.k1, &acc.b1, &acc.k2, &acc.b2, &acc.fc, &acc.b}) g.insert(g.end(), t->data().begin(), t->data().end());
  if (g.size() != TLB_NPARAM || w.size() != TLB_NPARAM) throw ShapeError("sgd_step: parameter/gradient shapes differ");
  std::vector<float> out(TLB_NPARAM);
  auto dev = detail::device();
  detail::check(tlb_sgd_step(dev.ctx, w.data(), g.data(), rate, batch, out.data()));
  return unflat<Params>(out.data());
}

namespace {
void epoch_trampoline(int epoch, double mean, void* user) {
  (*static_cast<const std::function<void(int, double)>*>(user))(epoch, mean);
}
}  // namespace

namespace {
// The training set of the last net::train calls: a set trained twice in a row has its image storage
// page-locked (tlb_host_register) from the second call on, so every later call DMAs straight from it
// instead of staging through the pinned bounce slots (the pageable path).  The Tensor copy keeps the
// storage alive -- and its address unique -- for as long as it is registered; a different set replaces
// it (the old range is unregistered first).  Accessed under the device lock.
struct PinnedSet {
  Tensor images;  // shares the caller's storage
  const float* ptr = nullptr;
  std::size_t bytes = 0;
  bool registered = false;
};
PinnedSet g_pinned;

void pin_training_set(tlb_ctx* ctx, const Tensor& images) {
  constexpr std::size_t kMinBytes = 4u << 20;  // smaller sets: the bounce path is as fast
  const std::span<const float> v = images.data();
  const std::size_t bytes = v.size_bytes();
  if (bytes < kMinBytes) return;
  if (v.data() == g_pinned.ptr && bytes == g_pinned.bytes) {  // seen before (and still alive: we hold it)
    if (!g_pinned.registered) g_pinned.registered = tlb_host_register(ctx, v.data(), bytes) == TLB_OK;
    return;
  }
  if (g_pinned.registered) (void)tlb_host_unregister(ctx, g_pinned.ptr);
  g_pinned = PinnedSet{images, v.data(), bytes, false};  // registered if the next call trains it again
}
}  // namespace

TrainResult train(const Params& p, const mnist::MnistSet& data, const Hyper& h,
                  const std::function<void(int, double)>& on_epoch) {
  p.validate();
  if (data.size() == 0) throw Error("train: empty dataset");
  if (h.epochs < 0) throw Error("train: negative epoch count");
  if (!(h.rate > 0.0f)) throw Error("train: rate must be > 0");
  if (h.batch < 1) throw Error("batches: size must be >= 1, got " + std::to_string(h.batch));
  std::vector<float> w = flat(p);
  // The dataset goes to the device straight from the MnistSet's own storage (no host copy): the image
  // tensor's contiguous floats and the label vector (int is int32_t here).
  static_assert(sizeof(int) == sizeof(std::int32_t), "labels are passed as int32");
  const std::span<const float> images = data.images.data();
  const auto* labels = reinterpret_cast<const std::int32_t*>(data.labels.data());
  std::vector<double> losses(static_cast<std::size_t>(h.epochs));
  {
    auto dev = detail::device();
    pin_training_set(dev.ctx, data.images);
    detail::check(tlb_train(dev.ctx, images.data(), labels, data.size(), w.data(), h.rate, h.epochs, h.batch,
                            losses.data(), on_epoch ? epoch_trampoline : nullptr,
                            const_cast<std::function<void(int, double)>*>(&on_epoch)));
  }
  return TrainResult{unflat<Params>(w.data()), std::move(losses)};
}

int predict(const Tensor& yhat) {
  if (yhat.shape() != Shape{10}) throw ShapeError("predict: shape " + yhat.shape().str() + ", expected [10]");
  const auto v = yhat.data();
  int best = 0;
  for (int i = 1; i < 10; ++i)
    if (v[static_cast<std::size_t>(i)] > v[static_cast<std::size_t>(best)]) best = i;
  return best;
}

double evaluate(const Params& p, const mnist::MnistSet& data) {
  p.validate();
  if (data.size() == 0) throw Error("evaluate: empty dataset");
  const std::vector<float> w = flat(p);
  const std::span<const float> images = data.images.data();
  const auto* labels = reinterpret_cast<const std::int32_t*>(data.labels.data());
  std::int64_t correct = 0;
  auto dev = detail::device();
  detail::check(tlb_evaluate(dev.ctx, images.data(), labels, data.size(), w.data(), nullptr, &correct));
  return static_cast<double>(correct) / static_cast<double>(data.size());
}

// ---- TLM1 checkpoints --------------------------------------------------------------------------
// Byte format (the reference's, so its own load_params reads our files: proj/src/network.cpp:282-362):
// "TLM1", then per tensor in write_flat order: u32 rank, u32 extents, f32 payload, all little-endian.
// Here a checkpoint is just the flat parameter vector framed by the section table below; the
// reader fills the flat vector section by section and rebuilds Params with unflat.
namespace {

struct Section {
  const char* name;
  const Shape* shape;
};
const Section kSections[6] = {{"k1", &kK1}, {"b1", &kB1}, {"k2", &kK2}, {"b2", &kB2}, {"fc", &kFc}, {"b", &kB}};

class LeWriter {
 public:
  void word(std::uint32_t v) {
    unsigned char b[4];
    for (int k = 0; k < 4; ++k) b[k] = static_cast<unsigned char>((v >> (8 * k)) & 0xffu);
    bytes.insert(bytes.end(), b, b + 4);
  }
  std::vector<unsigned char> bytes{'T', 'L', 'M', '1'};
};

class LeReader {
 public:
  explicit LeReader(const std::vector<unsigned char>& b) : b_(b) {}
  std::uint32_t word() {
    if (b_.size() < 4 || pos_ > b_.size() - 4) throw FormatError("checkpoint: truncated at byte " + std::to_string(pos_));
    std::uint32_t v = 0;
    for (int k = 3; k >= 0; --k) v = (v << 8) | b_[pos_ + static_cast<std::size_t>(k)];
    pos_ += 4;
    return v;
  }
  std::size_t pos() const { return pos_; }
  void seek(std::size_t p) { pos_ = p; }

 private:
  const std::vector<unsigned char>& b_;
  std::size_t pos_ = 0;
};

}  // namespace

void save_params(const std::filesystem::path& path, const Params& p) {
  p.validate();
  const std::vector<float> w = flat(p);
  LeWriter out;
  std::size_t at = 0;
  for (const Section& sec : kSections) {
    const Shape& s = *sec.shape;
    out.word(static_cast<std::uint32_t>(s.rank()));
    for (int a = 0; a < s.rank(); ++a) out.word(static_cast<std::uint32_t>(s[a]));
    for (std::int64_t i = 0; i < s.count(); ++i) out.word(std::bit_cast<std::uint32_t>(w[at++]));
  }
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw FormatError("cannot open checkpoint for writing: " + path.string());
  f.write(reinterpret_cast<const char*>(out.bytes.data()), static_cast<std::streamsize>(out.bytes.size()));
  if (!f) throw FormatError("write failure on checkpoint: " + path.string());
}

Params load_params(const std::filesystem::path& path) {
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  if (!f) throw FormatError("cannot open checkpoint: " + path.string());
  std::vector<unsigned char> bytes(static_cast<std::size_t>(std::max<std::streamoff>(0, f.tellg())));
  f.seekg(0);
  if (!bytes.empty()) f.read(reinterpret_cast<char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
  if (f.bad()) throw FormatError("read failure on checkpoint: " + path.string());
  if (bytes.size() < 4 || std::memcmp(bytes.data(), "TLM1", 4) != 0)
    throw FormatError("checkpoint: bad magic, expected \"TLM1\"");
  LeReader in(bytes);
  in.seek(4);
  std::vector<float> w;
  w.reserve(TLB_NPARAM);
  for (const Section& sec : kSections) {
    const std::uint32_t rank = in.word();
    if (rank > static_cast<std::uint32_t>(Shape::kMaxRank))
      throw FormatError("checkpoint: tensor " + std::string(sec.name) + " has rank " + std::to_string(rank));
    std::int64_t ext[Shape::kMaxRank];
    for (std::uint32_t a = 0; a < rank; ++a) ext[a] = in.word();
    const Shape got{std::span<const std::int64_t>(ext, rank)};
    if (got != *sec.shape)
      throw FormatError("checkpoint: tensor " + std::string(sec.name) + " has shape " + got.str() + ", expected " +
                        sec.shape->str());
    for (std::int64_t i = 0; i < got.count(); ++i) w.push_back(std::bit_cast<float>(in.word()));
  }
  if (in.pos() != bytes.size()) throw FormatError("checkpoint: " + std::to_string(bytes.size() - in.pos()) + " trailing bytes");
  return unflat<Params>(w.data());
}

}  // namespace tloom::net
