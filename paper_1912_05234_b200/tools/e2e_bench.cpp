// e2e_bench.cpp -- end-to-end timing of the C++ drop-in: tloom::net::train called exactly as the
// reference's callers call it (proj/tools/tensorloom_cli.cpp:102-112, proj/tests/acceptance.cpp:245):
// a host MnistSet (std::vector storage) in, TrainResult out, one epoch per call.  Every call moves the
// dataset host -> device and the parameters back inside the timed region (the mirror page-locks the set's
// storage from its second call on, so the timed calls DMA straight from it; the H2D itself stays per call).
//
//   tloom-e2e-bench [--n 10000] [--batch 100] [--rate 0.05] [--steps 10] [--warmup 3] [--mode fast|exact]
//
// Prints one JSON line: images/s over the timed calls (wall clock, std::chrono::steady_clock), per-call
// milliseconds, the bytes each call moves, and the epoch losses of the timed calls.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "tloom/errors.hpp"
#include "tloom/mnist.hpp"
#include "tloom/network.hpp"
#include "tloom/synth.hpp"

namespace {

long long arg_i64(int argc, char** argv, const char* name, long long dflt) {
  for (int i = 1; i + 1 < argc; ++i)
    if (!std::strcmp(argv[i], name)) return std::atoll(argv[i + 1]);
  return dflt;
}
std::string arg_str(int argc, char** argv, const char* name, const char* dflt) {
  for (int i = 1; i + 1 < argc; ++i)
    if (!std::strcmp(argv[i], name)) return argv[i + 1];
  return dflt;
}

}  // namespace

int main(int argc, char** argv) {
  const std::int64_t n = arg_i64(argc, argv, "--n", 10000);
  const std::int64_t batch = arg_i64(argc, argv, "--batch", 100);
  const int steps = (int)arg_i64(argc, argv, "--steps", 10);
  const int warmup = (int)arg_i64(argc, argv, "--warmup", 3);
  const float rate = std::strtof(arg_str(argc, argv, "--rate", "0.05").c_str(), nullptr);
  const std::string mode = arg_str(argc, argv, "--mode", "fast");
  if (mode != "fast" && mode != "exact") {
    std::fprintf(stderr, "--mode: expected fast or exact\n");
    return 2;
  }
  setenv("TLOOM_B200_MODE", mode.c_str(), 1);  // read once, when the device context is created
  try {
    const tloom::mnist::MnistSet data = tloom::synth::make_set(n, 1);
    tloom::net::Params p = tloom::net::init_params(42);
    const tloom::net::Hyper h{rate, 1, batch, 42};
    for (int i = 0; i < warmup; ++i) p = tloom::net::train(p, data, h).params;
    std::vector<double> call_ms, losses;
    using Clock = std::chrono::steady_clock;
    const auto t0 = Clock::now();
    for (int i = 0; i < steps; ++i) {
      const auto c0 = Clock::now();
      tloom::net::TrainResult r = tloom::net::train(p, data, h);
      call_ms.push_back(std::chrono::duration<double, std::milli>(Clock::now() - c0).count());
      losses.push_back(r.epoch_mean_loss.at(0));
      p = std::move(r.params);
    }
    const double total_s = std::chrono::duration<double>(Clock::now() - t0).count();
    std::vector<double> sorted = call_ms;
    std::sort(sorted.begin(), sorted.end());
    const double med = sorted.empty() ? 0.0 : sorted[sorted.size() / 2];
    const long long h2d = (long long)n * 784 * 4 + (long long)n * 4 + 3898 * 4;
    const long long d2h = 3898 * 4 + 8;
    std::printf("{\"api\": \"tloom::net::train (C++ drop-in on a host MnistSet; the mirror page-locks a set it trains twice)\", "
                "\"mode\": \"%s\", "
                "\"n\": %lld, \"batch\": %lld, \"steps\": %d, \"warmup\": %d, \"images_per_s\": %.6f, "
                "\"call_ms\": {\"median\": %.6f, \"min\": %.6f, \"max\": %.6f}, \"h2d_bytes_per_step\": %lld, "
                "\"d2h_bytes_per_step\": %lld, \"epoch_loss\": [",
                mode.c_str(), (long long)n, (long long)batch, steps, warmup,
                steps > 0 ? (double)n * steps / total_s : 0.0, med, sorted.empty() ? 0.0 : sorted.front(),
                sorted.empty() ? 0.0 : sorted.back(), h2d, d2h);
    for (std::size_t i = 0; i < losses.size(); ++i) std::printf("%s%.17g", i ? ", " : "", losses[i]);
    std::printf("]}\n");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "e2e_bench: %s\n", e.what());
    return 4;
  }
  return 0;
}
