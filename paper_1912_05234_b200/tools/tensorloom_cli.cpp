// tensorloom_cli.cpp -- the `tensorloom` command-line driver (train / bench / eval) on the B200.
//
// Same sub-commands, flags, defaults, stdout/stderr split and exit codes as the reference CLI
// (proj/tools/tensorloom_cli.cpp:18-213): results and CSV on stdout, progress on stderr; exit 0 ok,
// 2 usage error, 3 FormatError (bad IDX / checkpoint file), 4 any other error or a determinism
// mismatch in `bench`.  Every tloom:: call goes through the C++ mirror (include/tloom/) to the
// sm_100a kernels.  The reference parses with CLI11 (not vendored there); this driver carries its own
// small parser with the same option set and range checks.
//
// B200 specifics: `--mt` keeps its meaning for the host-side helpers (results do not depend on it,
// exactly as in the reference); `--mode exact|fast` selects the bitwise (default) or FFMA path
// (also TLOOM_B200_MODE).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "tloom/errors.hpp"
#include "tloom/mnist.hpp"
#include "tloom/network.hpp"
#include "tloom/runtime.hpp"

namespace {

using Clock = std::chrono::steady_clock;

double seconds_since(Clock::time_point start) {
  return std::chrono::duration<double>(Clock::now() - start).count();
}

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct CommonArgs {
  std::string train_images, train_labels, test_images, test_labels;
  std::string checkpoint;
  int epochs = 10;
  std::int64_t batch = 100;
  float rate = 0.05f;
  int mt = 1;
  std::uint64_t seed = 42;
  std::int64_t limit_train = 10000;
  std::int64_t limit_test = 10000;
  std::vector<int> bench_workers = {1, 2, 4, 8};
};

// --- minimal option parser (long options, "--name value" or "--name=value") ---------------------
struct Parsed {
  std::map<std::string, std::string> opts;
};

Parsed parse_opts(int argc, char** argv, int first, const std::vector<std::string>& known) {
  Parsed p;
  for (int i = first; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + a);
    std::string name = a.substr(2), val;
    const auto eq = name.find('=');
    if (eq != std::string::npos) {
      val = name.substr(eq + 1);
      name = name.substr(0, eq);
    } else {
      if (i + 1 >= argc) throw UsageError("--" + name + " requires an argument");
      val = argv[++i];
    }
    bool ok = false;
    for (const auto& k : known) ok |= (k == name);
    if (!ok) throw UsageError("unknown option: --" + name);
    p.opts[name] = val;
  }
  return p;
}

std::int64_t to_i64(const std::string& name, const std::string& v, std::int64_t lo, std::int64_t hi) {
  char* end = nullptr;
  const long long x = std::strtoll(v.c_str(), &end, 10);
  if (v.empty() || *end) throw UsageError("--" + name + ": not an integer: " + v);
  if (x < lo || x > hi)
    throw UsageError("--" + name + ": value " + v + " not in range [" + std::to_string(lo) + " - " +
                     std::to_string(hi) + "]");
  return x;
}

double to_f64(const std::string& name, const std::string& v, double lo, double hi) {
  char* end = nullptr;
  const double x = std::strtod(v.c_str(), &end);
  if (v.empty() || *end) throw UsageError("--" + name + ": not a number: " + v);
  if (!(x >= lo && x <= hi)) throw UsageError("--" + name + ": value " + v + " out of range");
  return x;
}

void apply_mt(CommonArgs& a, const Parsed& p) {
  if (const char* env = std::getenv("TENSORLOOM_MT"); env && !p.opts.count("mt"))
    a.mt = (int)to_i64("mt", env, 1, 64);
  if (p.opts.count("mt")) a.mt = (int)to_i64("mt", p.opts.at("mt"), 1, 64);
}

void apply_mode(const Parsed& p) {
  if (!p.opts.count("mode")) return;
  const std::string m = p.opts.at("mode");
  if (m != "exact" && m != "fast") throw UsageError("--mode: expected exact or fast, got " + m);
  setenv("TLOOM_B200_MODE", m.c_str(), 1);
}

std::string required(const Parsed& p, const std::string& name) {
  if (!p.opts.count(name)) throw UsageError("--" + name + " is required");
  return p.opts.at(name);
}

void apply_test(CommonArgs& a, const Parsed& p) {
  a.test_images = required(p, "test-images");
  a.test_labels = required(p, "test-labels");
  if (p.opts.count("limit-test")) a.limit_test = to_i64("limit-test", p.opts.at("limit-test"), -1, std::int64_t{1} << 40);
}

void apply_train(CommonArgs& a, const Parsed& p) {
  a.train_images = required(p, "train-images");
  a.train_labels = required(p, "train-labels");
  apply_test(a, p);
  if (p.opts.count("limit-train"))
    a.limit_train = to_i64("limit-train", p.opts.at("limit-train"), -1, std::int64_t{1} << 40);
  if (p.opts.count("epochs")) a.epochs = (int)to_i64("epochs", p.opts.at("epochs"), 0, 1000000);
  if (p.opts.count("batch")) a.batch = to_i64("batch", p.opts.at("batch"), 1, std::int64_t{1} << 40);
  if (p.opts.count("rate")) a.rate = (float)to_f64("rate", p.opts.at("rate"), 1e-9, 1e9);
  if (p.opts.count("seed")) {
    const std::string v = p.opts.at("seed");
    char* end = nullptr;
    a.seed = std::strtoull(v.c_str(), &end, 10);
    if (v.empty() || *end) throw UsageError("--seed: not an integer: " + v);
  }
  apply_mt(a, p);
}

// --- workloads (proj/tools/tensorloom_cli.cpp:77-180) ----------------------------------------------
struct RunOutcome {
  tloom::net::Params params;
  std::vector<double> epoch_losses;
  double accuracy = 0.0;
  double seconds = 0.0;
};

RunOutcome run_workload(const CommonArgs& a, bool log_epochs) {
  const auto start = Clock::now();
  tloom::runtime::set_global_config({a.mt, tloom::runtime::ExecConfig{}.parallel_threshold});
  std::fprintf(stderr, "workers %d\n", a.mt);
  std::fprintf(stderr, "loading %s\n", a.train_images.c_str());
  const auto train_set = tloom::mnist::load_set(a.train_images, a.train_labels, a.limit_train);
  std::fprintf(stderr, "loading %s\n", a.test_images.c_str());
  const auto test_set = tloom::mnist::load_set(a.test_images, a.test_labels, a.limit_test);
  std::fprintf(stderr, "train %lld examples, test %lld examples\n", static_cast<long long>(train_set.size()),
               static_cast<long long>(test_set.size()));
  tloom::net::Hyper hyper;
  hyper.rate = a.rate;
  hyper.epochs = a.epochs;
  hyper.batch = a.batch;
  hyper.seed = a.seed;
  auto epoch_start = Clock::now();
  auto result = tloom::net::train(tloom::net::init_params(a.seed), train_set, hyper, [&](int epoch, double mean_loss) {
    if (log_epochs)
      std::fprintf(stderr, "epoch %d/%d mean_loss %.6f (%.1fs)\n", epoch, a.epochs, mean_loss,
                   seconds_since(epoch_start));
    epoch_start = Clock::now();
  });
  RunOutcome out;
  out.accuracy = tloom::net::evaluate(result.params, test_set);
  out.seconds = seconds_since(start);
  out.params = std::move(result.params);
  out.epoch_losses = std::move(result.epoch_mean_loss);
  return out;
}

bool params_equal(const tloom::net::Params& a, const tloom::net::Params& b) {
  using tloom::bitwise_equal;
  return bitwise_equal(a.k1, b.k1) && bitwise_equal(a.b1, b.b1) && bitwise_equal(a.k2, b.k2) &&
         bitwise_equal(a.b2, b.b2) && bitwise_equal(a.fc, b.fc) && bitwise_equal(a.b, b.b);
}

int cmd_train(const CommonArgs& a) {
  const RunOutcome out = run_workload(a, /*log_epochs=*/true);
  if (!a.checkpoint.empty()) {
    tloom::net::save_params(a.checkpoint, out.params);
    std::fprintf(stderr, "checkpoint written to %s\n", a.checkpoint.c_str());
  }
  std::printf("final_test_accuracy %.6f\n", out.accuracy);
  std::printf("total_wall_seconds %.3f\n", out.seconds);
  return 0;
}

int cmd_bench(CommonArgs a) {
  std::printf("workers,seconds,speedup_vs_1\n");
  std::fflush(stdout);
  std::optional<RunOutcome> baseline;
  for (int workers : a.bench_workers) {
    a.mt = workers;
    std::fprintf(stderr, "bench: running with %d worker(s)\n", workers);
    RunOutcome out = run_workload(a, /*log_epochs=*/false);
    const double base_seconds = baseline ? baseline->seconds : out.seconds;
    std::printf("%d,%.3f,%.3f\n", workers, out.seconds, base_seconds / out.seconds);
    std::fflush(stdout);
    if (!baseline) {
      baseline = std::move(out);
    } else if (!params_equal(baseline->params, out.params) || baseline->accuracy != out.accuracy) {
      std::fprintf(stderr, "bench: results differ across worker counts\n");
      return 4;
    }
  }
  std::fprintf(stderr, "determinism: final params identical across all worker counts\n");
  return 0;
}

int cmd_eval(const CommonArgs& a) {
  tloom::runtime::set_global_config({a.mt, tloom::runtime::ExecConfig{}.parallel_threshold});
  const auto params = tloom::net::load_params(a.checkpoint);
  const auto test_set = tloom::mnist::load_set(a.test_images, a.test_labels, a.limit_test);
  std::printf("test_accuracy %.6f\n", tloom::net::evaluate(params, test_set));
  return 0;
}

const char* kUsage =
    "tensorloom: a small CNN on a rank-polymorphic array kernel (B200 build)\n"
    "Usage: tensorloom SUBCOMMAND [OPTIONS]\n\n"
    "Subcommands:\n"
    "  train   train the digit network and report accuracy\n"
    "  bench   run the training workload per worker count, emit CSV\n"
    "  eval    evaluate a checkpoint on a test set\n\n"
    "train/bench options: --train-images F --train-labels F --test-images F --test-labels F (required)\n"
    "  --limit-train N (10000)  --limit-test N (10000)  --epochs N (10)  --batch N (100)  --rate R (0.05)\n"
    "  --seed S (42)  --mt N (1, env TENSORLOOM_MT)  --mode exact|fast (exact)\n"
    "  train: --checkpoint F    bench: --bench-workers 1,2,4,8\n"
    "eval options: --checkpoint F --test-images F --test-labels F (required)  --limit-test N  --mt N  --mode\n";

}  // namespace

int main(int argc, char** argv) {
  CommonArgs args;
  std::string sub;
  try {
    if (argc < 2) throw UsageError("A subcommand is required");
    sub = argv[1];
    if (sub == "-h" || sub == "--help") {
      std::fputs(kUsage, stdout);
      return 0;
    }
    for (int i = 2; i < argc; ++i)
      if (std::string(argv[i]) == "-h" || std::string(argv[i]) == "--help") {
        std::fputs(kUsage, stdout);
        return 0;
      }
    const std::vector<std::string> common = {"train-images", "train-labels", "test-images", "test-labels",
                                             "limit-train",  "limit-test",   "epochs",      "batch",
                                             "rate",         "seed",         "mt",          "mode"};
    if (sub == "train") {
      auto known = common;
      known.push_back("checkpoint");
      const Parsed p = parse_opts(argc, argv, 2, known);
      apply_train(args, p);
      apply_mode(p);
      if (p.opts.count("checkpoint")) args.checkpoint = p.opts.at("checkpoint");
    } else if (sub == "bench") {
      auto known = common;
      known.push_back("bench-workers");
      const Parsed p = parse_opts(argc, argv, 2, known);
      apply_train(args, p);
      apply_mode(p);
      if (p.opts.count("bench-workers")) {
        args.bench_workers.clear();
        std::string v = p.opts.at("bench-workers");
        size_t pos = 0;
        while (pos <= v.size()) {
          const size_t c = v.find(',', pos);
          const std::string tok = v.substr(pos, c == std::string::npos ? std::string::npos : c - pos);
          args.bench_workers.push_back((int)to_i64("bench-workers", tok, 1, 64));
          if (c == std::string::npos) break;
          pos = c + 1;
        }
      }
    } else if (sub == "eval") {
      const Parsed p = parse_opts(argc, argv, 2, {"checkpoint", "test-images", "test-labels", "limit-test", "mt", "mode"});
      args.checkpoint = required(p, "checkpoint");
      apply_test(args, p);
      apply_mt(args, p);
      apply_mode(p);
    } else {
      throw UsageError("The following argument was not expected: " + sub);
    }
  } catch (const UsageError& e) {
    std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.what());
    return 2;
  }

  try {
    if (sub == "train") return cmd_train(args);
    if (sub == "bench") return cmd_bench(args);
    return cmd_eval(args);
  } catch (const tloom::FormatError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 4;
  }
}
