// runtime.cpp -- host execution settings (include/tloom/runtime.hpp).
// Semantics follow the reference scheduler (proj/src/runtime.cpp): ceil-block static chunks, caller runs
// chunk 0, nested regions run inline, lowest failing chunk's exception wins.  The training path does not
// use it: batches run on the GPU grid.
#include "tloom/runtime.hpp"

#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>

#include "tloom/errors.hpp"

namespace tloom::runtime {

namespace {

thread_local bool t_in_region = false;

struct RegionGuard {
  bool saved;
  RegionGuard() : saved(t_in_region) { t_in_region = true; }
  ~RegionGuard() { t_in_region = saved; }
};

ExecConfig from_env() {
  ExecConfig cfg;
  if (const char* v = std::getenv("TENSORLOOM_MT")) {
    char* end = nullptr;
    const long w = std::strtol(v, &end, 10);
    if (end != v && *end == '\0' && w >= 1) cfg.workers = static_cast<int>(w);
  }
  return cfg;
}

std::mutex& cfg_mutex() {
  static std::mutex m;
  return m;
}

ExecConfig& cfg_store() {
  static ExecConfig cfg = from_env();
  return cfg;
}

}  // namespace

ExecConfig global_config() {
  std::lock_guard<std::mutex> lk(cfg_mutex());
  return cfg_store();
}

void set_global_config(const ExecConfig& cfg) {
  if (cfg.workers < 1) throw Error("ExecConfig: workers must be >= 1");
  if (cfg.parallel_threshold < 0) throw Error("ExecConfig: parallel_threshold must be >= 0");
  std::lock_guard<std::mutex> lk(cfg_mutex());
  cfg_store() = cfg;
}

std::pair<std::int64_t, std::int64_t> static_chunk(std::int64_t n, int workers, int w) {
  if (n < 0 || workers < 1 || w < 0 || w >= workers) throw Error("static_chunk: invalid arguments");
  const std::int64_t block = (n + workers - 1) / workers;
  const std::int64_t lo = std::min<std::int64_t>(static_cast<std::int64_t>(w) * block, n);
  return {lo, std::min<std::int64_t>(lo + block, n)};
}

bool inside_parallel_region() { return t_in_region; }

void run_static(std::int64_t n, const ExecConfig& cfg, const std::function<void(std::int64_t, std::int64_t)>& body) {
  if (cfg.workers < 1) throw Error("run_static: workers must be >= 1");
  if (n <= 0) return;
  if (cfg.workers == 1 || n < cfg.parallel_threshold || t_in_region) {
    body(0, n);
    return;
  }
  std::vector<std::exception_ptr> errs(static_cast<std::size_t>(cfg.workers));
  auto chunk = [&](int w) {
    const auto [lo, hi] = static_chunk(n, cfg.workers, w);
    if (lo >= hi) return;
    RegionGuard g;
    try {
      body(lo, hi);
    } catch (...) {
      errs[static_cast<std::size_t>(w)] = std::current_exception();
    }
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < cfg.workers; ++w) pool.emplace_back(chunk, w);
  chunk(0);
  for (auto& t : pool) t.join();
  for (auto& e : errs)  // chunks are ordered by index: the first stored error is the lowest chunk's
    if (e) std::rethrow_exception(e);
}

std::vector<float> parallel_build(std::int64_t frame_count, std::int64_t cell_size, const ExecConfig& cfg,
                                  const std::function<void(std::int64_t, float*)>& elem) {
  if (frame_count < 0 || cell_size < 0) throw Error("parallel_build: negative extent");
  std::vector<float> out(static_cast<std::size_t>(frame_count * cell_size));
  run_static(frame_count, cfg, [&](std::int64_t lo, std::int64_t hi) {
    for (std::int64_t i = lo; i < hi; ++i) elem(i, out.data() + i * cell_size);
  });
  return out;
}

}  // namespace tloom::runtime
