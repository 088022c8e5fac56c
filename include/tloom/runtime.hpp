// tloom/runtime.hpp -- execution settings of the tensorloom API (B200 build).
//
// Source-compatible with the reference scheduler interface (proj/include/tloom/runtime.hpp:15-48).
// In the reference, `workers` sets how many CPU threads run the example-parallel batch step.  Here the
// batch step runs on the GPU (CTA grid of the persistent train kernel; results are bitwise identical for
// every setting, as in the reference), so ExecConfig only drives the host-side generic comprehension
// helpers of tloom/tensor.hpp.
#pragma once

#include <cstdint>
#include <functional>
#include <utility>
#include <vector>

namespace tloom::runtime {

struct ExecConfig {
  int workers = 1;
  std::int64_t parallel_threshold = 4096;
};

// Process-wide default; TENSORLOOM_MT seeds `workers` once at start-up.
ExecConfig global_config();
void set_global_config(const ExecConfig& cfg);

// [lo, hi) owned by worker w of `workers` over n items: ceil-sized blocks, trailing blocks may be empty.
std::pair<std::int64_t, std::int64_t> static_chunk(std::int64_t n, int workers, int w);

bool inside_parallel_region();

// body(lo, hi) over a static partition of [0, n); sequential for workers <= 1, n < threshold or when
// nested.  If several chunks throw, the lowest chunk's exception is rethrown after all finish.
void run_static(std::int64_t n, const ExecConfig& cfg,
                const std::function<void(std::int64_t, std::int64_t)>& body);

// frame_count * cell_size floats; element i fills [i*cell_size, (i+1)*cell_size).
std::vector<float> parallel_build(std::int64_t frame_count, std::int64_t cell_size, const ExecConfig& cfg,
                                  const std::function<void(std::int64_t, float*)>& elem);

}  // namespace tloom::runtime
