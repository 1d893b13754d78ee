// intergrams/pipeline.hpp — the CountingOptions of
// /root/reference/proj/include/intergrams/pipeline.hpp:19-25.  The reference's
// worker pipeline itself is replaced by the GPU; the options are accepted for
// API parity and never change results (tests/test_dense_pass.cpp:141-161).
#pragma once

#include <cstddef>

#include "intergrams/counting.hpp"

namespace intergrams {

struct CountingOptions {
  CountMode mode = CountMode::kOnce;
  MergeStrategy merge = MergeStrategy::kBatchedFlush;
  size_t workers = 1;
  size_t flush_batch_size = 8;
  size_t queue_capacity = 0;
};

}  // namespace intergrams
