// Shared helpers of libfse_b200: thread-local error reporting and the plan type.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/fse_b200.h"

namespace fse {

void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

// Per-frame plan produced by the host scheduler (fse_plan.cpp) and consumed by
// the device pipeline (fse_cuda.cu).
struct Plan {
    int32_t H = 0, W = 0, B = 1, rows = 0, cols = 0, d = 0, order = 0;
    int32_t iterations = 0, fft1 = 0, fft2 = 0;
    double rho = 0.8, delta = 0.2, gamma = 0.5;
    int32_t n_lossy = 0, n_processed = 0;
    int32_t max_wr = 0, max_wc = 0;  // largest window (clipped) rows / cols
    std::vector<int32_t> rank;       // effective rank per block, INT32_MAX = never written
    std::vector<int32_t> batch_ptr, batch_blocks;  // ConcealReport.batches
    std::vector<int32_t> level_ptr, level_blocks;  // dependency levels
    std::vector<int32_t> unconcealed;
};

}  // namespace fse

struct FsePlan {
    fse::Plan p;
};
