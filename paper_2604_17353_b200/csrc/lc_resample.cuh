// Internal interface between the C-ABI files and the resample kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lc_b200.h"

namespace lcb {
int64_t workspace_bytes(int64_t n_tasks, int64_t vocab);
int resample_launch(const void* rows, int dtype, int64_t vocab, int64_t row_stride, const lc_task* tasks,
                    int64_t n_tasks, lc_draws draws, const int32_t* pages, int max_pages, int page_rows, void* ws,
                    int64_t ws_bytes, int64_t* counters, cudaStream_t st);
}  // namespace lcb
