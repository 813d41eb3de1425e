// Internal interface of the NCCL gradient exchange (dpb_comm.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dpb {
struct Comm;
// In-place average allreduce of n fp32 values on `st` (ncclAvg).
int comm_allreduce_avg(Comm* c, float* buf, int64_t n, cudaStream_t st);
int comm_ranks(const Comm* c);
}  // namespace dpb
