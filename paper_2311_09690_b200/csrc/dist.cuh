// NCCL communicator handle shared by dist.cu and the training loop.
#pragma once

#include <nccl.h>

#include "common.cuh"

struct tpcb_comm {
  ncclComm_t comm;
  int rank, nranks;
  // [nranks * gather_cap] floats: the rank-ordered gradient reduction's
  // all-gather buffer (allocated outside graph capture, ensure_gather)
  float* gather = nullptr;
  int64_t gather_cap = 0;
};

namespace tpcb {
int allreduce_sum(tpcb_comm* c, void* buf, int64_t count, int is_f64, cudaStream_t stream);
// sum of every rank's `buf` added in rank order (r = 0, 1, ...): all-gather
// + one ordered-sum kernel, so the reduced gradient does not depend on the
// collective algorithm NCCL picks (ring / tree / NVLS) — the same
// fixed-order rule the point-sharded KMeans follows (sampling.py)
int ensure_gather(tpcb_comm* c, int64_t count);
int ordered_allreduce_sum(tpcb_comm* c, float* buf, int64_t count, cudaStream_t stream);
int group_start();
int group_end();
}  // namespace tpcb
