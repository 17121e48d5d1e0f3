// NCCL communicator handle shared by dist.cu and the training loop.
#pragma once

#include <nccl.h>

#include "common.cuh"

struct tpcb_comm {
  ncclComm_t comm;
  int rank, nranks;
};

namespace tpcb {
int allreduce_sum(tpcb_comm* c, void* buf, int64_t count, int is_f64, cudaStream_t stream);
int group_start();
int group_end();
}  // namespace tpcb
