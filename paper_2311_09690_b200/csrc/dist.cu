// NCCL plumbing for data-parallel training (one process per GPU).  The
// communicator is created from a unique id the host broadcasts through
// torch.distributed; the epoch loop (capi_train.cu) issues its all-reduces
// on the training stream, so they are captured into the epoch graph with
// the kernels around them.
#include <nccl.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "dist.cuh"

using namespace tpcb;

extern "C" int tpcb_nccl_unique_id(void* out, int32_t cap) {
  if (!out || cap < (int32_t)sizeof(ncclUniqueId)) return TPCB_ERR_VALIDATION;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return TPCB_ERR_CUDA;
  memcpy(out, &id, sizeof(id));
  return TPCB_OK;
}

extern "C" int tpcb_nccl_comm_create(const void* id, int32_t nranks, int32_t rank,
                                     tpcb_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return TPCB_ERR_VALIDATION;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  tpcb_comm* c = new tpcb_comm();
  c->rank = rank;
  c->nranks = nranks;
  if (ncclCommInitRank(&c->comm, nranks, uid, rank) != ncclSuccess) {
    delete c;
    return TPCB_ERR_CUDA;
  }
  *out = c;
  return TPCB_OK;
}

extern "C" void tpcb_nccl_comm_destroy(tpcb_comm* c) {
  if (!c) return;
  ncclCommDestroy(c->comm);
  if (c->gather) cudaFree(c->gather);
  delete c;
}

namespace tpcb {

int allreduce_sum(tpcb_comm* c, void* buf, int64_t count, int is_f64, cudaStream_t stream) {
  if (!c) return TPCB_OK;
  ncclResult_t r = ncclAllReduce(buf, buf, (size_t)count, is_f64 ? ncclFloat64 : ncclFloat32,
                                 ncclSum, c->comm, stream);
  return r == ncclSuccess ? TPCB_OK : TPCB_ERR_CUDA;
}

namespace {
__global__ void ordered_sum_kernel(const float* __restrict__ g, int nranks, int64_t count,
                                   float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = g[i];
    for (int r = 1; r < nranks; ++r) s += g[(int64_t)r * count + i];
    out[i] = s;
  }
}
}  // namespace

int ensure_gather(tpcb_comm* c, int64_t count) {
  if (!c || c->nranks < 2 || count <= c->gather_cap) return TPCB_OK;
  if (c->gather) TPCB_CUDA_CHECK(cudaFree(c->gather));
  c->gather = nullptr;
  TPCB_CUDA_CHECK(cudaMalloc(&c->gather, (size_t)c->nranks * count * sizeof(float)));
  c->gather_cap = count;
  return TPCB_OK;
}

int ordered_allreduce_sum(tpcb_comm* c, float* buf, int64_t count, cudaStream_t stream) {
  if (!c || c->nranks < 2) return TPCB_OK;  // one rank: the local gradient is the sum
  if (count > c->gather_cap) return TPCB_ERR_VALIDATION;  // ensure_gather before capture
  if (ncclAllGather(buf, c->gather, (size_t)count, ncclFloat32, c->comm, stream) != ncclSuccess)
    return TPCB_ERR_CUDA;
  const int grid = (int)std::min<int64_t>((count + 255) / 256, (int64_t)kNumSMs * 4);
  ordered_sum_kernel<<<grid, 256, 0, stream>>>(c->gather, c->nranks, count, buf);
  TPCB_LAUNCH_CHECK("ordered_sum");
  return TPCB_OK;
}

int group_start() { return ncclGroupStart() == ncclSuccess ? TPCB_OK : TPCB_ERR_CUDA; }
int group_end() { return ncclGroupEnd() == ncclSuccess ? TPCB_OK : TPCB_ERR_CUDA; }

}  // namespace tpcb

extern "C" int tpcb_nccl_allreduce_sum(tpcb_comm* c, void* d_buf, int64_t count, int32_t is_f64,
                                       void* stream) {
  return allreduce_sum(c, d_buf, count, is_f64, (cudaStream_t)stream);
}
