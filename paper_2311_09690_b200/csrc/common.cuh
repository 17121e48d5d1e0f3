// Shared definitions for the tpcb200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/tpcb200.h"

namespace tpcb {

// Offsets (in floats) of every tensor of one encoder layer inside the flat
// parameter vector.  Order of creation follows costmodel.py:130-140.
struct LayerOff {
  int Wq, Wk, Wv, Wo, bq, bk, bv, bo;
  int ln1g, ln1b, fhW, fhb, foW, fob, ln2g, ln2b;
};

// Device-visible model description: dims + canonical tensor offsets.
// Passed to kernels by value (~1.3 KB, below the 4 KB parameter limit).
struct Model {
  int d, n_layers, n_heads, dh, d_ff, d_e, d_dev, n_dec, n_leaf_max;
  int dec[TPCB_MAX_DEC];
  int inW, inb;
  LayerOff layer[TPCB_MAX_LAYERS];
  int leafW[TPCB_MAX_LEAF + 1], leafb[TPCB_MAX_LEAF + 1];
  int devhW, devhb, devpW, devpb;
  int decW[TPCB_MAX_DEC], decb[TPCB_MAX_DEC];
  int outW, outb;
  int total;
  // first / last+1 float of the tensors touched by every batch regardless of
  // its leaf count (everything except leaf_embed.*) — see optim.cu
  int shared_lo, shared_hi;  // [inW, leafW[1])
  int tail_lo;               // devhW .. total
};

// 2-D tensors of the flat parameter vector (for the transposed copy)
constexpr int kMaxT2 = 160;
struct T2Table {
  int n;
  int off[kMaxT2], rows[kMaxT2], cols[kMaxT2], cum[kMaxT2 + 1];
};

struct TensorInfo {
  std::string name;
  int64_t offset;
  int rows, cols;
};

}  // namespace tpcb

struct tpcb_model {
  tpcb_config cfg;
  tpcb::Model dev;
  tpcb::T2Table t2;
  std::vector<tpcb::TensorInfo> tensors;
};

namespace tpcb {

void set_last_error(const char* what, cudaError_t e);

// Developer A/B switches, read once from the environment on first use and
// immutable afterwards (no process-global state a caller can flip while
// another thread trains): TPCB_TRAIN_IMPL (0 automatic, 2 generic kernel,
// 4 desk fast path), TPCB_GRID_CAP (cap on the training grid), TPCB_POLL_NS
// (stage-wait poll interval of the overlapped reduce), TPCB_GEMM_BK (16 / 32
// k-slab of the large-path GEMM), TPCB_GEMM_CLUSTER, TPCB_GEMM_MODE (probe),
// TPCB_WGRAD_TC (0: encoder weight gradients in the per-sample slots).
struct Knobs {
  int train_impl, grid_cap, gemm_bk, gemm_cluster, gemm_mode;
  unsigned poll_ns;
  int wgrad_tc;  // TPCB_WGRAD_TC (default 1): encoder weight gradients on tcgen05
};
const Knobs& knobs();

#define TPCB_CUDA_CHECK(call)                              \
  do {                                                     \
    cudaError_t _e = (call);                               \
    if (_e != cudaSuccess) {                               \
      ::tpcb::set_last_error(#call, _e);                   \
      return TPCB_ERR_CUDA;                                \
    }                                                      \
  } while (0)

#define TPCB_LAUNCH_CHECK(what)                            \
  do {                                                     \
    cudaError_t _e = cudaGetLastError();                   \
    if (_e != cudaSuccess) {                               \
      ::tpcb::set_last_error(what, _e);                    \
      return TPCB_ERR_CUDA;                                \
    }                                                      \
  } while (0)

// device status word: first error wins (atomicCAS from 0)
__device__ __forceinline__ void raise_status(int32_t* st, int32_t code) {
  if (st) atomicCAS(st, 0, code);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

constexpr int kNumSMs = 148;

}  // namespace tpcb
