// K0 — compact-AST builder over a flattened forest.
//
// Replaces the host tree walk build_compact_ast + compute_vector
// (features.py:155-245): for every program of a forest stored as pre-order
// node arrays it writes the marker-annotated pre-order serialization, the
// leaf ordering (serialized position of every leaf) and the 24-entry
// computation vector of every leaf — the CompactAst fields — straight into
// the ragged SoA that K1 (tpcb_featurize_pack) consumes.
//
// Layout (all device, caller-owned; see include/tpcb200.h):
//   node_off [P+1] i64   node range of program p (pre-order, local ids 0..)
//   parent   [N]   i32   local index of the parent loop, -1 for the root
//   extent   [N]   i64   loop extent (>= 1); 0 marks a compute leaf
//   annot    [N]   u8    bit 0 vectorize, 1 unroll, 2 parallel
//   leaf_off [P+1] i64   leaf range of program p (leaves in pre-order)
//   stats    [NL,9] i64  fma add mul div special bytes_read bytes_written
//                        buffers_read buffers_written (ir.py:53-64)
// Outputs: vectors [NL,24] f64, ordering [NL] i32,
//          serialized [N+NL] i32 at offset node_off[p] + leaf_off[p].
//
// One warp per program: lanes take 32 nodes at a time; a ballot over
// "is leaf" gives every node its serialized position (node id + markers
// before it) and every leaf its leaf index, and the lane holding a leaf walks
// its parent chain (depth <= 64, ir.py:49) to form the enclosing-loop
// aggregates.  Integer products are exact in 128 bits (counts are limited to
// < 2^56 and extents to < 2^63 by the host validation), so the 2^62 overflow
// guard of _log_extent_product (features.py:158-169) is exact, and every
// int -> float conversion and the intensity quotient (entry 22, a Python
// int/int true division) are correctly rounded like CPython's.  log2 is the
// CUDA libdevice log2 (<= 1 ulp), the only non-bit-exact step.

#include <algorithm>

#include "common.cuh"

namespace tpcb {
namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ int bitlen128(u128 v) {
  const uint64_t hi = (uint64_t)(v >> 64), lo = (uint64_t)v;
  return hi ? 128 - __clzll((long long)hi) : (lo ? 64 - __clzll((long long)lo) : 0);
}

// correctly rounded (nearest-even) conversion, like CPython's PyLong_AsDouble
__device__ double u128_to_double(u128 v) {
  const int n = bitlen128(v);
  if (n <= 64) return __ull2double_rn((unsigned long long)v);
  const int sh = n - 64;
  uint64_t m = (uint64_t)(v >> sh);
  if ((v & ((((u128)1) << sh) - 1)) != 0) m |= 1;  // sticky below 11 guard bits
  return ldexp(__ull2double_rn(m), sh);
}

// correctly rounded a / b for integers (CPython long_true_divide), b > 0
__device__ double div_u128(u128 a, u128 b) {
  if (a == 0) return 0.0;
  if ((a >> 53) == 0 && (b >> 53) == 0) return (double)(uint64_t)a / (double)(uint64_t)b;
  const int e = bitlen128(a) - bitlen128(b);
  u128 r = a, D = b;
  if (e >= 0) D <<= e; else r <<= -e;  // same bit length now; r / D in (1/2, 2)
  uint64_t q = 0;
  for (int i = 0; i < 56; ++i) {  // 55-56 significant quotient bits
    q <<= 1;
    if (r >= D) { r -= D; q |= 1; }
    r <<= 1;
  }
  if (r != 0) q |= 1;  // sticky (>= 2 guard bits below the 53-bit mantissa)
  return ldexp(__ull2double_rn(q), e - 55);
}

__device__ __forceinline__ double log2_1p_int(u128 v) { return log2(u128_to_double(v + 1)); }

constexpr u128 kProductLimit = ((u128)1) << 62;  // features.py:26

struct CompactOut {
  double* vectors;
  int32_t* ordering;
  int32_t* serialized;
  unsigned long long* first_bad;  // min program index that overflowed
};

__global__ void __launch_bounds__(256) build_compact_kernel(
    const int64_t* __restrict__ node_off, const int32_t* __restrict__ parent,
    const int64_t* __restrict__ extent, const uint8_t* __restrict__ annot,
    const int64_t* __restrict__ leaf_off, const int64_t* __restrict__ stats, int64_t n_prog,
    CompactOut out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < n_prog;
       p += warps) {
    const int64_t n0 = node_off[p], nn = node_off[p + 1] - n0;
    const int64_t l0 = leaf_off[p];
    const int n_leaf = (int)(leaf_off[p + 1] - l0);
    const int64_t s0 = n0 + l0;
    int before = 0;  // leaves in earlier chunks
    for (int64_t c = 0; c < nn; c += 32) {
      const int64_t i = c + lane;
      const bool valid = i < nn;
      const int64_t ext = valid ? extent[n0 + i] : 1;
      const bool is_leaf = valid && ext == 0;
      const unsigned ball = __ballot_sync(0xffffffffu, is_leaf);
      const int k = before + __popc(ball & ((1u << lane) - 1u));  // leaf index
      if (valid) {
        const int64_t pos = i + k;  // node id + markers emitted before it
        out.serialized[s0 + pos] = (int32_t)i;
        if (is_leaf) out.serialized[s0 + pos + 1] = -1;  // MARKER
      }
      if (is_leaf) {
        out.ordering[l0 + k] = (int32_t)(i + k);
        // enclosing loops: parent chain, innermost first
        int depth = 0;
        u128 prod = 1, tprod[3] = {1, 1, 1};
        int tcount[3] = {0, 0, 0};
        int64_t inner = 0, outer = 0;
        bool overflow = false;
        for (int32_t a = parent[n0 + i]; a >= 0; a = parent[n0 + a]) {
          const int64_t e = extent[n0 + a];
          const unsigned bits = annot[n0 + a];
          if (depth == 0) inner = e;
          outer = e;
          ++depth;
          prod *= (u128)e;
          if (prod > kProductLimit) overflow = true;
          if (overflow) prod = kProductLimit;  // keep the walk well-defined
          for (int t = 0; t < 3; ++t)
            if (bits >> t & 1u) { ++tcount[t]; tprod[t] *= (u128)e; if (tprod[t] > kProductLimit) tprod[t] = kProductLimit; }
        }
        if (overflow) atomicMin(out.first_bad, (unsigned long long)p);
        const int64_t* st = stats + (l0 + k) * 9;
        double* v = out.vectors + (l0 + k) * TPCB_FEAT;
        const u128 iters = depth ? prod : (u128)1;
        v[0] = (double)depth;
        v[1] = depth ? log2_1p_int(prod) : 0.0;
        v[2] = depth ? log2_1p_int((u128)inner) : 0.0;
        v[3] = depth ? log2_1p_int((u128)outer) : 0.0;
        for (int t = 0; t < 3; ++t) {
          v[4 + t] = (double)tcount[t];
          v[7 + t] = tcount[t] ? log2_1p_int(tprod[t]) : 0.0;
        }
        u128 per_iter = 2 * (u128)st[0];
        for (int t = 0; t < 5; ++t) {
          v[10 + t] = log2_1p_int((u128)st[t]);
          if (t) per_iter += (u128)st[t];
        }
        const u128 tot_flops = per_iter * iters;
        const u128 tot_read = (u128)st[5] * iters, tot_written = (u128)st[6] * iters;
        v[15] = log2_1p_int(tot_flops);
        v[16] = log2_1p_int((u128)st[5]);
        v[17] = log2_1p_int((u128)st[6]);
        v[18] = log2_1p_int(tot_read);
        v[19] = log2_1p_int(tot_written);
        v[20] = u128_to_double((u128)st[7]);
        v[21] = u128_to_double((u128)st[8]);
        v[22] = div_u128(tot_flops, tot_read + tot_written + 1);
        v[23] = (double)k / (double)n_leaf;
      }
      before += __popc(ball);
    }
  }
}

}  // namespace
}  // namespace tpcb

extern "C" int tpcb_build_compact(const int64_t* d_node_off, const int32_t* d_parent,
                                  const int64_t* d_extent, const uint8_t* d_annot,
                                  const int64_t* d_leaf_off, const int64_t* d_stats,
                                  int64_t n_prog, double* d_vectors, int32_t* d_ordering,
                                  int32_t* d_serialized, unsigned long long* d_first_overflow,
                                  void* stream) {
  if (n_prog < 0 || !d_first_overflow) return TPCB_ERR_VALIDATION;
  cudaStream_t s = (cudaStream_t)stream;
  TPCB_CUDA_CHECK(cudaMemsetAsync(d_first_overflow, 0xff, sizeof(unsigned long long), s));
  if (n_prog == 0) return TPCB_OK;
  int dev = 0, sms = 148;
  TPCB_CUDA_CHECK(cudaGetDevice(&dev));
  TPCB_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t blocks_needed = (n_prog + 7) / 8;  // 8 warps per block
  const int blocks = (int)std::min<int64_t>(blocks_needed, (int64_t)sms * 8);
  tpcb::CompactOut out{d_vectors, d_ordering, d_serialized, d_first_overflow};
  tpcb::build_compact_kernel<<<blocks, 256, 0, s>>>(d_node_off, d_parent, d_extent, d_annot,
                                                     d_leaf_off, d_stats, n_prog, out);
  TPCB_LAUNCH_CHECK("build_compact_kernel");
  return TPCB_OK;
}
