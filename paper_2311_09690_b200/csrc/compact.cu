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
// int/int true division) are correctly rounded like CPython's.  log2 of
// arguments below 4096 is the host libm's own value (a table); above, the
// CUDA libdevice log2 (<= 1 ulp) is the only non-bit-exact step.

#include <algorithm>
#include <cmath>
#include <mutex>

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

// log2(1 + v): small arguments (counts, extents, per-iteration bytes — 7 of
// the 13 log2 entries on typical programs) come from a table the host fills
// with its own libm log2, i.e. the very values CPython's math.log2 returns to
// the reference; larger ones use the device log2 (<= 1 ulp).
constexpr int kLog2Table = 4096;
__device__ double g_log2_table[kLog2Table];

__device__ __forceinline__ double log2_1p_int(u128 v) {
  if (v < (u128)kLog2Table) return __ldg(&g_log2_table[(int)v]);
  return log2(u128_to_double(v + 1));
}

constexpr uint64_t kProductLimit = 1ull << 62;  // features.py:26

// a * e clamped at kProductLimit, exact: a <= 2^62 and e < 2^63, so the full
// product fits 128 bits and "exceeds the limit" is hi != 0 || lo > limit
__device__ __forceinline__ uint64_t sat_mul(uint64_t a, uint64_t e, bool& over) {
  const uint64_t lo = a * e, hi = __umul64hi(a, e);
  over = hi != 0 || lo > kProductLimit;
  return over ? kProductLimit : lo;
}

__device__ __forceinline__ double log2_1p_u64(uint64_t v) {
  if (v < (uint64_t)kLog2Table) return __ldg(&g_log2_table[(int)v]);
  return log2(u128_to_double((u128)v + 1));
}

struct CompactOut {
  double* vectors;
  int32_t* ordering;
  int32_t* serialized;
  unsigned long long* first_bad;  // min program index that overflowed
};

// Enclosing-loop aggregates of one leaf from its parent chain (innermost
// first); Tree gives parent(i) / extent(i) / annot(i) in program-local ids.
struct Chain {
  int depth;
  uint64_t prod, tprod[3];  // clamped at kProductLimit (< 2^64)
  int tcount[3];
  int64_t inner, outer;
  bool overflow;
};

template <class Tree>
__device__ __forceinline__ Chain walk_chain(const Tree& t, int32_t leaf) {
  Chain c;
  c.depth = 0;
  c.prod = 1;
  c.inner = c.outer = 0;
  c.overflow = false;
  for (int q = 0; q < 3; ++q) { c.tprod[q] = 1; c.tcount[q] = 0; }
  for (int32_t a = t.parent(leaf); a >= 0; a = t.parent(a)) {
    const int64_t e = t.extent(a);
    const unsigned bits = t.annot(a);
    if (c.depth == 0) c.inner = e;
    c.outer = e;
    ++c.depth;
    bool over;
    c.prod = sat_mul(c.prod, (uint64_t)e, over);
    c.overflow |= over;
#pragma unroll
    for (int q = 0; q < 3; ++q) {  // branch-free: select the annotated products
      const bool on = bits >> q & 1u;
      const uint64_t tp = sat_mul(c.tprod[q], (uint64_t)e, over);
      c.tcount[q] += on;
      c.tprod[q] = on ? tp : c.tprod[q];
    }
  }
  return c;
}

// compute_vector (features.py:172-206) into v[0..23] (any address space)
__device__ __forceinline__ void leaf_vector(const Chain& c, const int64_t* __restrict__ st,
                                            int k, int n_leaf, double* v) {
  // stats first: st may be this leaf's own staging row (columns 16..24 of v)
  int64_t s[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) s[q] = st[q];
  const u128 iters = c.depth ? (u128)c.prod : (u128)1;
  double2* v2 = reinterpret_cast<double2*>(v);  // 16-byte aligned; pairs stored as they are ready
  const auto lg = [](uint64_t x, bool on) { return on ? log2_1p_u64(x) : 0.0; };
  v2[0] = make_double2((double)c.depth, lg(c.prod, c.depth));
  v2[1] = make_double2(lg((uint64_t)c.inner, c.depth), lg((uint64_t)c.outer, c.depth));
  v2[2] = make_double2((double)c.tcount[0], (double)c.tcount[1]);
  v2[3] = make_double2((double)c.tcount[2], lg(c.tprod[0], c.tcount[0]));
  v2[4] = make_double2(lg(c.tprod[1], c.tcount[1]), lg(c.tprod[2], c.tcount[2]));
  v2[5] = make_double2(log2_1p_u64((uint64_t)s[0]), log2_1p_u64((uint64_t)s[1]));
  v2[6] = make_double2(log2_1p_u64((uint64_t)s[2]), log2_1p_u64((uint64_t)s[3]));
  const u128 per_iter = 2 * (u128)s[0] + (u128)s[1] + (u128)s[2] + (u128)s[3] + (u128)s[4];
  const u128 tot_flops = per_iter * iters;
  const u128 tot_read = (u128)s[5] * iters, tot_written = (u128)s[6] * iters;
  v2[7] = make_double2(log2_1p_u64((uint64_t)s[4]), log2_1p_int(tot_flops));
  v2[8] = make_double2(log2_1p_u64((uint64_t)s[5]), log2_1p_u64((uint64_t)s[6]));
  v2[9] = make_double2(log2_1p_int(tot_read), log2_1p_int(tot_written));
  v2[10] = make_double2(__ull2double_rn((unsigned long long)s[7]),
                        __ull2double_rn((unsigned long long)s[8]));
  v2[11] = make_double2(div_u128(tot_flops, tot_read + tot_written + 1),
                        (double)k / (double)n_leaf);
}

struct GlobalTree {  // one program's arrays in global memory
  const int32_t* par;
  const int64_t* ext;
  const uint8_t* ann;
  __device__ int32_t parent(int32_t i) const { return par[i]; }
  __device__ int64_t extent(int32_t i) const { return ext[i]; }
  __device__ unsigned annot(int32_t i) const { return ann[i]; }
};

// Tile path (the default): a block owns kProgsPerBlock consecutive programs whose node
// arrays (one contiguous range) are staged in shared memory with coalesced
// loads; a block-wide scan of "is leaf" gives every node its serialized
// position, then one thread per leaf walks its chain in shared memory and
// writes its vector into a padded staging tile that the block streams out
// with coalesced 8-byte stores (the vectors of a block are contiguous).
constexpr int kProgsPerBlock = 64;  // (≤ 255: the node → program map is uint8)
static_assert(4 * kProgsPerBlock <= 256, "four map-filling threads per program");
constexpr int kThreads = 256;
constexpr int kNodeCap = 1280;   // nodes staged per block (3 blocks per SM; 64 programs average ~740)
constexpr int kVecPitch = 26;    // doubles per staged row: 16-byte rows, conflict-free v2 stores
constexpr int kStatsCol = 16;    // prefetched stats (9 × int64) at columns 16..24 of a row

struct SmemTree {  // block-local ids; base = first node of the program
  const int16_t* par;
  const int64_t* ext;
  const uint8_t* ann;
  int base;
  __device__ int32_t parent(int32_t i) const {
    return par[base + i];
  }
  __device__ int64_t extent(int32_t i) const { return ext[base + i]; }
  __device__ unsigned annot(int32_t i) const { return ann[base + i]; }
};

struct TileSmem {
  int64_t ext[kNodeCap];
  double vec[kThreads * kVecPitch];
  int16_t par[kNodeCap];
  int16_t leaf_node[kNodeCap];  // block-local node of block-local leaf g
  int64_t node_off[kProgsPerBlock + 1], leaf_off[kProgsPerBlock + 1];
  int warp_sum[kThreads / 32];
  uint8_t ann[kNodeCap];
  uint8_t prog[kNodeCap];  // block-local program of every staged node
};


// warp-per-program path for blocks whose programs exceed the node cap
__device__ void program_warp(const int64_t* __restrict__ node_off,
                             const int32_t* __restrict__ parent,
                             const int64_t* __restrict__ extent,
                             const uint8_t* __restrict__ annot,
                             const int64_t* __restrict__ leaf_off,
                             const int64_t* __restrict__ stats, int64_t p, const CompactOut& out) {
  const int lane = threadIdx.x & 31;
  const int64_t n0 = node_off[p], nn = node_off[p + 1] - n0;
  const int64_t l0 = leaf_off[p];
  const int n_leaf = (int)(leaf_off[p + 1] - l0);
  const int64_t s0 = n0 + l0;
  const GlobalTree tree{parent + n0, extent + n0, annot + n0};
  int before = 0;
  for (int64_t c = 0; c < nn; c += 32) {
    const int64_t i = c + lane;
    const bool valid = i < nn;
    const bool is_leaf = valid && extent[n0 + i] == 0;
    const unsigned ball = __ballot_sync(0xffffffffu, is_leaf);
    const int k = before + __popc(ball & ((1u << lane) - 1u));
    if (valid) {
      out.serialized[s0 + i + k] = (int32_t)i;
      if (is_leaf) out.serialized[s0 + i + k + 1] = -1;
    }
    if (is_leaf) {
      out.ordering[l0 + k] = (int32_t)(i + k);
      const Chain ch = walk_chain(tree, (int32_t)i);
      if (ch.overflow) atomicMin(out.first_bad, (unsigned long long)p);
      leaf_vector(ch, stats + (l0 + k) * 9, k, n_leaf, out.vectors + (l0 + k) * TPCB_FEAT);
    }
    before += __popc(ball);
  }
}

__global__ void __launch_bounds__(kThreads, 3) build_compact_kernel(
    const int64_t* __restrict__ node_off, const int32_t* __restrict__ parent,
    const int64_t* __restrict__ extent, const uint8_t* __restrict__ annot,
    const int64_t* __restrict__ leaf_off, const int64_t* __restrict__ stats, int64_t n_prog,
    CompactOut out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t p0 = (int64_t)blockIdx.x * kProgsPerBlock;
  const int np = (int)(n_prog - p0 < kProgsPerBlock ? n_prog - p0 : kProgsPerBlock);
  if (t <= np) {
    sm.node_off[t] = node_off[p0 + t];
    sm.leaf_off[t] = leaf_off[p0 + t];
  }
  __syncthreads();
  const int64_t gn0 = sm.node_off[0], gl0 = sm.leaf_off[0];
  const int nodes = (int)(sm.node_off[np] - gn0);
  const int leaves = (int)(sm.leaf_off[np] - gl0);
  if (nodes > kNodeCap) {  // oversized programs: warp per program from global memory
    for (int q = warp; q < np; q += kThreads / 32)
      program_warp(node_off, parent, extent, annot, leaf_off, stats, p0 + q, out);
    return;
  }
  // stage the node arrays (coalesced), parents as block-local indices: four
  // nodes per thread per round with every load issued before any store
  for (int j0 = t; j0 < nodes; j0 += 4 * kThreads) {
    int64_t e[4];
    int32_t pa[4];
    uint8_t an[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * kThreads;
      if (j < nodes) {
        e[u] = extent[gn0 + j];
        an[u] = annot[gn0 + j];
        pa[u] = parent[gn0 + j];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * kThreads;
      if (j < nodes) {
        sm.ext[j] = e[u];
        sm.ann[j] = an[u];
        sm.par[j] = (int16_t)pa[u];  // local ids
      }
    }
  }
  // this block's first 256 leaf stats rows → columns 16..24 of the staging
  // rows of the threads that will own them (coalesced 8-byte cp.async; each
  // thread reads its own row's stats before it writes the vector over them)
  const int pre = min(leaves, kThreads) * 9;
  for (int e = t; e < pre; e += kThreads) {
    const int r = e / 9, q = e - r * 9;
    const unsigned dst = (unsigned)__cvta_generic_to_shared(sm.vec + r * kVecPitch + kStatsCol + q);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst),
                 "l"(stats + (gl0 * 9 + e)) : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  {  // node → program map (replaces a binary search per node and per leaf):
     // four threads per program, interleaved over its nodes
    const int q = t >> 2;
    if (q < np) {
      const int j0 = (int)(sm.node_off[q] - gn0), j1 = (int)(sm.node_off[q + 1] - gn0);
      for (int j = j0 + (t & 3); j < j1; j += 4) sm.prog[j] = (uint8_t)q;
    }
  }
  // block-wide exclusive scan of is_leaf, 256 nodes per round
  int carry = 0;
  for (int c = 0; c < nodes; c += kThreads) {
    const int j = c + t;
    const bool is_leaf = j < nodes && sm.ext[j] == 0;
    const unsigned ball = __ballot_sync(0xffffffffu, is_leaf);
    if (lane == 0) sm.warp_sum[warp] = __popc(ball);
    __syncthreads();
    int before = carry;
    for (int w = 0; w < warp; ++w) before += sm.warp_sum[w];
    int total = 0;
    for (int w = 0; w < kThreads / 32; ++w) total += sm.warp_sum[w];
    const int g = before + __popc(ball & ((1u << lane) - 1u));  // block-local leaf rank
    if (j < nodes) {
      const int p = sm.prog[j];
      const int64_t pn0 = sm.node_off[p], pl0 = sm.leaf_off[p];
      const int i = (int)(gn0 + j - pn0);              // program-local node id
      const int k = (int)(gl0 + g - pl0);              // leaves before it in the program
      const int64_t pos = pn0 + pl0 + i + k;
      out.serialized[pos] = i;
      if (is_leaf) {
        out.serialized[pos + 1] = -1;
        out.ordering[gl0 + g] = i + k;
        sm.leaf_node[g] = (int16_t)j;
      }
    }
    carry += total;
    __syncthreads();  // warp_sum reuse
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  // one thread per leaf, staged vectors, coalesced stores
  for (int c = 0; c < leaves; c += kThreads) {
    const int g = c + t;
    if (g < leaves) {
      const int j = sm.leaf_node[g];
      const int p = sm.prog[j];
      const int base = (int)(sm.node_off[p] - gn0);
      const SmemTree tree{sm.par, sm.ext, sm.ann, base};
      const Chain ch = walk_chain(tree, j - base);
      if (ch.overflow) atomicMin(out.first_bad, (unsigned long long)(p0 + p));
      const int k = (int)(gl0 + g - sm.leaf_off[p]);
      const int n_leaf = (int)(sm.leaf_off[p + 1] - sm.leaf_off[p]);
      double* row = sm.vec + t * kVecPitch;
      const int64_t* st = c == 0 ? reinterpret_cast<const int64_t*>(row + kStatsCol)
                                 : stats + (gl0 + g) * 9;
      leaf_vector(ch, st, k, n_leaf, row);
    }
    // each warp writes its own 32 consecutive leaves (a contiguous 6 KB run,
    // coalesced) from its part of the staging tile: warp barriers only
    __syncwarp();
    const int w0 = c + 32 * warp;
    const int n = max(0, min(32, leaves - w0));
    double2* dst = reinterpret_cast<double2*>(out.vectors + (gl0 + w0) * TPCB_FEAT);
    const double2* src = reinterpret_cast<const double2*>(sm.vec + 32 * warp * kVecPitch);
    // 12 double2 per row; lane + 32 i walks 8 rows every 3 steps
    for (int e = lane; e < n * (TPCB_FEAT / 2); e += 32) {
      const int r = e / (TPCB_FEAT / 2), col = e - r * (TPCB_FEAT / 2);
      dst[e] = src[r * (kVecPitch / 2) + col];
    }
    __syncwarp();
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
  {  // per-device one-time upload of the host-libm log2 table
    static double host_table[tpcb::kLog2Table];
    static bool table_built = false;
    static bool uploaded[64] = {};
    static std::mutex mu;
    int dev = 0;
    TPCB_CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (!table_built) {
      for (int i = 0; i < tpcb::kLog2Table; ++i) host_table[i] = std::log2(1.0 + (double)i);
      table_built = true;
    }
    if (dev >= 64) return TPCB_ERR_UNSUPPORTED;
    if (!uploaded[dev]) {
      TPCB_CUDA_CHECK(cudaMemcpyToSymbol(tpcb::g_log2_table, host_table, sizeof(host_table)));
      uploaded[dev] = true;
    }
  }
  const int64_t blocks = (n_prog + tpcb::kProgsPerBlock - 1) / tpcb::kProgsPerBlock;
  if (blocks > 0x7fffffff) return TPCB_ERR_UNSUPPORTED;
  const size_t smem = sizeof(tpcb::TileSmem);
  TPCB_CUDA_CHECK(cudaFuncSetAttribute(tpcb::build_compact_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tpcb::CompactOut out{d_vectors, d_ordering, d_serialized, d_first_overflow};
  tpcb::build_compact_kernel<<<(unsigned)blocks, tpcb::kThreads, smem, s>>>(d_node_off, d_parent, d_extent, d_annot,
                                                     d_leaf_off, d_stats, n_prog, out);
  TPCB_LAUNCH_CHECK("build_compact_kernel");
  return TPCB_OK;
}
