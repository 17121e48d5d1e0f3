// K8–K11 — KMeans task sampler (sampling.py:40-144), float64.
//
// Every distance is evaluated with the reference's exact floating-point
// recipe — diff = x − c, square, then numpy's pairwise summation over the
// feature axis (8 interleaved accumulators for 8 ≤ d ≤ 128, recursive
// halving above, a plain loop below 8), sqrt for the assignment — and every
// centre is the sequential row sum of its members in point order divided by
// the member count, as `members.mean(axis=0)` computes it.  Assignments,
// centres and the Ψ table therefore match the reference bit for bit; the only
// non-bit-exact quantity is the k-means++ CDF (a parallel scan instead of
// numpy's sequential cumsum), which can change a draw only when the uniform
// falls within rounding distance of a CDF step.
//
//   K10 kmeanspp_*     closest-distance update, total, CDF search (per centre)
//   K8  kmeans_assign  distances to all centres (centres tiled through smem),
//                      first-index argmin, own distance, cluster counts
//   K9  kmeans_update  stable counting sort of points by cluster (CUB radix
//                      sort), then one thread per (cluster, feature) summing
//                      its members in order
//   K11 distance_table Ψ[e, t] = mean over task t's rows of dist(row, c_e)
#include <cub/cub.cuh>

#include "async.cuh"
#include "common.cuh"

namespace tpcb {
namespace {

constexpr int kMaxDim = 128;  // widest feature vector supported

// Σ_k (a_k − b_k)² in numpy's pairwise order (umath pairwise_sum), no FMA
// contraction (each product and sum rounded separately like numpy).
__device__ __forceinline__ double sqd(const double* a, const double* b, int i) {
  const double t = __dsub_rn(a[i], b[i]);
  return __dmul_rn(t, t);
}

__device__ double pw_sq_range(const double* a, const double* b, int lo, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, sqd(a, b, lo + i));
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = sqd(a, b, lo + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], sqd(a, b, lo + i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, sqd(a, b, lo + i));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  // one level of recursion is enough for d ≤ 256; deeper splits loop
  return __dadd_rn(pw_sq_range(a, b, lo, n2), pw_sq_range(a, b, lo + n2, n - n2));
}

__device__ __forceinline__ double pw_sq(const double* a, const double* b, int d) {
  return pw_sq_range(a, b, 0, d);
}

// closest[i] = dist²(x_i, c) (init) or min(closest[i], dist²(x_i, c)); block
// partial sums of the updated closest into part[blockIdx.x].  HBM-bound: a
// block stages 128 consecutive rows (one contiguous span of x) into shared
// memory with coalesced 16-byte loads, rows padded to an odd number of
// doubles so each thread then walks its own row conflict-free, in numpy's
// pairwise summation order (pw_sq_range).
constexpr int kCuRows = 128;
__host__ __device__ inline int cu_stride(int d) { return d | 1; }

__global__ void __launch_bounds__(kCuRows) closest_update_kernel(
    const double* __restrict__ x, int64_t n, int d, const double* __restrict__ c,
    double* __restrict__ closest, int init, double* __restrict__ part) {
  extern __shared__ double sx[];  // [kCuRows][stride] rows, then the centre
  __shared__ double red[kCuRows / 32];
  const int st = cu_stride(d);
  double* sc = sx + kCuRows * st;
  for (int k = threadIdx.x; k < d; k += blockDim.x) sc[k] = c[k];
  const int d2 = d >> 1;                       // 16-byte columns per row
  const bool d2_ok = d2 >= 1 && d2 <= kCuRows;
  const int rpp = d2_ok ? kCuRows / d2 : 1;    // rows per pass
  const int r_off = d2_ok ? threadIdx.x / d2 : 0, k2 = d2_ok ? threadIdx.x % d2 : 0;
  const bool active = r_off < rpp;
  double acc = 0.0;
  const int64_t n_tiles = (n + kCuRows - 1) / kCuRows;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int64_t i0 = t * kCuRows;
    const int rows = (int)(n - i0 < kCuRows ? n - i0 : kCuRows);
    const int total = rows * d;
    const double* src = x + i0 * d;
    __syncthreads();  // previous tile consumed (and the centre staged)
    if (((reinterpret_cast<uintptr_t>(src) & 15) == 0) && ((d & 1) == 0) && d2_ok) {
      // thread -> (row offset, 16-byte column): no division in the loop, 8
      // loads in flight per thread
      const double2* s2 = reinterpret_cast<const double2*>(src);
      constexpr int U = 8;
      for (int r0 = r_off; r0 < rows; r0 += U * rpp) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int r = r0 + u * rpp;
          if (r < rows && active) v[u] = __ldcs(s2 + (size_t)r * d2 + k2);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int r = r0 + u * rpp;
          if (r < rows && active) {
            sx[r * st + 2 * k2] = v[u].x;
            sx[r * st + 2 * k2 + 1] = v[u].y;
          }
        }
      }
    } else {
      for (int e = threadIdx.x; e < total; e += kCuRows) {
        const int r = e / d, k = e - r * d;
        sx[r * st + k] = __ldcs(src + e);
      }
    }
    __syncthreads();
    if (threadIdx.x < rows) {
      const int64_t i = i0 + threadIdx.x;
      const double v = pw_sq(sx + threadIdx.x * st, sc, d);
      const double nv = init ? v : fmin(closest[i], v);
      closest[i] = nv;
      acc += nv;
    }
  }
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < kCuRows / 32; ++w) v += red[w];
    part[blockIdx.x] = v;
  }
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += part[i];  // fixed order per thread
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum_d(v);
    if (threadIdx.x == 0) *out = v;
  }
}


// First j in [0, n) whose monotone predicate holds (n if none): one warp,
// 32-ary narrowing — 4 rounds of one load per lane for n = 1 M (the old
// grid-wide scan hammered one atomicMin from every thread past the answer).
template <class Pred>
__device__ void warp_first_true(int64_t n, Pred pred, unsigned long long* found) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = n;  // answer in [lo, hi]
  while (lo < hi) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t j = lo + lane * step;
    const bool p = j >= hi || pred(j);
    const unsigned b = __ballot_sync(0xffffffffu, p);
    if (b == 0u) {  // all 32 probes false: answer after the last probe
      lo = lo + 31 * step + 1;
      continue;
    }
    const int f = __ffs(b) - 1;
    if (f == 0) {
      hi = lo;
    } else {
      const int64_t nlo = lo + (f - 1) * step + 1, nhi = lo + f * step;
      lo = nlo;
      hi = nhi < hi ? nhi : hi;
    }
  }
  if (lane == 0) *found = (unsigned long long)lo;
}

// first j with cdf[j] / cdf[n-1] > u  (Generator.choice: cdf /= cdf[-1];
// cdf.searchsorted(u, side="right")); the CDF is non-decreasing, so the
// predicate is monotone
__global__ void search_kernel(const double* __restrict__ cdf, int64_t n, double u,
                              unsigned long long* __restrict__ found,
                              const double* __restrict__ total = nullptr,
                              int32_t* __restrict__ zero_step = nullptr, int step = 0) {
  // speculative multi-step launch (tpcb_kmeanspp_steps): a step whose total
  // is 0 takes the reference's other RNG branch (rng.integers) — record the
  // first such step; the host replays from it
  if (zero_step && !(*total > 0.0)) {
    if (threadIdx.x == 0) atomicMin(zero_step, step);
    if (threadIdx.x == 0) *found = 0;
    return;
  }
  const double last = cdf[n - 1];
  warp_first_true(n, [&](int64_t j) { return cdf[j] / last > u; }, found);
}

__global__ void set_center_kernel(const double* __restrict__ x, int d,
                                  const unsigned long long* __restrict__ found, int64_t n,
                                  double* __restrict__ center, int64_t* __restrict__ chosen) {
  unsigned long long j = *found;
  if (j >= (unsigned long long)n) j = n - 1;  // u ≥ cdf_norm[-1] cannot happen for u < 1
  for (int k = threadIdx.x; k < d; k += blockDim.x) center[k] = x[j * d + k];
  if (threadIdx.x == 0 && chosen) *chosen = (int64_t)j;
}

__global__ void set_center_direct_kernel(const double* __restrict__ x, int d, int64_t j,
                                         double* __restrict__ center) {
  for (int k = threadIdx.x; k < d; k += blockDim.x) center[k] = x[j * d + k];
}

// fixed-width variant: the whole point row lives in registers
template <int D>
__device__ __forceinline__ double pw_sq_fixed(const double* a, const double* b) {
  if (D < 8) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) r = __dadd_rn(r, sqd(a, b, i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = sqd(a, b, j);
#pragma unroll
  for (int i = 8; i < D - (D % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], sqd(a, b, i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
  for (int i = D - (D % 8); i < D; ++i) res = __dadd_rn(res, sqd(a, b, i));
  return res;
}

// K8: one thread per point, centres streamed through shared memory in tiles.
// D > 0: compile-time width (row in registers); D == 0: runtime width.
constexpr int kTileCenters = 64;

template <int D>
__global__ void __launch_bounds__(256) assign_kernel(const double* __restrict__ x, int64_t n,
                                                     int d_rt, const double* __restrict__ centers,
                                                     int kappa, int64_t* __restrict__ assign,
                                                     double* __restrict__ own,
                                                     int32_t* __restrict__ counts) {
  extern __shared__ double sc[];  // [kTileCenters][d] then (D == 0) rows [256][d+1]
  const int d = D > 0 ? D : d_rt;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < n;
  double xr[D > 0 ? D : 1];
  double* xs = sc + kTileCenters * d + threadIdx.x * (d + 1);
  if (live) {
    if (D > 0) {
#pragma unroll
      for (int k = 0; k < (D > 0 ? D : 1); ++k) xr[k] = x[i * d + k];
    } else {
      for (int k = 0; k < d; ++k) xs[k] = x[i * d + k];
    }
  }
  double best = INFINITY;
  int bi = 0;
  for (int c0 = 0; c0 < kappa; c0 += kTileCenters) {
    const int tc = min(kTileCenters, kappa - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < tc * d; e += blockDim.x) sc[e] = centers[(size_t)c0 * d + e];
    __syncthreads();
    if (live) {
      for (int j = 0; j < tc; ++j) {
        const double sq = D > 0 ? pw_sq_fixed<(D > 0 ? D : 1)>(xr, sc + j * d)
                                : pw_sq(xs, sc + j * d, d);
        const double dist = sqrt(sq);
        if (dist < best) {  // strict: first index wins ties (np.argmin)
          best = dist;
          bi = c0 + j;
        }
      }
    }
  }
  if (live) {
    assign[i] = bi;
    own[i] = best;
    atomicAdd(&counts[bi], 1);
  }
}

__global__ void to_key_kernel(const int64_t* __restrict__ a, int32_t* __restrict__ key,
                              int32_t* __restrict__ idx, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = (int32_t)a[i];
    idx[i] = (int32_t)i;
  }
}

// K9: centre c feature k = (Σ members in point order) / count
__global__ void member_mean_kernel(const double* __restrict__ x, int d, int kappa,
                                   const int32_t* __restrict__ sorted_idx,
                                   const int32_t* __restrict__ offs,
                                   const int32_t* __restrict__ counts, double* __restrict__ centers) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)kappa * d) return;
  const int c = (int)(e / d), k = (int)(e - (int64_t)c * d);
  const int m = counts[c];
  if (m == 0) return;  // empty cluster keeps its centre (sampling.py:101-104)
  const int32_t* mem = sorted_idx + offs[c];
  double acc = x[(int64_t)mem[0] * d + k];
  int r = 1;
  for (; r + 8 <= m; r += 8) {  // loads in flight, adds in order
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = x[(int64_t)mem[r + j] * d + k];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = __dadd_rn(acc, v[j]);
  }
  for (; r < m; ++r) acc = __dadd_rn(acc, x[(int64_t)mem[r] * d + k]);
  centers[(size_t)c * d + k] = acc / (double)m;
}

// data-parallel k-means++: first local j with (offset + cdf[j]) / total > u
__global__ void search_offset_kernel(const double* __restrict__ cdf, int64_t n, double offset,
                                     double total, double u,
                                     unsigned long long* __restrict__ found) {
  warp_first_true(n, [&](int64_t j) { return (offset + cdf[j]) / total > u; }, found);
}

__global__ void found_to_i64_kernel(const unsigned long long* __restrict__ found, int64_t n,
                                    int64_t* __restrict__ out) {
  const unsigned long long j = *found;
  *out = j < (unsigned long long)n ? (int64_t)j : -1;
}

// data-parallel Lloyd: per-cluster member sums in point order (the partial
// sums one rank contributes to the all-reduce; K9 without the division)
__global__ void member_sum_kernel(const double* __restrict__ x, int d, int kappa,
                                  const int32_t* __restrict__ sorted_idx,
                                  const int32_t* __restrict__ offs,
                                  const int32_t* __restrict__ counts, double* __restrict__ sums) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)kappa * d) return;
  const int c = (int)(e / d), k = (int)(e - (int64_t)c * d);
  const int m = counts[c];
  double acc = 0.0;
  if (m > 0) {  // same order as member_mean_kernel: first member, then in order
    const int32_t* mem = sorted_idx + offs[c];
    acc = x[(int64_t)mem[0] * d + k];
    int r = 1;
    for (; r + 8 <= m; r += 8) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = x[(int64_t)mem[r + j] * d + k];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc = __dadd_rn(acc, v[j]);
    }
    for (; r < m; ++r) acc = __dadd_rn(acc, x[(int64_t)mem[r] * d + k]);
  }
  sums[(size_t)c * d + k] = acc;
}

__global__ void compare_kernel(const int64_t* __restrict__ a, const int64_t* __restrict__ b,
                               int64_t n, int32_t* __restrict__ changed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (a[i] != b[i]) {
      atomicOr(changed, 1);
      return;
    }
}

// K11: Ψ[e, t] — one thread per (centre, task), rows of the task in order
__global__ void psi_kernel(const double* __restrict__ f, const int64_t* __restrict__ off, int nt,
                           int d, const double* __restrict__ centers, int kappa,
                           double* __restrict__ psi) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)kappa * nt) return;
  const int c = (int)(e / nt), t = (int)(e - (int64_t)c * nt);
  const double* cc = centers + (size_t)c * d;
  const int64_t r0 = off[t], r1 = off[t + 1];
  double acc = sqrt(pw_sq(f + r0 * d, cc, d));
  for (int64_t r = r0 + 1; r < r1; ++r) acc = __dadd_rn(acc, sqrt(pw_sq(f + r * d, cc, d)));
  psi[(size_t)c * nt + t] = acc / (double)(r1 - r0);
}

// p[i] = closest[i] / total, read on the fly by the CDF scan (div_kernel's
// arithmetic, no p array round trip through HBM)
struct DivByTotal {
  const double* total;
  __host__ __device__ double operator()(double a) const { return a / *total; }
};
inline cub::TransformInputIterator<double, DivByTotal, const double*> p_iter(const double* c,
                                                                              const double* t) {
  return cub::TransformInputIterator<double, DivByTotal, const double*>(c, DivByTotal{t});
}

// closest_update: 4 tiles of 128 rows per block at least, up to 8 blocks per SM
int closest_grid(int64_t n) {
  const int64_t tiles = (n + kCuRows - 1) / kCuRows;
  return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, kNumSMs * 8));
}
size_t closest_smem(int d) { return (size_t)(kCuRows * cu_stride(d) + d) * sizeof(double); }
cudaError_t prep_closest(int d) {
  return cudaFuncSetAttribute(closest_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)closest_smem(d));
}

// closest_update for d ∈ {24, 32} (the sampler's feature widths): same values,
// a bulk-copy pipeline instead of load-then-compute.  Thread t owns row t of a
// 128-row tile: it issues the 16-byte-aligned bulk copy of that row for the
// NEXT tile (cp.async.bulk → smem, padded pitch so the LDS.128 row walk is
// conflict-free) before computing the current one, arriving on the buffer's
// mbarrier with its byte count — no CTA barrier in the loop, ~2 tiles in flight
// per block, 3 blocks per SM.
template <int D>
__global__ void __launch_bounds__(kCuRows) closest_bulk_kernel(
    const double* __restrict__ x, int64_t n, const double* __restrict__ c,
    double* __restrict__ closest, int init, double* __restrict__ part,
    double* __restrict__ total, unsigned* __restrict__ done, double* __restrict__ wsum) {
  constexpr int kPitch = D * 8 + 16;  // bytes per staged row
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double sc[D];
  __shared__ double red[kCuRows / 32];
  const int t = threadIdx.x;
  if (t < D) sc[t] = c[t];
  if (t == 0) {
    mbar_init(&bar[0], kCuRows);
    mbar_init(&bar[1], kCuRows);
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t n_tiles = (n + kCuRows - 1) / kCuRows;
  auto issue = [&](int64_t tile, int b) {  // this thread's row of `tile` → buffer b
    const int64_t i = tile * kCuRows + t;
    if (i < n) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // WAR vs the last reads
      mbar_arrive_expect_tx(&bar[b], (uint32_t)(D * 8));
      bulk_g2s(sm + (size_t)(b * kCuRows + t) * kPitch, x + i * D, (uint32_t)(D * 8), &bar[b]);
    } else {
      mbar_arrive(&bar[b]);
    }
  };
  double acc = 0.0;
  uint32_t ph[2] = {0, 0};
  int b = 0;
  if ((int64_t)blockIdx.x < n_tiles) issue(blockIdx.x, 0);
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, b ^= 1) {
    const int64_t next = tile + gridDim.x;
    if (next < n_tiles) issue(next, b ^ 1);
    const int64_t i = tile * kCuRows + t;
    const double old = (i < n && !init) ? closest[i] : 0.0;
    mbar_wait(&bar[b], ph[b]);
    ph[b] ^= 1;
    double nv = 0.0;
    if (i < n) {
      double v[D];
      const double2* row = reinterpret_cast<const double2*>(sm + (size_t)(b * kCuRows + t) * kPitch);
#pragma unroll
      for (int k = 0; k < D / 2; ++k) {
        const double2 q = row[k];
        v[2 * k] = q.x;
        v[2 * k + 1] = q.y;
      }
      const double dist = pw_sq_fixed<D>(v, sc);
      nv = init ? dist : fmin(old, dist);
      closest[i] = nv;
      acc += nv;
    }
    // per-warp partial of this tile (32 consecutive points) for pick_kernel
    const double ws = warp_sum_d(nv);
    if ((t & 31) == 0) wsum[tile * (kCuRows / 32) + (t >> 5)] = ws;
  }
  acc = warp_sum_d(acc);
  if ((t & 31) == 0) red[t >> 5] = acc;
  __syncthreads();
  __shared__ bool last;
  if (t == 0) {
    double v = 0.0;
    for (int w = 0; w < kCuRows / 32; ++w) v += red[w];
    part[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {  // the total over the partials in a fixed order (sum_parts_kernel's fold)
    __threadfence();
    double v = 0.0;
    for (int i = t; i < (int)gridDim.x; i += kCuRows) v += __ldcg(part + i);
    v = warp_sum_d(v);
    if ((t & 31) == 0) red[t >> 5] = v;
    __syncthreads();
    if (t == 0) {
      double r = 0.0;
      for (int w = 0; w < kCuRows / 32; ++w) r += red[w];
      *total = r;
      *done = 0;  // ready for the next launch on this workspace
    }
  }
}

bool closest_is_bulk(const double* x, int d) {
  return (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (d == 24 || d == 32);
}

// the next k-means++ centre from the last bulk closest update's per-warp
// partials (wsum, W = 4 per 128-point tile): first j with C_j > u·C_last,
// C the prefix sums of closest (cdf[j] / cdf[n-1] > u, the reference's
// searchsorted on the normalised CDF; like the scan path, the prefix order is
// parallel — warp partials, a fixed-order block scan, then the 32 points of
// the crossing warp in sequence); writes the centre row.  A zero total is the
// reference's other RNG branch: record the step, leave the centre.
__global__ void __launch_bounds__(1024) pick_kernel(
    const double* __restrict__ wsum, int64_t W, const double* __restrict__ closest, int64_t n,
    double u, const double* __restrict__ total, int32_t* __restrict__ zero_step, int step,
    const double* __restrict__ x, int d, double* __restrict__ center) {
  // three levels, every load coalesced: super-chunks of 1024 warp partials
  // (one warp each), their 32 sub-chunks of 32 (one warp each), then 32
  // partials and 32 points in sequence; a level whose partial sums round
  // short of the threshold falls back to its last element
  __shared__ double s_sum[32];
  __shared__ int64_t s_c, s_k;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (!(*total > 0.0)) {
    if (t == 0 && zero_step) atomicMin(zero_step, step);
    return;
  }
  const int64_t n_super = (W + 1023) / 1024;
  // level 1: super-chunk sums, then the crossing super-chunk (thread 0, in order)
  double thr = 0.0, base = 0.0;
  {
    constexpr int kKeep = 128;  // super-chunk sums kept from the first pass (n ≤ 4 M points)
    __shared__ double s_super[32], s_keep[kKeep];
    __shared__ double s_thr, s_base;
    double run_all = 0.0;
    for (int64_t c0 = 0; c0 < n_super; c0 += 32) {  // ≤ 32 super-chunks per pass
      const int64_t c = c0 + warp;
      double v = 0.0;
      if (c < n_super)
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int64_t i = c * 1024 + k * 32 + lane;
          v += i < W ? wsum[i] : 0.0;
        }
      v = warp_sum_d(v);
      if (lane == 0) {
        s_super[warp] = v;
        if (c < kKeep) s_keep[c] = v;
      }
      __syncthreads();
      if (t == 0) {
        for (int w = 0; w < 32 && c0 + w < n_super; ++w) run_all += s_super[w];
        s_sum[0] = run_all;
      }
      __syncthreads();
    }
    if (t == 0) {
      s_thr = u * s_sum[0];
      s_c = n_super - 1;
    }
    __syncthreads();
    thr = s_thr;
    double run = 0.0;
    bool found = false;
    if (n_super <= kKeep) {  // the crossing from the kept sums (same values, same order)
      if (t == 0) {
        for (int64_t c1 = 0; c1 < n_super; ++c1) {
          if (run + s_keep[c1] > thr) {
            s_c = c1;
            found = true;
            break;
          }
          run += s_keep[c1];
        }
        s_base = run;
      }
      found = true;  // s_base set (the last super-chunk on a rounding miss)
    }
    // otherwise a second pass over the super-chunk sums (recomputed
    // identically: same loads, same order)
    for (int64_t c0 = 0; c0 < n_super && !found; c0 += 32) {
      const int64_t c = c0 + warp;
      double v = 0.0;
      if (c < n_super)
        for (int k = 0; k < 32; ++k) {
          const int64_t i = c * 1024 + k * 32 + lane;
          v += i < W ? wsum[i] : 0.0;
        }
      v = warp_sum_d(v);
      if (lane == 0) s_super[warp] = v;
      __syncthreads();
      if (t == 0) {
        for (int w = 0; w < 32 && c0 + w < n_super; ++w) {
          if (run + s_super[w] > thr) {
            s_c = c0 + w;
            found = true;
            break;
          }
          run += s_super[w];
        }
        s_base = run;
        s_sum[1] = found ? 1.0 : 0.0;
      }
      __syncthreads();
      found = s_sum[1] != 0.0;
      __syncthreads();
    }
    if (t == 0 && !found) s_base = run;  // rounding: the last super-chunk
    __syncthreads();
    base = s_base;
  }
  // level 2: the 32 sub-chunks of the crossing super-chunk (warp k sums sub-chunk k)
  const int64_t c = s_c;
  {
    const int64_t i = c * 1024 + warp * 32 + lane;
    double v = i < W ? wsum[i] : 0.0;
    v = warp_sum_d(v);
    if (lane == 0) s_sum[warp] = v;
    __syncthreads();
    if (t == 0) {
      double run = base;
      int64_t k = 31;
      for (int w = 0; w < 32; ++w) {
        if (run + s_sum[w] > thr) {
          k = w;
          break;
        }
        run += s_sum[w];
      }
      s_k = c * 1024 + k * 32;  // first warp partial of the sub-chunk
      s_sum[0] = run;           // prefix before it (level-3 base)
    }
    __syncthreads();
  }
  // level 3 (warp 0): 32 partials in sequence, then 32 points in sequence
  if (warp == 0) {
    const int64_t i0 = s_k;
    const double pv = i0 + lane < W ? wsum[i0 + lane] : 0.0;
    double run = s_sum[0];
    int64_t wi = -1;
    for (int k = 0; k < 32; ++k) {
      const double v = __shfl_sync(0xffffffffu, pv, k);
      if (wi < 0 && i0 + k < W) {
        if (run + v > thr) wi = i0 + k;
        else run += v;
      }
    }
    if (wi < 0) wi = (i0 + 31 < W ? i0 + 31 : W - 1);  // rounding: the last partial
    const int64_t r0 = wi * 32;
    const double cv = r0 + lane < n ? closest[r0 + lane] : 0.0;
    int64_t j = -1;
    for (int k = 0; k < 32; ++k) {
      const double v = __shfl_sync(0xffffffffu, cv, k);
      if (j < 0 && r0 + k < n) {
        run += v;
        if (run > thr) j = r0 + k;
      }
    }
    if (j < 0) j = (r0 + 31 < n ? r0 + 31 : n - 1);
    if (lane == 0) s_k = j;
  }
  __syncthreads();
  const int64_t j = s_k;
  for (int k = t; k < d; k += 1024) center[k] = x[j * d + k];
}

// closest update + the total Σ closest → *total (done: a zeroed counter the
// bulk kernel leaves zeroed; wsum: per-warp partials for pick_kernel)
cudaError_t launch_closest(const double* x, int64_t n, int d, const double* c, double* closest,
                           int init, double* part, double* total, unsigned* done,
                           double* wsum, cudaStream_t stream) {
  const int64_t tiles = (n + kCuRows - 1) / kCuRows;
  if (closest_is_bulk(x, d)) {
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 3 * kNumSMs));
    const int smem = 2 * kCuRows * (d * 8 + 16);
    cudaError_t e;
    if (d == 32) {
      e = cudaFuncSetAttribute(closest_bulk_kernel<32>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      closest_bulk_kernel<32><<<g, kCuRows, smem, stream>>>(x, n, c, closest, init, part, total,
                                                             done, wsum);
    } else {
      e = cudaFuncSetAttribute(closest_bulk_kernel<24>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      closest_bulk_kernel<24><<<g, kCuRows, smem, stream>>>(x, n, c, closest, init, part, total,
                                                             done, wsum);
    }
    return cudaGetLastError();
  }
  const int g = closest_grid(n);
  cudaError_t e = prep_closest(d);
  if (e != cudaSuccess) return e;
  closest_update_kernel<<<g, kCuRows, closest_smem(d), stream>>>(x, n, d, c, closest, init, part);
  sum_parts_kernel<<<1, 1024, 0, stream>>>(part, g, total);
  return cudaGetLastError();
}

int grid_for(int64_t n, int block = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + block - 1) / block, kNumSMs * 16));
}

}  // namespace
}  // namespace tpcb

using namespace tpcb;

// workspace: partial sums, scan temp, found index, sort buffers
extern "C" int tpcb_kmeans_ws_size(int64_t n, int32_t d, int32_t kappa, size_t* bytes) {
  if (n < 1 || d < 1 || kappa < 1 || !bytes) return TPCB_ERR_VALIDATION;
  if (d > kMaxDim) return TPCB_ERR_UNSUPPORTED;
  if (n > 0x7fffffff) return TPCB_ERR_UNSUPPORTED;
  size_t scan_tmp = 0, sort_tmp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, scan_tmp, (double*)nullptr, (double*)nullptr, (int)n);
  size_t scan_tmp2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, scan_tmp2, p_iter(nullptr, nullptr), (double*)nullptr,
                                (int)n);
  scan_tmp = std::max(scan_tmp, scan_tmp2);
  cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (int32_t*)nullptr, (int32_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  size_t b = 0;
  b += 4096 * 8;                  // block partials
  b += 256;                       // found + flags
  b += (size_t)n * 8 * 2;         // p, cdf
  b += (size_t)n * 4 * 4;         // keys/idx in/out
  b += (size_t)(kappa + 1) * 4;   // offsets
  b += std::max(scan_tmp, sort_tmp) + 16 * 256;  // + per-region 256-B alignment slack
  *bytes = b;
  return TPCB_OK;
}

namespace {
struct KWs {
  double* part;
  unsigned long long* found;
  int32_t* flag;
  double* p;
  double* cdf;
  int32_t *kin, *kout, *iin, *iout, *offs;
  void* tmp;
  size_t tmp_bytes;
};

KWs carve(void* ws, size_t bytes, int64_t n, int kappa) {
  KWs w{};
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t sz) {
    char* r = p;
    p += (sz + 255) & ~(size_t)255;
    return r;
  };
  w.part = reinterpret_cast<double*>(take(4096 * 8));
  w.found = reinterpret_cast<unsigned long long*>(take(128));
  w.flag = reinterpret_cast<int32_t*>(take(128));
  w.p = reinterpret_cast<double*>(take((size_t)n * 8));
  w.cdf = reinterpret_cast<double*>(take((size_t)n * 8));
  w.kin = reinterpret_cast<int32_t*>(take((size_t)n * 4));
  w.kout = reinterpret_cast<int32_t*>(take((size_t)n * 4));
  w.iin = reinterpret_cast<int32_t*>(take((size_t)n * 4));
  w.iout = reinterpret_cast<int32_t*>(take((size_t)n * 4));
  w.offs = reinterpret_cast<int32_t*>(take((size_t)(kappa + 1) * 4));
  w.tmp = p;
  const size_t used = (size_t)(p - static_cast<char*>(ws));
  w.tmp_bytes = bytes > used ? bytes - used : 0;
  return w;
}
}  // namespace

extern "C" int tpcb_kmeanspp_init(const double* d_x, int64_t n, int32_t d, int64_t first,
                                  double* d_centers, double* d_closest, double* d_total,
                                  void* ws, size_t ws_bytes, void* stream_) {
  if (!d_x || !d_centers || !d_closest || !d_total || !ws) return TPCB_ERR_VALIDATION;
  if (first < 0 || first >= n || d > kMaxDim) return TPCB_ERR_VALIDATION;
  cudaStream_t stream = (cudaStream_t)stream_;
  KWs w = carve(ws, ws_bytes, n, 1);
  TPCB_CUDA_CHECK(cudaMemsetAsync(w.flag, 0, 4, stream));  // launch_closest's counter
  set_center_direct_kernel<<<1, 128, 0, stream>>>(d_x, d, first, d_centers);
  TPCB_CUDA_CHECK(launch_closest(d_x, n, d, d_centers, d_closest, 1, w.part, d_total,
                                 reinterpret_cast<unsigned*>(w.flag), w.p, stream));
  TPCB_LAUNCH_CHECK("kmeanspp_init");
  return TPCB_OK;
}

extern "C" int tpcb_kmeanspp_step(const double* d_x, int64_t n, int32_t d, int32_t i, double u,
                                  int64_t direct, double* d_centers, double* d_closest,
                                  double* d_total, int64_t* d_chosen, void* ws, size_t ws_bytes,
                                  void* stream_) {
  if (!d_x || !d_centers || !d_closest || !d_total || !ws) return TPCB_ERR_VALIDATION;
  if (d > kMaxDim) return TPCB_ERR_UNSUPPORTED;
  cudaStream_t stream = (cudaStream_t)stream_;
  KWs w = carve(ws, ws_bytes, n, 1);
  TPCB_CUDA_CHECK(cudaMemsetAsync(w.flag, 0, 4, stream));  // launch_closest's counter
  double* center = d_centers + (size_t)i * d;
  if (u >= 0.0) {
    size_t tb = w.tmp_bytes;  // cdf of p = closest / total, the division fused into the scan
    TPCB_CUDA_CHECK(cub::DeviceScan::InclusiveSum(w.tmp, tb, p_iter(d_closest, d_total), w.cdf,
                                                  (int)n, stream));
    search_kernel<<<1, 32, 0, stream>>>(w.cdf, n, u, w.found);
    set_center_kernel<<<1, 128, 0, stream>>>(d_x, d, w.found, n, center, d_chosen);
  } else {
    if (direct < 0 || direct >= n) return TPCB_ERR_VALIDATION;
    set_center_direct_kernel<<<1, 128, 0, stream>>>(d_x, d, direct, center);
  }
  TPCB_CUDA_CHECK(launch_closest(d_x, n, d, center, d_closest, 0, w.part, d_total,
                                 reinterpret_cast<unsigned*>(w.flag), w.p, stream));
  TPCB_LAUNCH_CHECK("kmeanspp_step");
  return TPCB_OK;
}

// steps i0 .. i1-1 of k-means++ with the uniforms pre-drawn on the host
// (h_u[i - i0]: the reference draws rng.random() once per step while the
// running total is > 0), enqueued back to back without host synchronisation;
// *d_zero_step (initialised by the caller to INT32_MAX) receives the first
// step whose total was 0 — there the reference draws rng.integers instead, so
// the caller replays from that step with tpcb_kmeanspp_step.
extern "C" int tpcb_kmeanspp_steps(const double* d_x, int64_t n, int32_t d, int32_t i0,
                                   int32_t i1, const double* h_u, double* d_centers,
                                   double* d_closest, double* d_total, int32_t* d_zero_step,
                                   void* ws, size_t ws_bytes, void* stream_) {
  if (!d_x || !d_centers || !d_closest || !d_total || !ws || !h_u || !d_zero_step)
    return TPCB_ERR_VALIDATION;
  if (d > kMaxDim) return TPCB_ERR_UNSUPPORTED;
  if (i0 < 1 || i1 < i0) return TPCB_ERR_VALIDATION;
  cudaStream_t stream = (cudaStream_t)stream_;
  KWs w = carve(ws, ws_bytes, n, 1);
  TPCB_CUDA_CHECK(cudaMemsetAsync(w.flag, 0, 4, stream));  // launch_closest's counter
  for (int i = i0; i < i1; ++i) {
    double* center = d_centers + (size_t)i * d;
    if (closest_is_bulk(d_x, d)) {  // one launch: search + centre (w.p: the warp partials)
      const int64_t W = (n + kCuRows - 1) / kCuRows * (kCuRows / 32);
      pick_kernel<<<1, 1024, 0, stream>>>(w.p, W, d_closest, n, h_u[i - i0], d_total,
                                          d_zero_step, i, d_x, d, center);
    } else {
      size_t tb = w.tmp_bytes;
      TPCB_CUDA_CHECK(cub::DeviceScan::InclusiveSum(w.tmp, tb, p_iter(d_closest, d_total),
                                                    w.cdf, (int)n, stream));
      search_kernel<<<1, 32, 0, stream>>>(w.cdf, n, h_u[i - i0], w.found, d_total, d_zero_step,
                                          i);
      set_center_kernel<<<1, 128, 0, stream>>>(d_x, d, w.found, n, center, nullptr);
    }
    TPCB_CUDA_CHECK(launch_closest(d_x, n, d, center, d_closest, 0, w.part, d_total,
                                   reinterpret_cast<unsigned*>(w.flag), w.p, stream));
  }
  TPCB_LAUNCH_CHECK("kmeanspp_steps");
  return TPCB_OK;
}

extern "C" int tpcb_kmeans_assign(const double* d_x, int64_t n, int32_t d,
                                  const double* d_centers, int32_t kappa, int64_t* d_assign,
                                  double* d_own, int32_t* d_counts, void* stream_) {
  if (!d_x || !d_centers || !d_assign || !d_own || !d_counts) return TPCB_ERR_VALIDATION;
  if (d > kMaxDim) return TPCB_ERR_UNSUPPORTED;
  cudaStream_t stream = (cudaStream_t)stream_;
  TPCB_CUDA_CHECK(cudaMemsetAsync(d_counts, 0, sizeof(int32_t) * kappa, stream));
  const unsigned grid = (unsigned)((n + 255) / 256);
  if (d == 24 || d == 32) {
    const size_t smem = (size_t)kTileCenters * d * sizeof(double);
    if (d == 24)
      assign_kernel<24><<<grid, 256, smem, stream>>>(d_x, n, d, d_centers, kappa, d_assign, d_own,
                                                     d_counts);
    else
      assign_kernel<32><<<grid, 256, smem, stream>>>(d_x, n, d, d_centers, kappa, d_assign, d_own,
                                                     d_counts);
  } else {
    const size_t smem = ((size_t)kTileCenters * d + 256 * (size_t)(d + 1)) * sizeof(double);
    if (smem > 227 * 1024) return TPCB_ERR_UNSUPPORTED;
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(assign_kernel<0>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    assign_kernel<0><<<grid, 256, smem, stream>>>(d_x, n, d, d_centers, kappa, d_assign, d_own,
                                                  d_counts);
  }
  TPCB_LAUNCH_CHECK("kmeans_assign");
  return TPCB_OK;
}

extern "C" int tpcb_kmeans_update(const double* d_x, int64_t n, int32_t d, int32_t kappa,
                                  const int64_t* d_assign, const int32_t* d_counts,
                                  double* d_centers, void* ws, size_t ws_bytes, void* stream_) {
  if (!d_x || !d_assign || !d_counts || !d_centers || !ws) return TPCB_ERR_VALIDATION;
  cudaStream_t stream = (cudaStream_t)stream_;
  KWs w = carve(ws, ws_bytes, n, kappa);
  to_key_kernel<<<grid_for(n), 256, 0, stream>>>(d_assign, w.kin, w.iin, n);
  int bits = 1;
  while ((1 << bits) < kappa) ++bits;
  size_t tb = w.tmp_bytes;
  TPCB_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.kin, w.kout, w.iin, w.iout, (int)n,
                                                  0, bits, stream));
  tb = w.tmp_bytes;
  TPCB_CUDA_CHECK(cudaMemsetAsync(w.offs, 0, sizeof(int32_t), stream));
  TPCB_CUDA_CHECK(
      cub::DeviceScan::InclusiveSum(w.tmp, tb, d_counts, w.offs + 1, kappa, stream));
  const int64_t items = (int64_t)kappa * d;
  member_mean_kernel<<<(unsigned)((items + 127) / 128), 128, 0, stream>>>(d_x, d, kappa, w.iout,
                                                                         w.offs, d_counts,
                                                                         d_centers);
  TPCB_LAUNCH_CHECK("kmeans_update");
  return TPCB_OK;
}

extern "C" int tpcb_kmeans_changed(const int64_t* d_a, const int64_t* d_b, int64_t n,
                                   int32_t* d_flag, void* stream_) {
  if (!d_a || !d_b || !d_flag) return TPCB_ERR_VALIDATION;
  cudaStream_t stream = (cudaStream_t)stream_;
  TPCB_CUDA_CHECK(cudaMemsetAsync(d_flag, 0, sizeof(int32_t), stream));
  compare_kernel<<<grid_for(n), 256, 0, stream>>>(d_a, d_b, n, d_flag);
  TPCB_LAUNCH_CHECK("kmeans_changed");
  return TPCB_OK;
}

/* ---- data-parallel KMeans pieces (point-sharded; sampling.kmeans_sharded) ---- */

extern "C" int tpcb_kmeanspp_closest(const double* d_x, int64_t n, int32_t d,
                                     const double* d_center, int32_t init, double* d_closest,
                                     double* d_total, void* ws, size_t ws_bytes, void* stream_) {
  if (!d_x || !d_center || !d_closest || !d_total || !ws) return TPCB_ERR_VALIDATION;
  if (d > kMaxDim) return TPCB_ERR_UNSUPPORTED;
  cudaStream_t stream = (cudaStream_t)stream_;
  KWs w = carve(ws, ws_bytes, n, 1);
  TPCB_CUDA_CHECK(cudaMemsetAsync(w.flag, 0, 4, stream));  // launch_closest's counter
  TPCB_CUDA_CHECK(launch_closest(d_x, n, d, d_center, d_closest, init ? 1 : 0, w.part, d_total,
                                 reinterpret_cast<unsigned*>(w.flag), w.p, stream));
  TPCB_LAUNCH_CHECK("kmeanspp_closest");
  return TPCB_OK;
}

extern "C" int tpcb_kmeanspp_cdf(const double* d_closest, int64_t n, const double* d_total,
                                 double* d_local_sum, void* ws, size_t ws_bytes, void* stream_) {
  if (!d_closest || !d_total || !d_local_sum || !ws) return TPCB_ERR_VALIDATION;
  cudaStream_t stream = (cudaStream_t)stream_;
  KWs w = carve(ws, ws_bytes, n, 1);
  size_t tb = w.tmp_bytes;  // cdf of p = closest / total, the division fused into the scan
  TPCB_CUDA_CHECK(cub::DeviceScan::InclusiveSum(w.tmp, tb, p_iter(d_closest, d_total), w.cdf,
                                                (int)n, stream));
  TPCB_CUDA_CHECK(cudaMemcpyAsync(d_local_sum, w.cdf + (n - 1), sizeof(double),
                                  cudaMemcpyDeviceToDevice, stream));
  TPCB_LAUNCH_CHECK("kmeanspp_cdf");
  return TPCB_OK;
}

extern "C" int tpcb_kmeanspp_search(int64_t n, double offset, double total, double u,
                                    int64_t* d_found, void* ws, size_t ws_bytes, void* stream_) {
  if (!d_found || !ws) return TPCB_ERR_VALIDATION;
  cudaStream_t stream = (cudaStream_t)stream_;
  KWs w = carve(ws, ws_bytes, n, 1);
  search_offset_kernel<<<1, 32, 0, stream>>>(w.cdf, n, offset, total, u, w.found);
  found_to_i64_kernel<<<1, 1, 0, stream>>>(w.found, n, d_found);
  TPCB_LAUNCH_CHECK("kmeanspp_search");
  return TPCB_OK;
}

extern "C" int tpcb_kmeans_partial(const double* d_x, int64_t n, int32_t d, int32_t kappa,
                                   const int64_t* d_assign, const int32_t* d_counts,
                                   double* d_sums, void* ws, size_t ws_bytes, void* stream_) {
  if (!d_x || !d_assign || !d_counts || !d_sums || !ws) return TPCB_ERR_VALIDATION;
  cudaStream_t stream = (cudaStream_t)stream_;
  KWs w = carve(ws, ws_bytes, n, kappa);
  to_key_kernel<<<grid_for(n), 256, 0, stream>>>(d_assign, w.kin, w.iin, n);
  int bits = 1;
  while ((1 << bits) < kappa) ++bits;
  size_t tb = w.tmp_bytes;
  TPCB_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.kin, w.kout, w.iin, w.iout, (int)n,
                                                  0, bits, stream));
  tb = w.tmp_bytes;
  TPCB_CUDA_CHECK(cudaMemsetAsync(w.offs, 0, sizeof(int32_t), stream));
  TPCB_CUDA_CHECK(
      cub::DeviceScan::InclusiveSum(w.tmp, tb, d_counts, w.offs + 1, kappa, stream));
  const int64_t items = (int64_t)kappa * d;
  member_sum_kernel<<<(unsigned)((items + 127) / 128), 128, 0, stream>>>(d_x, d, kappa, w.iout,
                                                                        w.offs, d_counts, d_sums);
  TPCB_LAUNCH_CHECK("kmeans_partial");
  return TPCB_OK;
}

extern "C" int tpcb_distance_table(const double* d_feats, const int64_t* d_task_off,
                                   int32_t n_tasks, int32_t d, const double* d_centers,
                                   int32_t kappa, double* d_psi, void* stream_) {
  if (!d_feats || !d_task_off || !d_centers || !d_psi) return TPCB_ERR_VALIDATION;
  if (n_tasks < 1) return TPCB_ERR_TOO_FEW_TASKS;
  if (d > kMaxDim) return TPCB_ERR_UNSUPPORTED;
  const int64_t items = (int64_t)kappa * n_tasks;
  psi_kernel<<<(unsigned)((items + 127) / 128), 128, 0, (cudaStream_t)stream_>>>(
      d_feats, d_task_off, n_tasks, d, d_centers, kappa, d_psi);
  TPCB_LAUNCH_CHECK("distance_table");
  return TPCB_OK;
}
