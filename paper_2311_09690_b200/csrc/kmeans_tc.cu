// K8, tensor-core mode: KMeans assignment as a distance GEMM on tcgen05.
//
// Reference: sampling.kmeans assignment step (sampling.py:40-42, 80-88):
// assign[i] = argmin_e ‖x_i − c_e‖ (first index on ties), own[i] = that
// distance, float64.
//
// Here a positive ranking score for every (point, centre) pair,
//   q_e = ‖c_e‖² − 2·x·c_e + X,   X = ‖x‖²·(1 + 2^-16) + 2^-16·max_e ‖c_e‖²
// (X exceeds the rounding error of the rest, so q_e > 0), is formed from a
// 3×TF32 tensor-core GEMM (x·c ≈ x_hi·c_hi + x_hi·c_lo + x_lo·c_hi, fp32
// accumulation in TMEM — about fp32 accuracy), and the candidates are chosen
// in the TMEM epilogue, branch-free: the scores of one group of G consecutive
// centres are packed into keys (q with its log2(G) low mantissa bits replaced
// by the position in the group — one LOP3 per score, order-preserving because
// q > 0), the group's minimum key is a tree of three-input FMNMX3, and each
// group winner enters the point's sorted top-4 through a compare-exchange
// chain.  The four candidates are re-ranked with the exact float64 distance in
// numpy's summation order.  The result is the reference's argmin whenever the
// true nearest centre is a candidate: unless another centre of its group
// scores within the key quantum (2^-18 relative for G = 32) or four groups
// beat it (north_star asks ≥ 99.9 % agreement; tests/test_gpu_kmeans.py
// measures it at 262,144 × 1024, d = 24 and 32).  G = 32 for κ ≥ 512; below
// that G = 1 — every score enters the top-4 (exact fp32 top-4, unquantised),
// which costs 20 ALU operations per score but keeps the candidate set robust
// to two near-tied centres falling in one group.  For d ≤ 30 the two spare K
// columns carry ‖c‖² and X (centres −2c | ‖c‖² | 1, points x | 1 | X), so the
// GEMM forms q itself and the scan starts from the TMEM values (d = 24: 0.50 →
// 0.44 ms per 1 M × 1024 pass).
//
// Why this shape (profiles/r02/ncu_kmeans_tc_summary.txt): the epilogue, not
// the tensor core, bounds the pass.  The round-1 kernel kept an exact fp32
// top-4 with a per-score branch; with random centre order each point inserts
// ~26 times at random positions, so some lane of every warp inserts at almost
// every position, the warp pays all 32 lanes' insertions, and the top-4 array
// was dynamically indexed (local memory) — 3.4 ms per 1 M × 1024 pass.
//
// Layout.  Two CTAs per SM, each 4 scanning warps (thread = point = TMEM
// lane, one 128-point tile at a time) + 1 producer warp.  Points and centres
// are tf32 K-major 128-byte-swizzled UMMA tiles (d ≤ 32 → one 128-B row per
// point); the producer streams the pre-swizzled centre image in chunks of 128
// through a 2-deep smem ring (bulk copies; chunk norms through their own
// ring) and one lane issues the MMAs into two 128-column TMEM buffers, so the
// MMAs of chunk c+1 overlap the scan of chunk c.  Synchronisation is mbarriers
// only (loaded / done / empty per buffer, one for the staged points): the
// warps drift freely within a tile, and each warp stages its points of the
// next tile as soon as its scan ends, so the next tile's MMAs overlap this
// tile's fp64 re-rank.
#include <cmath>

#include "async.cuh"
#include "common.cuh"

namespace tpcb {

namespace {

constexpr int TP = 128;        // points per tile = TMEM lanes = threads
constexpr int CN = 128;        // centres per chunk (N of one MMA)
constexpr int kTop = 4;        // candidates re-ranked exactly
constexpr int kRowB = 128;     // bytes per operand row (32 fp32)
constexpr int kPtTile = TP * kRowB;   // 16 KB
constexpr int kCtTile = CN * kRowB;   // 16 KB
// smem: points hi, lo | centre buffers [2][hi, lo] | centre norms [2][128]
constexpr int kSmPtHi = 0, kSmPtLo = kPtTile, kSmCt = 2 * kPtTile;
constexpr int kSmNorm = kSmCt + 2 * 2 * kCtTile;
constexpr int kSmTotal = kSmNorm + 2 * CN * 4;
constexpr float kPadNorm = 1e37f;     // padding centres: finite, never a group winner
constexpr float kBias = 0x1p-16f;

__host__ __device__ inline uint32_t sw128f(int r, int k) {  // fp32 element (row r, col k < 32)
  return (r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 2) ^ (r & 7))) << 4) + (k & 3) * 4;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {  // tf32 × tf32 → fp32, K-major
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ float tf32_hi(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// numpy-order Σ (a−b)² (same as kmeans.cu), float64, no contraction
__device__ double exact_sq(const double* a, const double* b, int d) {
  auto sqd = [&](int i) {
    const double t = __dsub_rn(a[i], b[i]);
    return __dmul_rn(t, t);
  };
  if (d < 8) {
    double r = 0.0;
    for (int i = 0; i < d; ++i) r = __dadd_rn(r, sqd(i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = sqd(j);
  int i = 8;
  for (; i < d - (d % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], sqd(i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < d; ++i) res = __dadd_rn(res, sqd(i));
  return res;
}

// centres → per-chunk operand image: chunk c = [hi tile (16 KB) | lo tile (16 KB)],
// fp32 norms ‖c‖² (padding centres: zero rows, norm kPadNorm) and their maximum
// (float bits; norms ≥ 0, so the unsigned order is the float order)
// fold (d ≤ 30): the image holds −2·c in columns < d, ‖c‖² in column d and 1
// in column d + 1, so the GEMM itself forms ‖c‖² − 2x·c + X (the points carry
// 1 and X in those columns) and the scan reads scores straight from TMEM
__global__ void prep_centers_kernel(const double* __restrict__ c, int kappa, int d, int nchunks,
                                    int fold, uint8_t* __restrict__ img,
                                    float* __restrict__ norms, unsigned* __restrict__ max_norm) {
  const int total = nchunks * CN * 32;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int row = e / 32, k = e - row * 32;  // row = centre index
    const int ch = row / CN, r = row - ch * CN;
    const bool live = row < kappa;
    double s = 0.0;  // ‖c‖² (the thread of column 0 or, folded, of column d)
    if (k == (fold ? d : 0) && live)
      for (int i = 0; i < d; ++i) s += c[(size_t)row * d + i] * c[(size_t)row * d + i];
    double v = (live && k < d) ? c[(size_t)row * d + k] : 0.0;
    if (fold) {
      if (k < d) v *= -2.0;  // exact
      else if (k == d) v = live ? (double)(float)s : (double)kPadNorm;
      else if (k == d + 1) v = 1.0;
    }
    const float hi = tf32_hi((float)v);
    const float lo = tf32_hi((float)(v - (double)hi));
    uint8_t* base = img + (size_t)ch * 2 * kCtTile;
    *reinterpret_cast<float*>(base + sw128f(r, k)) = hi;
    *reinterpret_cast<float*>(base + kCtTile + sw128f(r, k)) = lo;
    if (k == (fold ? d : 0)) {
      norms[row] = live ? (float)s : kPadNorm;
      if (live) atomicMax(max_norm, __float_as_uint((float)s));
    }
  }
}

__device__ __forceinline__ void mma3(uint32_t tmem, uint32_t ph, uint32_t pl, uint32_t ch,
                                     uint32_t cl) {
  const uint32_t id = idesc_tf32(TP, CN);
  const uint32_t a_[3] = {ph, ph, pl}, b_[3] = {ch, cl, ch};
  for (int s = 0; s < 3; ++s)
    for (int k = 0; k < 4; ++k) {
      const uint64_t a = sdesc(a_[s] + k * 32), b = sdesc(b_[s] + k * 32);
      const uint32_t acc = (s | k) != 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(a), "l"(b), "r"(id), "r"(acc));
    }
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      smem_u32(bar)));
}

__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {  // FFMA2
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {  // FADD2
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float min3(float a, float b, float c) {  // FMNMX3
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// (w & mask) | u in ONE LOP3: the mask lives in a register, u is the immediate
// (with both as constants the compiler spends two LOP3s per score)
__device__ __forceinline__ uint32_t pack_key(uint32_t w, uint32_t mask, uint32_t u) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "r"(mask), "r"(u));  // (a & b) | c
  return r;
}

// minimum of G packed keys
template <int G>
__device__ __forceinline__ float group_min(const float* k) {  // G = 1, 8 or 32
  if constexpr (G == 1) {
    return k[0];
  } else if constexpr (G == 8) {
    return min3(min3(k[0], k[1], k[2]), min3(k[3], k[4], k[5]), fminf(k[6], k[7]));
  } else {
    float t[11];
#pragma unroll
    for (int i = 0; i < 10; ++i) t[i] = min3(k[3 * i], k[3 * i + 1], k[3 * i + 2]);
    t[10] = fminf(k[30], k[31]);
    return fminf(min3(min3(t[0], t[1], t[2]), min3(t[3], t[4], t[5]), min3(t[6], t[7], t[8])),
                 fminf(t[9], t[10]));
  }
}

template <int G, bool FOLD>
__global__ void __launch_bounds__(TP + 32, 2) assign_tc_kernel(
    const double* __restrict__ x, int64_t n, int d, const double* __restrict__ centers,
    int kappa, int nchunks, const uint8_t* __restrict__ img, const float* __restrict__ norms,
    const unsigned* __restrict__ max_norm, int64_t* __restrict__ assign,
    double* __restrict__ own, int32_t* __restrict__ counts) {
  extern __shared__ __align__(1024) uint8_t smb[];
  // loaded: chunk image in smem buffer b; done: its MMAs complete (TMEM buffer b
  // holds chunk scores); empty: the 4 scanning warps finished TMEM buffer b;
  // pts: the 4 warps staged the next tile's points; nld: chunk norms in slot b
  __shared__ __align__(8) uint64_t loaded[2], done[2], empty[2], nld[2], pts;
  __shared__ uint32_t s_tmem;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&loaded[i], 1);
      mbar_init(&done[i], 1);
      mbar_init(&empty[i], 4);
      mbar_init(&nld[i], 1);
    }
    mbar_init(&pts, 4);
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const uint32_t sb = smem_u32(smb);
  float* s_norm = reinterpret_cast<float*>(smb + kSmNorm);
  const int64_t stride = (int64_t)gridDim.x * TP, first = (int64_t)blockIdx.x * TP;
  const int ntiles = first < n ? (int)((n - first + stride - 1) / stride) : 0;
  const int total = ntiles * nchunks;  // chunk steps of this CTA, buffers alternate across tiles

  if (warp == 4) {  // producer: bulk loads of the centre image + MMA issue, one lane
    if (lane == 0 && total > 0) {
      auto load = [&](int gc) {
        const int b = gc & 1, c = gc % nchunks;
        mbar_arrive_expect_tx(&loaded[b], (uint32_t)(2 * kCtTile));
        bulk_g2s(smb + kSmCt + b * 2 * kCtTile, img + (size_t)c * 2 * kCtTile, 2 * kCtTile,
                 &loaded[b]);
      };
      load(0);
      if (total > 1) load(1);
      for (int gc = 0; gc < total; ++gc) {
        const int b = gc & 1;
        if (gc % nchunks == 0) mbar_wait(&pts, (gc / nchunks) & 1);
        mbar_wait(&loaded[b], (gc >> 1) & 1);
        if (gc >= 2) mbar_wait(&empty[b], ((gc - 2) >> 1) & 1);  // TMEM buffer b scanned
        mbar_arrive_expect_tx(&nld[b], (uint32_t)(CN * 4));
        bulk_g2s(s_norm + b * CN, norms + (size_t)(gc % nchunks) * CN, CN * 4, &nld[b]);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t cb = sb + kSmCt + b * 2 * kCtTile;
        mma3(tmem + b * CN, sb + kSmPtHi, sb + kSmPtLo, cb, cb + kCtTile);
        commit(&done[b]);
        if (gc + 2 < total) {  // smem buffer b is free once these MMAs complete
          mbar_wait(&done[b], (gc >> 1) & 1);
          load(gc + 2);
        }
      }
    }
  } else {  // warps 0-3: thread = point = TMEM lane
    const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
    const float bias_c = kBias * __uint_as_float(__ldg(max_norm));
    // point i → hi / lo rows of the A operands; returns its score offset X
    auto stage = [&](int64_t i) {
      const bool live = i < n;
      float hv[32], lv[32], xx = 0.f, xf[32];
      if ((d & 1) == 0) {  // 16-B loads
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const double2 v = (live && k < d) ? *reinterpret_cast<const double2*>(x + i * d + k)
                                            : make_double2(0.0, 0.0);
          xf[k] = (float)v.x;
          xf[k + 1] = (float)v.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) xf[k] = (live && k < d) ? (float)x[i * d + k] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) xx = fmaf(xf[k], xf[k], xx);  // columns ≥ d are 0
      const float Xp = fmaf(xx, kBias, xx) + bias_c;
      if (FOLD) {  // 1 and X in columns d, d + 1 (selects: d is not a constant)
#pragma unroll
        for (int k = 0; k < 32; ++k) xf[k] = k == d ? 1.f : (k == d + 1 ? Xp : xf[k]);
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) {  // fp32 split: the 2^-24 rounding of x is below 3xTF32's
        const float vf = xf[k];
        hv[k] = tf32_hi(vf);
        lv[k] = tf32_hi(vf - hv[k]);
      }
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        *reinterpret_cast<float4*>(smb + kSmPtHi + sw128f(t, 4 * c4)) =
            make_float4(hv[4 * c4], hv[4 * c4 + 1], hv[4 * c4 + 2], hv[4 * c4 + 3]);
        *reinterpret_cast<float4*>(smb + kSmPtLo + sw128f(t, 4 * c4)) =
            make_float4(lv[4 * c4], lv[4 * c4 + 1], lv[4 * c4 + 2], lv[4 * c4 + 3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&pts);
      return Xp;
    };
    float X = ntiles > 0 ? stage(first + t) : 0.f;
    int gc = 0;
    for (int it = 0; it < ntiles; ++it) {
      const int64_t i = first + it * stride + t;
      const bool live = i < n;
      float bs[kTop];  // sorted packed keys of the group winners
      int bj[kTop];
#pragma unroll
      for (int q = 0; q < kTop; ++q) {
        bs[q] = INFINITY;
        bj[q] = 0x7fffffff;
      }
      const uint64_t m2 = pk2(-2.f, -2.f), x2 = pk2(X, X);
      // n ≥ 1, so the OR adds nothing — it only keeps the mask a runtime register
      const uint32_t kmask = ~(uint32_t)(G - 1) | (uint32_t)((uint64_t)n >> 63);
      for (int c = 0; c < nchunks; ++c, ++gc) {
        const int b = gc & 1;
        mbar_wait(&done[b], (gc >> 1) & 1);
        if (!FOLD) mbar_wait(&nld[b], (gc >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const float4* nrm4 = reinterpret_cast<const float4*>(s_norm + b * CN);
#pragma unroll 1
        for (int j0 = 0; j0 < CN; j0 += 32) {
          uint32_t r[32];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
              "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]),
                "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
                "=r"(r[30]), "=r"(r[31])
              : "r"(tmem + lane_off + b * CN + j0));
          float4 nv[8];
          if (!FOLD) {
#pragma unroll
            for (int v = 0; v < 8; ++v) nv[v] = nrm4[j0 / 4 + v];
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float key[32];
          if (FOLD) {  // the GEMM formed the scores
#pragma unroll
            for (int u = 0; u < 32; ++u) key[u] = __uint_as_float(pack_key(r[u], kmask, u % G));
          } else {
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const uint64_t s01 =
                fma2(pk2(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1])), m2,
                     add2(pk2(nv[v].x, nv[v].y), x2));
            const uint64_t s23 =
                fma2(pk2(__uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3])), m2,
                     add2(pk2(nv[v].z, nv[v].w), x2));
            const uint32_t w[4] = {(uint32_t)s01, (uint32_t)(s01 >> 32), (uint32_t)s23,
                                   (uint32_t)(s23 >> 32)};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int u = 4 * v + e;
              key[u] = __uint_as_float(pack_key(w[e], kmask, u % G));
            }
          }
          }
#pragma unroll
          for (int g = 0; g < 32 / G; ++g) {
            float m = group_min<G>(key + g * G);
            int jj = c * CN + j0 + g * G + (int)(__float_as_uint(m) & (G - 1));
#pragma unroll
            for (int q = 0; q < kTop; ++q) {  // compare-exchange chain, strict: earlier wins ties
              const bool p = m < bs[q];
              const float nb = p ? m : bs[q];
              const int nj = p ? jj : bj[q];
              m = p ? bs[q] : m;
              jj = p ? bj[q] : jj;
              bs[q] = nb;
              bj[q] = nj;
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[b]);
      }
      // every MMA of this tile has completed (done waited for its last chunk):
      // stage the next tile's points so its MMAs overlap this tile's re-rank
      if (it + 1 < ntiles) X = stage(i + stride);
    if (live) {  // exact float64 re-rank of the candidates (numpy argmin semantics)
      const double* xi = x + i * d;
      double best = INFINITY;
      int bi = 0;
      int cand[kTop];
#pragma unroll
      for (int q = 0; q < kTop; ++q) cand[q] = bj[q];
      // ascending index order so strict '<' keeps the first index among exact ties
#pragma unroll
      for (int q0 = 0; q0 < kTop; ++q0)
#pragma unroll
        for (int q1 = 0; q1 + 1 < kTop - q0; ++q1)
          if (cand[q1] > cand[q1 + 1]) {
            const int tmp = cand[q1];
            cand[q1] = cand[q1 + 1];
            cand[q1 + 1] = tmp;
          }
      double sq[kTop];
      if (d % 8 == 0) {  // all four candidates at once: 8-wide loads, 32 independent chains
        const double* cr[kTop];
#pragma unroll
        for (int q = 0; q < kTop; ++q) cr[q] = centers + (size_t)min(cand[q], kappa - 1) * d;
        double acc[kTop][8];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (8 * b >= d) break;
          double xv[8], cv[kTop][8];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const double2 v = *reinterpret_cast<const double2*>(xi + 8 * b + 2 * h);
            xv[2 * h] = v.x;
            xv[2 * h + 1] = v.y;
          }
#pragma unroll
          for (int q = 0; q < kTop; ++q)
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const double2 v = __ldg(reinterpret_cast<const double2*>(cr[q] + 8 * b + 2 * h));
              cv[q][2 * h] = v.x;
              cv[q][2 * h + 1] = v.y;
            }
#pragma unroll
          for (int q = 0; q < kTop; ++q)
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // numpy order: 8 running sums, i ≡ j (mod 8)
              const double t = __dsub_rn(xv[j], cv[q][j]);
              acc[q][j] = b == 0 ? __dmul_rn(t, t) : __dadd_rn(acc[q][j], __dmul_rn(t, t));
            }
        }
#pragma unroll
        for (int q = 0; q < kTop; ++q)
          sq[q] = __dadd_rn(__dadd_rn(__dadd_rn(acc[q][0], acc[q][1]),
                                      __dadd_rn(acc[q][2], acc[q][3])),
                            __dadd_rn(__dadd_rn(acc[q][4], acc[q][5]),
                                      __dadd_rn(acc[q][6], acc[q][7])));
      } else {
#pragma unroll
        for (int q = 0; q < kTop; ++q)
          sq[q] = exact_sq(xi, centers + (size_t)min(cand[q], kappa - 1) * d, d);
      }
#pragma unroll
      for (int q = 0; q < kTop; ++q) {
        const double dist = sqrt(sq[q]);
        if (cand[q] < kappa && dist < best) {
          best = dist;
          bi = cand[q];
        }
      }
      assign[i] = bi;
      own[i] = best;
      atomicAdd(&counts[bi], 1);
    }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int G, bool FOLD>
int launch_assign(const double* x, int64_t n, int d, const double* c, int kappa, int nchunks,
                   const uint8_t* img, const float* norms, const unsigned* max_norm,
                   int64_t* assign, double* own, int32_t* counts, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(assign_tc_kernel<G, FOLD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmTotal));
    attr = true;
  }
  const int64_t tiles = (n + TP - 1) / TP;
  const int grid = (int)std::min<int64_t>(tiles, 2 * kNumSMs);
  assign_tc_kernel<G, FOLD><<<grid, TP + 32, kSmTotal, stream>>>(x, n, d, c, kappa, nchunks, img, norms,
                                                      max_norm, assign, own, counts);
  return TPCB_OK;
}

}  // namespace

}  // namespace tpcb

using namespace tpcb;

/* KMeans assignment, tensor-core mode (see the file header): same outputs as
 * tpcb_kmeans_assign for d <= 32; d_ws: tpcb_kmeans_assign_tc_ws(kappa) bytes. */
extern "C" size_t tpcb_kmeans_assign_tc_ws(int32_t kappa) {
  const int nchunks = (kappa + CN - 1) / CN;
  return (size_t)nchunks * (2 * kCtTile + CN * 4) + 1024 + 64;
}

extern "C" int tpcb_kmeans_assign_tc(const double* d_x, int64_t n, int32_t d,
                                     const double* d_centers, int32_t kappa, int64_t* d_assign,
                                     double* d_own, int32_t* d_counts, void* d_ws,
                                     size_t ws_bytes, void* stream_) {
  if (!d_x || !d_centers || !d_assign || !d_own || !d_counts || !d_ws) return TPCB_ERR_VALIDATION;
  if (d < 1 || d > 32 || kappa < 1 || n < 1) return TPCB_ERR_UNSUPPORTED;
  if (ws_bytes < tpcb_kmeans_assign_tc_ws(kappa)) return TPCB_ERR_VALIDATION;
  cudaStream_t stream = (cudaStream_t)stream_;
  const int nchunks = (kappa + CN - 1) / CN;
  uint8_t* img = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(d_ws) + 1023) & ~static_cast<uintptr_t>(1023));
  float* norms = reinterpret_cast<float*>(img + (size_t)nchunks * 2 * kCtTile);
  unsigned* max_norm = reinterpret_cast<unsigned*>(norms + nchunks * CN);
  TPCB_CUDA_CHECK(cudaMemsetAsync(d_counts, 0, sizeof(int32_t) * kappa, stream));
  TPCB_CUDA_CHECK(cudaMemsetAsync(max_norm, 0, sizeof(unsigned), stream));
  const bool fold = d <= 30;  // two spare K columns carry the norms and X
  prep_centers_kernel<<<std::min(nchunks * CN * 32 / 256 + 1, 4 * kNumSMs), 256, 0, stream>>>(
      d_centers, kappa, d, nchunks, fold ? 1 : 0, img, norms, max_norm);
  TPCB_LAUNCH_CHECK("prep_centers");
#define TPCB_ASSIGN(G, F)                                                                    \
  launch_assign<G, F>(d_x, n, d, d_centers, kappa, nchunks, img, norms, max_norm, d_assign, \
                      d_own, d_counts, stream)
  const int rc = kappa >= 512 ? (fold ? TPCB_ASSIGN(32, true) : TPCB_ASSIGN(32, false))
                              : (fold ? TPCB_ASSIGN(1, true) : TPCB_ASSIGN(1, false));
#undef TPCB_ASSIGN
  if (rc != TPCB_OK) return rc;
  TPCB_LAUNCH_CHECK("kmeans_assign_tc");
  return TPCB_OK;
}
