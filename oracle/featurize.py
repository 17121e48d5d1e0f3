"""Oracle: compact-AST featurisation and bucket packing (test infrastructure).

Restates
  * positional_encoding   features.py:248-263
  * device_vector         features.py:266-271
  * encode_input          features.py:274-279
  * _group_by_leaf + the sorted-bucket loop   costmodel.py:181-190, 241-261
and defines the packed tile contract the CUDA featurizer must reproduce
bit-exactly (perm, bucket offsets, tile plan, row mask, row→(ast, leaf) map).
"""

from __future__ import annotations

import numpy as np

N_ENTRY = 24          # features.py:18
THETA_DEFAULT = 10000.0  # features.py:19


def pe_denominators(theta: float = THETA_DEFAULT, width: int = N_ENTRY) -> np.ndarray:
    """theta ** (2*delta/width) for delta = 0..width/2-1 (features.py:257-258)."""
    if theta <= 0:
        raise ValueError("theta must be > 0")
    expo = 2.0 * np.arange(width // 2, dtype=np.float64) / width
    return theta ** expo


def positional_rows(positions, theta: float = THETA_DEFAULT) -> np.ndarray:
    """Sinusoidal encoding of serialized positions: (n, 24) float64.

    Column 2δ is sin(pos/θ^(2δ/24)), column 2δ+1 the cosine
    (features.py:248-263)."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 1)
    ang = pos / pe_denominators(theta)[None, :]
    out = np.empty((pos.shape[0], N_ENTRY), dtype=np.float64)
    out[:, 0::2] = np.sin(ang)
    out[:, 1::2] = np.cos(ang)
    return out


def device_features(clock_mhz, mem_gb, bandwidth_gbps, cores, peak_fp32_gflops,
                    l2_cache_mb) -> np.ndarray:
    """log2(1 + raw hardware fields) (features.py:266-271)."""
    raw = np.array([clock_mhz, mem_gb, bandwidth_gbps, float(cores),
                    peak_fp32_gflops, l2_cache_mb], dtype=np.float64)
    return np.log2(1.0 + raw)


def encode_rows(leaf_vectors: np.ndarray, ordering, theta: float = THETA_DEFAULT) -> np.ndarray:
    """leaf vectors + PE of their serialized positions (features.py:274-279)."""
    return np.asarray(leaf_vectors, dtype=np.float64) + positional_rows(ordering, theta)


# ---------------------------------------------------------------------------
# Bucket packing contract
# ---------------------------------------------------------------------------

def bucket_perm(n_leaf: np.ndarray, n_leaf_max: int) -> tuple[np.ndarray, np.ndarray]:
    """(perm, bucket_offsets).

    perm lists AST indices bucket by bucket in ascending n_leaf and, inside
    a bucket, in input order — exactly the order in which the reference
    visits samples (`_group_by_leaf` appends in input order,
    costmodel.py:184-189; buckets run in `sorted(groups)` order, :248).
    bucket_offsets[L] .. bucket_offsets[L+1] is bucket L's slice of perm
    (index 0 unused, length n_leaf_max + 2)."""
    n_leaf = np.asarray(n_leaf, dtype=np.int64)
    if n_leaf.size and (n_leaf.min() < 1 or n_leaf.max() > n_leaf_max):
        raise ValueError("leaf count outside 1..n_leaf_max")
    counts = np.bincount(n_leaf, minlength=n_leaf_max + 1)[: n_leaf_max + 1]
    offsets = np.zeros(n_leaf_max + 2, dtype=np.int64)
    offsets[1:] = np.cumsum(counts)
    # stable counting sort written out explicitly (no argsort), so the oracle
    # is an independent statement of the ordering rule
    perm = np.empty(n_leaf.size, dtype=np.int64)
    cursor = offsets[:-1].copy()
    for i, L in enumerate(n_leaf):
        perm[cursor[L]] = i
        cursor[L] += 1
    return perm, offsets


def tile_plan(bucket_offsets: np.ndarray, rows_per_tile: int):
    """Fixed-stride tiles: bucket L is cut into tiles of floor(R/L) ASTs.

    Returns (tile_L, tile_first, tile_count): bucket leaf count, first perm
    position and number of ASTs of every tile, buckets in ascending L."""
    tl, tf, tc = [], [], []
    n_leaf_max = len(bucket_offsets) - 2
    for L in range(1, n_leaf_max + 1):
        lo, hi = int(bucket_offsets[L]), int(bucket_offsets[L + 1])
        per = rows_per_tile // L
        for start in range(lo, hi, per):
            tl.append(L)
            tf.append(start)
            tc.append(min(per, hi - start))
    return (np.array(tl, dtype=np.int64), np.array(tf, dtype=np.int64),
            np.array(tc, dtype=np.int64))


def pack_tiles(rows_by_ast: list[np.ndarray], n_leaf_max: int, rows_per_tile: int,
               width: int = 32):
    """Packed fixed-stride layout the CUDA featurizer writes.

    Returns dict with perm, bucket_offsets, tile_L/first/count,
    tiles (n_tiles, R, width) float64 (features zero-padded to `width`),
    row_mask (n_tiles, R) uint8, row_ast (n_tiles, R) int64 (input AST index
    or -1), row_leaf (n_tiles, R) int64 (leaf index or -1) and ast_row (B,)
    (flat row of each AST's first leaf)."""
    n_leaf = np.array([r.shape[0] for r in rows_by_ast], dtype=np.int64)
    perm, boff = bucket_perm(n_leaf, n_leaf_max)
    tL, tF, tC = tile_plan(boff, rows_per_tile)
    nt = len(tL)
    tiles = np.zeros((nt, rows_per_tile, width))
    mask = np.zeros((nt, rows_per_tile), dtype=np.uint8)
    row_ast = np.full((nt, rows_per_tile), -1, dtype=np.int64)
    row_leaf = np.full((nt, rows_per_tile), -1, dtype=np.int64)
    ast_row = np.zeros(len(rows_by_ast), dtype=np.int64)
    for t in range(nt):
        L = int(tL[t])
        for a in range(int(tC[t])):
            i = int(perm[tF[t] + a])
            base = a * L
            ast_row[i] = t * rows_per_tile + base
            tiles[t, base:base + L, :N_ENTRY] = rows_by_ast[i]
            mask[t, base:base + L] = 1
            row_ast[t, base:base + L] = i
            row_leaf[t, base:base + L] = np.arange(L)
    return dict(perm=perm, bucket_offsets=boff, tile_L=tL, tile_first=tF,
                tile_count=tC, tiles=tiles, row_mask=mask, row_ast=row_ast,
                row_leaf=row_leaf, ast_row=ast_row)
