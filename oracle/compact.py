"""Oracle: compact-AST construction over flattened forests (test infrastructure).

Restates, with exact Python integers, over the pre-order SoA arrays of
`paper_2311_09690_b200.forest.FlatForest`:
  * build_compact_ast      features.py:209-245 (pre-order serialization with
                            a -1 marker after every leaf; ordering = the
                            serialized position of each leaf)
  * compute_vector         features.py:172-206 (24-entry schema)
  * _log_extent_product    features.py:158-169 (OverflowError above 2^62)
Python ints make every product exact and `math.log2(int)` / int true
division round exactly like the reference (they are the same CPython calls).
Pinned by tests/golden/compact.npz, produced by the reference itself
(tests/golden/make_compact_golden.py).
"""

from __future__ import annotations

from math import log2

import numpy as np

N_ENTRY = 24
LIMIT = 2 ** 62  # features.py:26


def _log_prod(extents):
    """(log2(1 + prod), prod); (0.0, 0) for no loops (features.py:158-169)."""
    if not extents:
        return 0.0, 0
    prod = 1
    for e in extents:
        prod *= e
    if prod > LIMIT:
        raise OverflowError(f"extent product {prod} exceeds 2^62")
    return log2(1 + prod), prod


def leaf_vector(stats, loops, leaf_index, n_leaf):
    """compute_vector (features.py:172-206).  stats: 9 ints in ComputeStats
    order; loops: [(extent, annot_bits)] outermost first."""
    v = np.zeros(N_ENTRY, dtype=np.float64)
    extents = [e for e, _ in loops]
    log_prod, iters = _log_prod(extents)
    if loops:
        v[0] = len(loops)
        v[1] = log_prod
        v[2] = log2(1 + extents[-1])
        v[3] = log2(1 + extents[0])
    else:
        iters = 1
    for t in range(3):  # vectorize, unroll, parallel
        tagged = [e for e, bits in loops if bits >> t & 1]
        v[4 + t] = len(tagged)
        v[7 + t], _ = _log_prod(tagged)
    fma, add, mul, div, special, br, bw, nbr, nbw = (int(s) for s in stats)
    for t, c in enumerate((fma, add, mul, div, special)):
        v[10 + t] = log2(1 + c)
    total_flops = (2 * fma + add + mul + div + special) * iters
    total_read, total_written = br * iters, bw * iters
    v[15] = log2(1 + total_flops)
    v[16] = log2(1 + br)
    v[17] = log2(1 + bw)
    v[18] = log2(1 + total_read)
    v[19] = log2(1 + total_written)
    v[20] = nbr
    v[21] = nbw
    v[22] = total_flops / (total_read + total_written + 1)
    v[23] = leaf_index / n_leaf
    return v


def build_program(parent, extent, annot, stats):
    """One program's arrays (local indices) -> (vectors, ordering, serialized)."""
    n = len(parent)
    serialized, ordering, vectors = [], [], []
    leaf_nodes = [i for i in range(n) if extent[i] == 0]
    n_leaf = len(leaf_nodes)
    k = 0
    for i in range(n):  # arrays are in pre-order: node id == index
        if extent[i] == 0:
            ordering.append(len(serialized))
            serialized += [i, -1]
            chain = []
            a = int(parent[i])
            while a >= 0:
                chain.append((int(extent[a]), int(annot[a])))
                a = int(parent[a])
            vectors.append(leaf_vector(stats[k], chain[::-1], k, n_leaf))
            k += 1
        else:
            serialized.append(i)
    vec = np.stack(vectors) if vectors else np.zeros((0, N_ENTRY))
    return vec, tuple(ordering), tuple(serialized)


def build_forest(node_off, parent, extent, annot, leaf_off, stats):
    """All programs; returns lists (vectors, ordering, serialized)."""
    out = []
    for p in range(len(node_off) - 1):
        a, b = int(node_off[p]), int(node_off[p + 1])
        la, lb = int(leaf_off[p]), int(leaf_off[p + 1])
        out.append(build_program(parent[a:b], extent[a:b], annot[a:b], stats[la:lb]))
    return out
