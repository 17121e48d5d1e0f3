"""Flattened program forests and the device compact-AST builder (K0).

`FlatForest` stores many loop-nest program trees as pre-order SoA arrays —
the binary form of the trees `features.build_compact_ast` walks
(features.py:155-245) — and `build_compact` turns a whole forest into compact
ASTs on the GPU in one launch (csrc/compact.cu), writing the ragged layout K1
(featurize + pack) reads.  `predict_forest` chains K0 → K1 → forward on the
device: trees in, decoded latencies out, one host→device copy.

Array layout (mirrors `tpcb_build_compact`, include/tpcb200.h):
    node_off [P+1] i64   pre-order node range of program p
    parent   [N]   i32   program-local parent index, -1 for the root
    extent   [N]   i64   loop extent (>= 1), 0 for a compute leaf
    annot    [N]   u8    bit 0 vectorize, bit 1 unroll, bit 2 parallel
    leaf_off [P+1] i64   leaf range of program p (leaves in pre-order)
    stats    [NL,9] i64  ComputeStats fields (ir.py:53-64 order)
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _lib, engine
from .errors import LeafCountExceeded, UnsupportedConfig, ValidationError
from .features import N_ENTRY, CompactAst, CompactBatch
from .ir import ANNOTATIONS, MAX_NEST_DEPTH, ComputeStats

STAT_FIELDS = ComputeStats.FIELDS
COUNT_LIMIT = 1 << 56   # per-field count bound of the flat format (exact 128-bit products)
EXTENT_CLAMP = (1 << 63) - 1  # larger extents overflow the 2^62 guard anyway


@dataclass
class FlatForest:
    node_off: np.ndarray
    parent: np.ndarray
    extent: np.ndarray
    annot: np.ndarray
    leaf_off: np.ndarray
    stats: np.ndarray
    names: list = field(default_factory=list)

    @property
    def n_prog(self) -> int:
        return int(self.node_off.shape[0]) - 1

    @property
    def n_nodes(self) -> int:
        return int(self.node_off[-1])

    @property
    def n_leaves(self) -> int:
        return int(self.leaf_off[-1])

    @property
    def n_leaf(self) -> np.ndarray:
        return np.diff(self.leaf_off)

    # -- construction ------------------------------------------------------

    @classmethod
    def from_programs(cls, programs) -> "FlatForest":
        """Flatten ProgramAst trees (this package's or the reference's own
        objects) into pre-order arrays; iterative, so any depth is safe."""
        node_off, leaf_off = [0], [0]
        parent, extent, annot, stats, names = [], [], [], [], []
        for prog in programs:
            base = len(parent)
            stack = [(prog.root, -1)]
            while stack:
                node, par = stack.pop()
                idx = len(parent) - base
                parent.append(par)
                if node.is_leaf:
                    extent.append(0)
                    annot.append(0)
                    st = node.stats
                    stats.append([int(getattr(st, f)) for f in STAT_FIELDS])
                else:
                    lp = node.loop
                    extent.append(min(int(lp.extent), EXTENT_CLAMP))
                    bits = 0
                    for b, a in enumerate(ANNOTATIONS):
                        if a in lp.annotations:
                            bits |= 1 << b
                    annot.append(bits)
                    stack.extend((c, idx) for c in reversed(node.children))
            node_off.append(len(parent))
            leaf_off.append(len(stats))
            names.append(getattr(prog, "name", ""))
        st = np.array(stats, dtype=object).reshape(-1, 9) if stats else np.zeros((0, 9), object)
        if st.size and (np.any(st >= COUNT_LIMIT) or np.any(st < 0)):
            bad = np.flatnonzero(np.any((st >= COUNT_LIMIT) | (st < 0), axis=1))[0]
            raise UnsupportedConfig(f"leaf {bad}: a ComputeStats count is outside 0..2^56")
        return cls(node_off=np.array(node_off, dtype=np.int64),
                   parent=np.array(parent, dtype=np.int32),
                   extent=np.array(extent, dtype=np.int64),
                   annot=np.array(annot, dtype=np.uint8),
                   leaf_off=np.array(leaf_off, dtype=np.int64),
                   stats=st.astype(np.int64), names=names)

    def validate(self) -> None:
        """Vectorised structural checks of the arrays (the invariants
        ir.make_program establishes for trees, ir.py:122-149)."""
        P, N = self.n_prog, self.parent.shape[0]
        if self.node_off[0] != 0 or np.any(np.diff(self.node_off) < 1) or self.node_off[-1] != N:
            raise ValidationError("node_off must start at 0, grow, and end at len(parent)")
        if self.leaf_off.shape != (P + 1,) or self.leaf_off[0] != 0 or \
                self.stats.shape != (int(self.leaf_off[-1]), 9):
            raise ValidationError("leaf_off / stats shape mismatch")
        if self.extent.shape != (N,) or self.annot.shape != (N,):
            raise ValidationError("extent / annot must have one entry per node")
        prog = np.repeat(np.arange(P), np.diff(self.node_off))
        local = np.arange(N) - self.node_off[prog]
        is_leaf = self.extent == 0
        if np.any(self.extent < 0):
            raise ValidationError("negative loop extent")
        if np.any((local == 0) != (self.parent == -1)):
            raise ValidationError("exactly the first node of each program is its root")
        nonroot = local > 0
        par = self.parent[nonroot].astype(np.int64)
        if np.any(par < 0) or np.any(par >= local[nonroot]):
            raise ValidationError("parent must precede its child in pre-order")
        gpar = par + self.node_off[prog[nonroot]]
        if np.any(is_leaf[gpar]):
            raise ValidationError("leaf node must have no children")
        # depth by fix-point (parents precede children), bounded by the nest limit
        gparent = np.full(N, -1, dtype=np.int64)
        gparent[nonroot] = gpar
        depth = np.zeros(N, dtype=np.int64)
        for _ in range(MAX_NEST_DEPTH + 2):
            new = np.zeros_like(depth)
            new[nonroot] = depth[gpar] + 1
            if np.array_equal(new, depth):
                break
            depth = new
        if np.any(depth > MAX_NEST_DEPTH):
            raise ValidationError(f"nesting deeper than {MAX_NEST_DEPTH}")
        # pre-order: the parent of node i is node i-1 or one of its ancestors
        idx = np.flatnonzero(nonroot)
        cur = idx - 1
        want = depth[idx] - 1
        for _ in range(MAX_NEST_DEPTH + 1):
            up = depth[cur] > want
            if not up.any():
                break
            cur[up] = gparent[cur[up]]
        if np.any(cur != gpar):
            raise ValidationError("node arrays are not in pre-order")
        has_child = np.zeros(N, dtype=bool)
        has_child[gpar] = True
        if np.any(~is_leaf & ~has_child):
            raise ValidationError("loop has empty body")
        if np.any(self.annot > 7):
            raise ValidationError("unknown annotation bits")
        if not np.array_equal(np.bincount(prog[is_leaf], minlength=P), np.diff(self.leaf_off)):
            raise ValidationError("leaf_off does not match the leaves of node arrays")
        if np.any(self.stats < 0) or np.any(self.stats >= COUNT_LIMIT):
            raise ValidationError("ComputeStats counts must be in 0..2^56")
        if np.any(self.stats[:, :7].sum(axis=1) == 0):
            raise ValidationError("compute leaf has no ops and no bytes")

    # -- binary file format --------------------------------

    def save(self, path) -> None:
        np.savez(path, node_off=self.node_off, parent=self.parent, extent=self.extent,
                 annot=self.annot, leaf_off=self.leaf_off, stats=self.stats,
                 names=np.array(self.names, dtype=np.str_))

    @classmethod
    def load(cls, path) -> "FlatForest":
        with np.load(Path(path), allow_pickle=False) as z:
            f = cls(node_off=z["node_off"].astype(np.int64), parent=z["parent"].astype(np.int32),
                    extent=z["extent"].astype(np.int64), annot=z["annot"].astype(np.uint8),
                    leaf_off=z["leaf_off"].astype(np.int64), stats=z["stats"].astype(np.int64),
                    names=[str(s) for s in z["names"]])
        f.validate()
        return f


@dataclass
class DeviceCompact:
    """K0 output on the device: the ragged compact-AST SoA."""

    vectors: torch.Tensor     # (NL, 24) f64
    ordering: torch.Tensor    # (NL,) i32
    serialized: torch.Tensor  # (N + NL,) i32
    leaf_off: torch.Tensor    # (P+1,) i64 on the device
    leaf_off_host: np.ndarray
    ser_off_host: np.ndarray

    @property
    def n_prog(self) -> int:
        return int(self.leaf_off_host.shape[0]) - 1

    def to_host(self) -> list:
        """CompactAst objects (features.py:60-75), one per program."""
        vec = self.vectors.cpu().numpy()
        order = self.ordering.cpu().numpy()
        ser = self.serialized.cpu().numpy()
        lo, so = self.leaf_off_host, self.ser_off_host
        out = []
        for p in range(self.n_prog):
            a, b = int(lo[p]), int(lo[p + 1])
            out.append(CompactAst(leaf_vectors=vec[a:b].copy(),
                                  ordering=tuple(int(i) for i in order[a:b]),
                                  serialized=tuple(int(i) for i in ser[so[p]:so[p + 1]]),
                                  n_leaf=b - a))
        return out

    def to_batch(self, device, device_index=None) -> CompactBatch:
        devs = device if isinstance(device, list) else [device]
        di = (np.zeros(self.n_prog, dtype=np.int32) if device_index is None
              else np.asarray(device_index, dtype=np.int32))
        return CompactBatch(self.vectors.cpu().numpy(), self.ordering.cpu().numpy(),
                            np.diff(self.leaf_off_host), di, devs)


def _check_leaf_limit(n_leaf: np.ndarray, max_leaves) -> int:
    """First program over the leaf limit (build_compact_ast raises
    LeafCountExceeded before walking, features.py:158-160), or P."""
    if max_leaves is None:
        return n_leaf.shape[0]
    bad = np.flatnonzero(n_leaf > max_leaves)
    return int(bad[0]) if bad.size else n_leaf.shape[0]


def build_compact(forest: FlatForest, max_leaves: int | None = None, device="cuda",
                  validate: bool = True) -> DeviceCompact:
    """K0 over a whole forest.  Errors follow the reference's per-program
    order: the first program that fails (leaf limit, then the 2^62 extent
    product guard) raises LeafCountExceeded / OverflowError."""
    engine._need_cuda()
    if validate:
        forest.validate()
    lib = _lib.load()
    n_leaf = forest.n_leaf
    first_lc = _check_leaf_limit(n_leaf, max_leaves)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
    d_node_off, d_parent, d_extent = up(forest.node_off), up(forest.parent), up(forest.extent)
    d_annot, d_leaf_off, d_stats = up(forest.annot), up(forest.leaf_off), up(forest.stats)
    NL, N = forest.n_leaves, forest.n_nodes
    vectors = torch.empty((NL, N_ENTRY), dtype=torch.float64, device=device)
    ordering = torch.empty(NL, dtype=torch.int32, device=device)
    serialized = torch.empty(N + NL, dtype=torch.int32, device=device)
    first_bad = torch.empty(1, dtype=torch.int64, device=device)
    _lib.check(lib.tpcb_build_compact(d_node_off.data_ptr(), d_parent.data_ptr(),
                                      d_extent.data_ptr(), d_annot.data_ptr(),
                                      d_leaf_off.data_ptr(), d_stats.data_ptr(), forest.n_prog,
                                      vectors.data_ptr(), ordering.data_ptr(),
                                      serialized.data_ptr(), first_bad.data_ptr(),
                                      engine.stream_ptr()), "build_compact")
    first_of = int(first_bad.item())  # UINT64_MAX (none) reads as -1
    first_of = forest.n_prog if first_of < 0 else first_of
    if first_lc < forest.n_prog and first_lc <= first_of:
        raise LeafCountExceeded(
            f"program {first_lc}: {int(n_leaf[first_lc])} leaves exceeds maximum {max_leaves}")
    if first_of < forest.n_prog:
        raise OverflowError(f"program {first_of}: extent product exceeds 2^62")
    return DeviceCompact(vectors, ordering, serialized, d_leaf_off, forest.leaf_off.copy(),
                         forest.node_off + forest.leaf_off)


def predict_forest(predictor, forest: FlatForest, device, normalizer=None, device_index=None,
                   validate: bool = True):
    """Trees → K0 compact ASTs → K1 PE + packing → fused forward (+ Box-Cox
    decode when a normalizer is given), all device resident.  Returns
    (pred, latency or None) as host arrays in program order."""
    devs = device if isinstance(device, list) else [device]
    dc = build_compact(forest, predictor.config.n_leaf_max, validate=validate)
    di = (np.zeros(forest.n_prog, dtype=np.int32) if device_index is None
          else np.asarray(device_index, dtype=np.int32))
    from .features import device_vector
    table = np.stack([device_vector(d) for d in devs]).astype(np.float32)
    devfeat = torch.from_numpy(table[di]).to(dc.vectors.device)
    if forest.n_prog == 0:
        from .errors import EmptyBatch
        raise EmptyBatch("forward needs at least one input")
    norm = None
    if normalizer is not None:
        normalizer._check()
        norm = normalizer
    pred, _, _, _, lat = predictor.forward_device(dc.vectors, dc.ordering, dc.leaf_off, devfeat,
                                                  forest.n_prog, False, norm, latents=False,
                                                  n_leaf=forest.n_leaf)
    predictor.status.check("predict_forest")
    return pred.cpu().numpy(), (None if lat is None else lat.cpu().numpy())
