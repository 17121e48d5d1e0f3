"""Compact-AST feature types and the device featurizer.

API of the reference module `tpcost.features` (features.py:60-279) on the
hot path: `CompactAst`, `DeviceSpec`, `EncodedInput`, `positional_encoding`,
`device_vector`, `encode_input` — plus `CompactBatch`, the bulk SoA batch the
GPU path is fed with (one host→device copy per batch instead of per-object
Python lists) — and `build_compact_ast`, the tree → compact-AST step, run on
the GPU by K0 over a flattened forest (forest.py, csrc/compact.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import engine
from .errors import LeafCountExceeded, ValidationError

N_ENTRY = 24
THETA_DEFAULT = 10000.0
MARKER = -1


@dataclass(frozen=True)
class CompactAst:
    """Per-leaf computation vectors + serialized-position ordering
    (features.py:60-75)."""

    leaf_vectors: np.ndarray
    ordering: tuple
    serialized: tuple
    n_leaf: int

    def __eq__(self, other) -> bool:
        if not isinstance(other, CompactAst):
            return NotImplemented
        return (self.n_leaf == other.n_leaf and tuple(self.ordering) == tuple(other.ordering)
                and tuple(self.serialized) == tuple(other.serialized)
                and np.array_equal(self.leaf_vectors, other.leaf_vectors))


@dataclass(frozen=True)
class DeviceSpec:
    """Hardware descriptor (features.py:78-119)."""

    name: str
    clock_mhz: float
    mem_gb: float
    bandwidth_gbps: float
    cores: int
    peak_fp32_gflops: float = 0.0
    l2_cache_mb: float = 0.0

    def validate(self) -> None:
        for attr in ("clock_mhz", "mem_gb", "bandwidth_gbps", "cores"):
            if getattr(self, attr) <= 0:
                raise ValidationError(f"device '{self.name}': {attr} must be > 0")
        if self.peak_fp32_gflops < 0 or self.l2_cache_mb < 0:
            raise ValidationError(f"device '{self.name}': negative optional field")

    def to_dict(self) -> dict:
        return {"name": self.name, "clock_mhz": self.clock_mhz, "mem_gb": self.mem_gb,
                "bandwidth_gbps": self.bandwidth_gbps, "cores": self.cores,
                "peak_fp32_gflops": self.peak_fp32_gflops, "l2_cache_mb": self.l2_cache_mb}

    @classmethod
    def from_dict(cls, d: dict) -> "DeviceSpec":
        spec = cls(name=d["name"], clock_mhz=float(d["clock_mhz"]), mem_gb=float(d["mem_gb"]),
                   bandwidth_gbps=float(d["bandwidth_gbps"]), cores=int(d["cores"]),
                   peak_fp32_gflops=float(d.get("peak_fp32_gflops", 0.0)),
                   l2_cache_mb=float(d.get("l2_cache_mb", 0.0)))
        spec.validate()
        return spec


@dataclass(frozen=True)
class EncodedInput:
    """Model-ready input: PE-augmented leaf vectors + device features
    (features.py:143-152)."""

    matrix: np.ndarray
    device_vector: np.ndarray

    @property
    def n_leaf(self) -> int:
        return self.matrix.shape[0]


def device_vector(device: DeviceSpec) -> np.ndarray:
    """log2(1 + [clock, mem, bw, cores, peak_fp32, l2]) (features.py:266-271);
    a 6-number descriptor transform, evaluated once per device."""
    raw = np.array([device.clock_mhz, device.mem_gb, device.bandwidth_gbps, float(device.cores),
                    device.peak_fp32_gflops, device.l2_cache_mb], dtype=np.float64)
    return np.log2(1.0 + raw)


def positional_encoding(compact: CompactAst, theta: float = THETA_DEFAULT) -> np.ndarray:
    """Sinusoidal encoding of serialized positions (features.py:248-263),
    evaluated in fp64 on the GPU (K1's PE term)."""
    if theta <= 0:
        raise ValidationError("theta must be > 0")
    return engine.positional_encoding_device(np.asarray(compact.ordering), theta)


def encode_input(compact: CompactAst, device: DeviceSpec,
                 theta: float = THETA_DEFAULT) -> EncodedInput:
    """leaf vectors + PE, with the device features attached (features.py:274-279)."""
    matrix = np.asarray(compact.leaf_vectors, dtype=np.float64) + positional_encoding(compact, theta)
    return EncodedInput(matrix=matrix, device_vector=device_vector(device))


def compute_vector(leaf, enclosing, leaf_index: int, n_leaf: int) -> np.ndarray:
    """The 24-entry computation vector of one leaf under its enclosing loops,
    outermost first (features.py:168-203), float64.  Computed by the device
    builder K0 on a one-leaf chain program — the same kernel and arithmetic
    as build_compact_ast (exact integer entries, exact quotient, table /
    device log2) —; entry 23 is the caller's position leaf_index / n_leaf.
    Raises OverflowError when the extent product exceeds 2^62."""
    from . import ir
    from .forest import COUNT_LIMIT, FlatForest, build_compact
    enclosing = list(enclosing)
    # no tree validation here (the reference's helper has none: an all-zero
    # leaf is fine); only what K0's exact arithmetic needs — extents >= 1
    # (0 marks a leaf in the node arrays) and counts in 0..2^56
    if any(int(lp.extent) < 1 for lp in enclosing):
        raise ValidationError("loop extents must be >= 1")
    if any(not 0 <= int(getattr(leaf, f)) < COUNT_LIMIT for f in ir.ComputeStats.FIELDS):
        raise ValidationError("ComputeStats counts must be in 0..2^56")
    node = ir.leaf("leaf", leaf)
    for lp in reversed(enclosing):
        node = ir.loop(lp, [node])
    prog = ir.ProgramAst(root=node, name="compute_vector", n_leaf=1)
    dc = build_compact(FlatForest.from_programs([prog]), validate=False)
    v = dc.to_host()[0].leaf_vectors[0].copy()
    v[23] = leaf_index / n_leaf
    return v


def build_compact_ast(ast, max_leaves: int | None = None) -> CompactAst:
    """Serialize a program tree pre-order (marker after each leaf) and build
    its leaf computation vectors (features.py:209-245) — one program through
    the device builder K0; `forest.build_compact` does many per launch.
    Raises LeafCountExceeded above `max_leaves`, OverflowError when an
    enclosing extent product exceeds 2^62, like the reference."""
    from .forest import FlatForest, build_compact
    if max_leaves is not None and ast.n_leaf > max_leaves:
        raise LeafCountExceeded(f"{ast.n_leaf} leaves exceeds maximum {max_leaves}")
    forest = FlatForest.from_programs([ast])
    if int(forest.n_leaf[0]) != ast.n_leaf:
        raise ValidationError(
            f"leaf count mismatch: tree has {int(forest.n_leaf[0])}, header says {ast.n_leaf}")
    return build_compact(forest).to_host()[0]


# ---------------------------------------------------------------------------
# bulk batch
# ---------------------------------------------------------------------------

@dataclass
class CompactBatch:
    """Ragged SoA of many compact ASTs — the bulk input of the GPU path.

    vectors (n_tok, 24) raw leaf vectors (float32 or float64), ordering
    (n_tok,) serialized positions, n_leaf (n_ast,), device_index (n_ast,)
    into `devices` (a list of DeviceSpec)."""

    vectors: np.ndarray
    ordering: np.ndarray
    n_leaf: np.ndarray
    device_index: np.ndarray
    devices: list

    @property
    def n_ast(self) -> int:
        return int(self.n_leaf.shape[0])

    @classmethod
    def from_compacts(cls, compacts, device: DeviceSpec | list, device_index=None,
                      dtype=np.float32) -> "CompactBatch":
        devs = device if isinstance(device, list) else [device]
        vec = np.concatenate([np.asarray(c.leaf_vectors) for c in compacts]).astype(dtype)
        order = np.concatenate([np.asarray(c.ordering, dtype=np.int32) for c in compacts])
        nl = np.array([c.n_leaf for c in compacts], dtype=np.int64)
        di = (np.zeros(len(compacts), dtype=np.int32) if device_index is None
              else np.asarray(device_index, dtype=np.int32))
        return cls(vec, order, nl, di, devs)

    def device_features(self) -> np.ndarray:
        table = np.stack([device_vector(d) for d in self.devices]).astype(np.float32)
        return table[self.device_index]

    def subset(self, idx) -> "CompactBatch":
        idx = np.asarray(idx, dtype=np.int64)
        off = np.zeros(self.n_ast + 1, dtype=np.int64)
        np.cumsum(self.n_leaf, out=off[1:])
        rows = np.concatenate([np.arange(off[i], off[i + 1]) for i in idx]) if len(idx) else \
            np.zeros(0, dtype=np.int64)
        return CompactBatch(self.vectors[rows], self.ordering[rows], self.n_leaf[idx],
                            self.device_index[idx], self.devices)

    def ragged(self) -> engine.RaggedHost:
        return engine.RaggedHost(rows=self.vectors, ordering=self.ordering, n_leaf=self.n_leaf,
                                 devfeat=self.device_features(), encoded=False)


def ragged_from_encoded(inputs: list[EncodedInput], n_leaf_max: int) -> engine.RaggedHost:
    """EncodedInput list (PE already added) → host SoA; validates leaf counts
    first, like costmodel._group_by_leaf (costmodel.py:181-190)."""
    nl = np.fromiter((e.n_leaf for e in inputs), dtype=np.int64, count=len(inputs))
    bad = np.flatnonzero((nl < 1) | (nl > n_leaf_max))
    if bad.size:
        i = int(bad[0])
        raise LeafCountExceeded(
            f"input {i} has {int(nl[i])} leaves, supported range is 1..{n_leaf_max}")
    rows = np.concatenate([np.asarray(e.matrix, dtype=np.float64) for e in inputs])
    dev = np.stack([np.asarray(e.device_vector, dtype=np.float64) for e in inputs])
    return engine.RaggedHost(rows=rows, ordering=np.zeros(rows.shape[0], dtype=np.int32),
                             n_leaf=nl, devfeat=dev.astype(np.float32), encoded=True)


def check_leaf_counts(n_leaf: np.ndarray, n_leaf_max: int) -> None:
    bad = np.flatnonzero((n_leaf < 1) | (n_leaf > n_leaf_max))
    if bad.size:
        i = int(bad[0])
        raise LeafCountExceeded(
            f"input {i} has {int(n_leaf[i])} leaves, supported range is 1..{n_leaf_max}")
