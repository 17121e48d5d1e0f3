"""Loop-nest program trees (the input of build_compact_ast).

The data types of the reference's `tpcost.ir` (ir.py:53-160) — compute-leaf
statistics, loop descriptors, tree nodes, a validated program — with the same
field names, so trees built by either package feed `features.build_compact_ast`
and `forest.FlatForest.from_programs` (which also accept the reference's own
objects by duck typing).  The text-IR parser (ir.py:170-414) is outside the
hot path and not provided.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ValidationError

ANNOTATIONS = ("vectorize", "unroll", "parallel")  # bit order of FlatForest.annot
MAX_LEAVES_DEFAULT = 16
MAX_NEST_DEPTH = 64  # ir.py:49


@dataclass(frozen=True)
class ComputeStats:
    """Per-innermost-iteration counts of one compute leaf (ir.py:53-75)."""

    fma_count: int = 0
    add_count: int = 0
    mul_count: int = 0
    div_count: int = 0
    special_count: int = 0
    bytes_read: int = 0
    bytes_written: int = 0
    buffers_read: int = 0
    buffers_written: int = 0

    FIELDS = ("fma_count", "add_count", "mul_count", "div_count", "special_count",
              "bytes_read", "bytes_written", "buffers_read", "buffers_written")

    def validate(self) -> None:
        vals = [getattr(self, f) for f in self.FIELDS]
        for name, v in zip(self.FIELDS, vals):
            if v < 0:
                raise ValidationError(f"{name} must be >= 0, got {v}")
        if sum(vals[:7]) == 0:
            raise ValidationError("compute leaf has no ops and no bytes")


@dataclass(frozen=True)
class LoopInfo:
    """One `for v in 0..extent` loop with its annotations (ir.py:78-90)."""

    var_name: str
    extent: int
    annotations: frozenset = frozenset()

    def validate(self) -> None:
        if self.extent < 1:
            raise ValidationError(f"loop '{self.var_name}': extent must be >= 1, got {self.extent}")
        unknown = set(self.annotations) - set(ANNOTATIONS)
        if unknown:
            raise ValidationError(f"unknown annotations: {sorted(unknown)}")


@dataclass(frozen=True)
class AstNode:
    """A loop (with children) or a compute leaf (ir.py:93-104)."""

    kind: str
    loop: LoopInfo | None = None
    stats: ComputeStats | None = None
    label: str = ""
    children: tuple = ()

    @property
    def is_leaf(self) -> bool:
        return self.kind == "leaf"


def loop(info: LoopInfo, children) -> AstNode:
    return AstNode(kind="loop", loop=info, children=tuple(children))


def leaf(label: str, stats: ComputeStats) -> AstNode:
    return AstNode(kind="leaf", stats=stats, label=label)


@dataclass(frozen=True)
class ProgramAst:
    root: AstNode
    name: str
    n_leaf: int = 0


def _check_tree(root) -> int:
    """Iterative structural validation (ir.py:122-140); returns the leaf count."""
    n_leaf = 0
    stack = [(root, 0)]
    while stack:
        node, depth = stack.pop()
        if depth > MAX_NEST_DEPTH:
            raise ValidationError(f"nesting deeper than {MAX_NEST_DEPTH}")
        if node.kind == "leaf":
            if node.children:
                raise ValidationError("leaf node must have no children")
            if node.stats is None:
                raise ValidationError("leaf node missing stats")
            node.stats.validate()
            n_leaf += 1
            continue
        if node.kind != "loop":
            raise ValidationError(f"unknown node kind {node.kind!r}")
        if node.loop is None:
            raise ValidationError("loop node missing loop info")
        node.loop.validate()
        if not node.children:
            raise ValidationError(f"loop '{node.loop.var_name}' has empty body")
        stack.extend((c, depth + 1) for c in node.children)
    return n_leaf


def make_program(name: str, root: AstNode, max_leaves: int = MAX_LEAVES_DEFAULT) -> ProgramAst:
    """Validate a tree and wrap it with its leaf count (ir.py:143-149)."""
    n = _check_tree(root)
    if n > max_leaves:
        raise ValidationError(f"program has {n} leaves, maximum is {max_leaves}")
    return ProgramAst(root=root, name=name, n_leaf=n)


def count_leaves(ast) -> int:
    """Number of compute leaves, iteratively (ir.py:152-162)."""
    n, stack = 0, [ast.root]
    while stack:
        node = stack.pop()
        if node.is_leaf:
            n += 1
        else:
            stack.extend(node.children)
    return n
