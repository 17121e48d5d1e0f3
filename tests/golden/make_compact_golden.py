"""Golden vectors for the compact-AST builder (K0), made by the REFERENCE.

    python tests/golden/make_compact_golden.py     (needs /root/reference)

Programs: the parsed examples of the reference's test_features.py:28-60,
random trees from the reference test-suite's generator
(pkg/tests/conftest.py:rand_program, depth <= 8, up to 16 leaves, extents up
to 63, random annotations) and the synthetic generator's programs
(dataset.random_program, the generate_synthetic workload).  Each is
flattened by this package's FlatForest.from_programs (it accepts the
reference's tree objects) and the reference's build_compact_ast output is
stored next to it: vectors, ordering, serialized.  Also writes a small
dataset in the reference's JSONL format (dataset_ref.jsonl).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(ROOT))

from conftest import rand_program  # noqa: E402  (reference test helper)
from tpcost.dataset import (DEFAULT_SYNTH_DEVICE, SynthOracleConfig,  # noqa: E402
                            generate_synthetic, random_program, save_dataset, split_dataset)
from tpcost.features import build_compact_ast  # noqa: E402
from tpcost.ir import parse_program  # noqa: E402

from paper_2311_09690_b200.forest import FlatForest  # noqa: E402

TEXTS = [
    """program q {
      for i in 0..2 { for j in 0..3 { compute a { fma=1 } } compute b { add=1 } }
    }""",
    "program s { compute only { fma=1 } }",
    """program cr {
      for n in 0..8 {
        for c in 0..16 { compute conv { fma=9 bytes_read=72 bytes_written=4 } }
        for c2 in 0..16 { compute relu { special=1 bytes_read=4 bytes_written=4 } }
      }
    }""",
    # large extents: products near the 2^62 guard and beyond 2^53 (int->float rounding)
    """program big {
      for a in 0..4294967296 @parallel { for b in 0..1073741823 @vectorize @unroll {
        compute x { fma=123456789 add=3 bytes_read=987654321 bytes_written=7 buffers_read=2 } } }
    }""",
    """program odd {
      for a in 0..3037000499 { for b in 0..1518500249 { compute y { mul=5 bytes_read=3 } } }
      compute z { div=1 }
    }""",
]


def main():
    rng = np.random.default_rng(2024)
    progs = [parse_program(t) for t in TEXTS]
    progs += [rand_program(rng, name=f"r{i}") for i in range(300)]
    progs += [random_program(rng, f"s{i}") for i in range(300)]
    forest = FlatForest.from_programs(progs)
    forest.validate()
    vec, order, ser = [], [], []
    for p in progs:
        c = build_compact_ast(p)
        vec.append(c.leaf_vectors)
        order.extend(c.ordering)
        ser.extend(c.serialized)
    np.savez_compressed(
        ROOT / "tests" / "golden" / "compact.npz",
        node_off=forest.node_off, parent=forest.parent, extent=forest.extent,
        annot=forest.annot, leaf_off=forest.leaf_off, stats=forest.stats,
        vectors=np.concatenate(vec), ordering=np.array(order, dtype=np.int32),
        serialized=np.array(ser, dtype=np.int32))
    print(f"{forest.n_prog} programs, {forest.n_nodes} nodes, {forest.n_leaves} leaves")
    # the reference's JSONL wire format (dataset.py:421-485), for the
    # byte-identical writer / reader round trip of the dataset persistence
    ds = split_dataset(generate_synthetic(40, [DEFAULT_SYNTH_DEVICE], SynthOracleConfig(), seed=3))
    save_dataset(ds, ROOT / "tests" / "golden" / "dataset_ref.jsonl")


if __name__ == "__main__":
    main()
