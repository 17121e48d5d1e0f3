"""Dataflow-graph duration fill through the bulk predictor.

`dedup_predict` keeps the reference's signature and semantics
(replayer.py:175-198: one prediction per distinct `tir_key`, every node's
`duration` set, ValidationError for a key without a program, an optional
custom `predictor(compact, device)`), but the cost-model branch predicts all
distinct programs in ONE device batch (K1 featurize+pack, fused forward,
Box-Cox decode) instead of one model call per key.  The graph types, the
simulator and the graph/program file readers are outside the hot path
 — any object with `.nodes` whose items have `.tir_key` and a
writable `.duration` (the reference's `Dfg`) is accepted.
"""

from __future__ import annotations

import numpy as np

from .errors import ValidationError


def dedup_predict(dfg, programs: dict, params, device, normalizer, predictor=None) -> dict:
    keys = []
    seen = set()
    for node in dfg.nodes:
        k = node.tir_key
        if k not in seen:
            if k not in programs:
                raise ValidationError(f"no program for tir_key '{k}'")
            seen.add(k)
            keys.append(k)
    if predictor is not None:  # caller-supplied model: the reference's per-key loop
        durations = {k: float(predictor(programs[k], device)) for k in keys}
    elif not keys:
        durations = {}
    else:
        from .costmodel import Predictor
        from .features import CompactBatch
        normalizer._check()
        model = params if isinstance(params, Predictor) else Predictor(params)
        batch = CompactBatch.from_compacts([programs[k] for k in keys], device,
                                           dtype=np.float64)
        _, _, _, _, lat = model.forward_batch(batch, normalizer)
        durations = {k: float(v) for k, v in zip(keys, lat)}
    for node in dfg.nodes:
        node.duration = durations[node.tir_key]
    return durations
