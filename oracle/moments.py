"""Oracle: central moment discrepancy and its gradient, float64 (test infra).

Restates costmodel.py:426-486 (`_cmd_forward_backward`) column by column as
power sums, the form the CUDA kernel reduces:

  s_c   = max(hi_c - lo_c, 1e-6)  (support of the union, floor ⇒ no s-grad)
  CMD   = ||(μs-μt)/s||₂ + Σ_{j=2..K} ||(Ω_j(zs) - Ω_j(zt)) / s^j||₂
  Ω_j   = mean over rows of (z - μ)^j

Gradients (each norm term skipped when it is exactly 0,
costmodel.py:449,467):
  mean term   dzs += u/(|u| s ns),  dzt -= u/(|u| s nt),  ds -= u²/(|u| s)
  moment j    dzs += (j/ns)(v/|v|)/s^j (c^{j-1} - mean c^{j-1}),  ds -= j v²/(|v| s)
  support     ds routed to the FIRST argmax (+) / argmin (−) row of the
              union in input order (costmodel.py:476-485).
"""

from __future__ import annotations

import numpy as np

SUPPORT_FLOOR = 1e-6  # costmodel.py:29


def cmd_grad(zs: np.ndarray, zt: np.ndarray, k: int = 5):
    zs = np.asarray(zs, dtype=np.float64)
    zt = np.asarray(zt, dtype=np.float64)
    ns, nt = zs.shape[0], zt.shape[0]
    both = np.vstack([zs, zt])
    lo, hi = both.min(axis=0), both.max(axis=0)
    raw = hi - lo
    flat = raw < SUPPORT_FLOOR
    s = np.where(flat, SUPPORT_FLOOR, raw)
    ms, mt = zs.mean(axis=0), zt.mean(axis=0)
    cs, ct = zs - ms, zt - mt
    gs, gt = np.zeros_like(zs), np.zeros_like(zt)
    gsup = np.zeros_like(s)

    u = (ms - mt) / s
    nu = float(np.sqrt(np.sum(u * u)))
    value = nu
    if nu > 0.0:
        gs += (u / nu) / (s * ns)
        gt -= (u / nu) / (s * nt)
        gsup -= (u / nu) * u / s

    ps, pt = cs.copy(), ct.copy()          # c^(j-1)
    for j in range(2, k + 1):
        qs, qt = ps * cs, pt * ct          # c^j
        sj = s ** j
        v = (qs.mean(axis=0) - qt.mean(axis=0)) / sj
        nv = float(np.sqrt(np.sum(v * v)))
        value += nv
        if nv > 0.0:
            w = (v / nv) / sj
            gs += (j / ns) * w * (ps - ps.mean(axis=0))
            gt -= (j / nt) * w * (pt - pt.mean(axis=0))
            gsup -= j * (v / nv) * v / s
        ps, pt = qs, qt

    gsup = np.where(flat, 0.0, gsup)
    if np.any(gsup != 0.0):
        gb = np.zeros_like(both)
        cols = np.arange(both.shape[1])
        np.add.at(gb, (both.argmax(axis=0), cols), gsup)
        np.add.at(gb, (both.argmin(axis=0), cols), -gsup)
        gs += gb[:ns]
        gt += gb[ns:]
    return float(value), gs, gt
