"""Oracle: the transformer cost model, float64 (test infrastructure).

A restatement of the reference predictor written over *bucket tensors*
(all ASTs of one leaf count stacked as (n, L, d)), the unit the CUDA kernels
tile over.  Citations (reference = /root/reference/pkg/src/tpcost):

  parameter names / init order    costmodel.py:116-150, nn.py:16-19
  encoder layer (post-LN)         costmodel.py:193-212, nn.py:26-96
  leaf-count routed embedding     costmodel.py:213-216
  device MLP + gate, decoder      costmodel.py:217-229
  bucketed forward / scatter      costmodel.py:233-262
  backward                        costmodel.py:280-336, nn.py:30-120
  hybrid / mse / mape losses      costmodel.py:343-423
  Box-Cox decode                  dataset.py:97-115, costmodel.py:358-373
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DEVICE_FEATURES = 6


@dataclass(frozen=True)
class Dims:
    d_model: int
    n_layers: int
    n_heads: int
    d_ff: int
    d_embed: int
    d_device: int
    decoder_dims: tuple
    n_leaf_max: int


def dims_of(cfg) -> Dims:
    return Dims(cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.d_embed,
                cfg.d_device, tuple(cfg.decoder_dims), cfg.n_leaf_max)


def tensor_specs(dm: Dims, n_entry: int = 24) -> list[tuple[str, tuple]]:
    """Canonical (name, shape) list in reference creation order
    (costmodel.py:127-149)."""
    d = dm.d_model
    out: list[tuple[str, tuple]] = []

    def lin(name, fi, fo):
        out.append((f"{name}.W", (fi, fo)))
        out.append((f"{name}.b", (fo,)))

    lin("input", n_entry, d)
    for i in range(dm.n_layers):
        p = f"enc{i}"
        for w in ("Wq", "Wk", "Wv", "Wo"):
            out.append((f"{p}.attn.{w}", (d, d)))
        for b in ("bq", "bk", "bv", "bo"):
            out.append((f"{p}.attn.{b}", (d,)))
        out.append((f"{p}.ln1.g", (d,)))
        out.append((f"{p}.ln1.b", (d,)))
        lin(f"{p}.ffn.h", d, dm.d_ff)
        lin(f"{p}.ffn.o", dm.d_ff, d)
        out.append((f"{p}.ln2.g", (d,)))
        out.append((f"{p}.ln2.b", (d,)))
    for L in range(1, dm.n_leaf_max + 1):
        lin(f"leaf_embed.{L}", L * d, dm.d_embed)
    lin("dev.hidden", DEVICE_FEATURES, dm.d_device)
    lin("dev.proj", dm.d_device, dm.d_embed)
    w = dm.d_embed
    for i, hdim in enumerate(dm.decoder_dims):
        lin(f"dec.{i}", w, hdim)
        w = hdim
    lin("dec.out", w, 1)
    return out


# ---------------------------------------------------------------------------
# primitive blocks (each returns what its backward needs)
# ---------------------------------------------------------------------------

def _ln(x, g, b, eps=1e-5):
    # nn.py:48-54 — biased variance, eps inside the sqrt
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    inv = 1.0 / np.sqrt(var + eps)
    xh = (x - mu) * inv
    return g * xh + b, xh, inv


def _ln_back(dy, xh, inv, g):
    # nn.py:57-66
    gx = dy * g
    dx = inv * (gx - gx.mean(axis=-1, keepdims=True)
                - xh * (gx * xh).mean(axis=-1, keepdims=True))
    red = tuple(range(dy.ndim - 1))
    return dx, (dy * xh).sum(axis=red), dy.sum(axis=red)


def _heads(t, H):
    n, L, d = t.shape
    return t.reshape(n, L, H, d // H).transpose(0, 2, 1, 3)


def _unheads(t):
    n, H, L, dh = t.shape
    return t.transpose(0, 2, 1, 3).reshape(n, L, H * dh)


def _wgrad(x, dy):
    return x.reshape(-1, x.shape[-1]).T @ dy.reshape(-1, dy.shape[-1])


# ---------------------------------------------------------------------------
# forward / backward over one bucket
# ---------------------------------------------------------------------------

def bucket_forward(T: dict, dm: Dims, x: np.ndarray, dev: np.ndarray):
    """x: (n, L, 24) encoded rows, dev: (n, 6) device vectors.
    Returns pred (n,), z_x, z_v, z and a tape for bucket_backward."""
    n, L, _ = x.shape
    H = dm.n_heads
    scale = 1.0 / math.sqrt(dm.d_model // H)
    tape = {"x": x, "dev": dev, "layers": []}
    h = x @ T["input.W"] + T["input.b"]
    for i in range(dm.n_layers):
        p = f"enc{i}."
        q = h @ T[p + "attn.Wq"] + T[p + "attn.bq"]
        k = h @ T[p + "attn.Wk"] + T[p + "attn.bk"]
        v = h @ T[p + "attn.Wv"] + T[p + "attn.bv"]
        qh, kh, vh = _heads(q, H), _heads(k, H), _heads(v, H)
        s = np.einsum("nhid,nhjd->nhij", qh, kh) * scale
        s = s - s.max(axis=-1, keepdims=True)
        e = np.exp(s)
        pr = e / e.sum(axis=-1, keepdims=True)
        ctx = _unheads(np.einsum("nhij,nhjd->nhid", pr, vh))
        a = ctx @ T[p + "attn.Wo"] + T[p + "attn.bo"]
        h1, xh1, inv1 = _ln(h + a, T[p + "ln1.g"], T[p + "ln1.b"])
        fpre = h1 @ T[p + "ffn.h.W"] + T[p + "ffn.h.b"]
        f = np.maximum(fpre, 0.0)
        o = f @ T[p + "ffn.o.W"] + T[p + "ffn.o.b"]
        h2, xh2, inv2 = _ln(h1 + o, T[p + "ln2.g"], T[p + "ln2.b"])
        tape["layers"].append(dict(h=h, qh=qh, kh=kh, vh=vh, pr=pr, ctx=ctx,
                                   xh1=xh1, inv1=inv1, h1=h1, f=f,
                                   xh2=xh2, inv2=inv2))
        h = h2
    flat = h.reshape(n, L * dm.d_model)
    z_x = flat @ T[f"leaf_embed.{L}.W"] + T[f"leaf_embed.{L}.b"]
    dpre = dev @ T["dev.hidden.W"] + T["dev.hidden.b"]
    z_v = np.maximum(dpre, 0.0)
    zp = z_v @ T["dev.proj.W"] + T["dev.proj.b"]
    z = z_x * zp
    u = z
    dec_in = []
    for j in range(len(dm.decoder_dims)):
        dec_in.append(u)
        u = np.maximum(u @ T[f"dec.{j}.W"] + T[f"dec.{j}.b"], 0.0)
    pred = (u @ T["dec.out.W"] + T["dec.out.b"])[:, 0]
    tape.update(flat=flat, z_x=z_x, z_v=z_v, zp=zp, dec_in=dec_in, u=u, L=L)
    return pred, z_x, z_v, z, tape


def bucket_backward(T: dict, dm: Dims, tape: dict, dpred: np.ndarray,
                    dz_extra: np.ndarray | None, G: dict) -> None:
    """Accumulate d(objective)/d(param) into G (costmodel.py:280-336)."""
    def acc(name, val):
        G[name] = G[name] + val if name in G else val

    H = dm.n_heads
    scale = 1.0 / math.sqrt(dm.d_model // H)
    L = tape["L"]
    n = dpred.shape[0]
    du = dpred[:, None]
    acc("dec.out.W", tape["u"].T @ du)
    acc("dec.out.b", du.sum(axis=0))
    du = du @ T["dec.out.W"].T
    for j in reversed(range(len(dm.decoder_dims))):
        uin = tape["dec_in"][j]
        out_j = tape["dec_in"][j + 1] if j + 1 < len(dm.decoder_dims) else tape["u"]
        du = du * (out_j > 0)
        acc(f"dec.{j}.W", uin.T @ du)
        acc(f"dec.{j}.b", du.sum(axis=0))
        du = du @ T[f"dec.{j}.W"].T
    dz = du if dz_extra is None else du + dz_extra
    dzx = dz * tape["zp"]
    dzp = dz * tape["z_x"]
    acc("dev.proj.W", tape["z_v"].T @ dzp)
    acc("dev.proj.b", dzp.sum(axis=0))
    dzv = (dzp @ T["dev.proj.W"].T) * (tape["z_v"] > 0)
    acc("dev.hidden.W", tape["dev"].T @ dzv)
    acc("dev.hidden.b", dzv.sum(axis=0))
    acc(f"leaf_embed.{L}.W", tape["flat"].T @ dzx)
    acc(f"leaf_embed.{L}.b", dzx.sum(axis=0))
    dh = (dzx @ T[f"leaf_embed.{L}.W"].T).reshape(n, L, dm.d_model)
    for i in reversed(range(dm.n_layers)):
        p = f"enc{i}."
        c = tape["layers"][i]
        dr2, dg, db = _ln_back(dh, c["xh2"], c["inv2"], T[p + "ln2.g"])
        acc(p + "ln2.g", dg)
        acc(p + "ln2.b", db)
        acc(p + "ffn.o.W", _wgrad(c["f"], dr2))
        acc(p + "ffn.o.b", dr2.reshape(-1, dr2.shape[-1]).sum(axis=0))
        dfpre = (dr2 @ T[p + "ffn.o.W"].T) * (c["f"] > 0)
        acc(p + "ffn.h.W", _wgrad(c["h1"], dfpre))
        acc(p + "ffn.h.b", dfpre.reshape(-1, dfpre.shape[-1]).sum(axis=0))
        dh1 = dr2 + dfpre @ T[p + "ffn.h.W"].T
        dr1, dg, db = _ln_back(dh1, c["xh1"], c["inv1"], T[p + "ln1.g"])
        acc(p + "ln1.g", dg)
        acc(p + "ln1.b", db)
        acc(p + "attn.Wo", _wgrad(c["ctx"], dr1))
        acc(p + "attn.bo", dr1.reshape(-1, dr1.shape[-1]).sum(axis=0))
        dctx = _heads(dr1 @ T[p + "attn.Wo"].T, H)
        pr = c["pr"]
        dpr = np.einsum("nhid,nhjd->nhij", dctx, c["vh"])
        dvh = np.einsum("nhij,nhid->nhjd", pr, dctx)
        ds = pr * (dpr - (dpr * pr).sum(axis=-1, keepdims=True)) * scale
        dqh = np.einsum("nhij,nhjd->nhid", ds, c["kh"])
        dkh = np.einsum("nhij,nhid->nhjd", ds, c["qh"])
        dh_in = dr1.copy()
        for nm, dt in (("q", dqh), ("k", dkh), ("v", dvh)):
            dm_ = _unheads(dt)
            acc(p + f"attn.W{nm}", _wgrad(c["h"], dm_))
            acc(p + f"attn.b{nm}", dm_.reshape(-1, dm_.shape[-1]).sum(axis=0))
            dh_in = dh_in + dm_ @ T[p + f"attn.W{nm}"].T
        dh = dh_in
    acc("input.W", _wgrad(tape["x"], dh))
    acc("input.b", dh.reshape(-1, dh.shape[-1]).sum(axis=0))


def forward(T: dict, dm: Dims, rows_by_ast: list[np.ndarray], dev: np.ndarray):
    """Whole-batch forward in input order (costmodel.py:233-262).
    rows_by_ast[i]: (L_i, 24) encoded matrix; dev: (B, 6)."""
    B = len(rows_by_ast)
    if B == 0:
        raise ValueError("empty batch")
    n_leaf = np.array([r.shape[0] for r in rows_by_ast])
    pred = np.empty(B)
    z_x = np.empty((B, dm.d_embed))
    z_v = np.empty((B, dm.d_device))
    z = np.empty((B, dm.d_embed))
    tapes = []
    for L in sorted(set(n_leaf.tolist())):
        idx = np.flatnonzero(n_leaf == L)
        x = np.stack([rows_by_ast[i] for i in idx])
        p, a, b, c, tape = bucket_forward(T, dm, x, dev[idx])
        pred[idx], z_x[idx], z_v[idx], z[idx] = p, a, b, c
        tape["idx"] = idx
        tapes.append(tape)
    return pred, z_x, z_v, z, tapes


def backward_from(T: dict, dm: Dims, tapes, dpred: np.ndarray,
                  dz_extra: np.ndarray | None, G: dict | None = None) -> dict:
    G = {} if G is None else G
    for tape in tapes:
        idx = tape["idx"]
        bucket_backward(T, dm, tape, dpred[idx],
                        None if dz_extra is None else dz_extra[idx], G)
    return G


# ---------------------------------------------------------------------------
# losses and label transform
# ---------------------------------------------------------------------------

def boxcox_decode(e, lam, shift, t_mean, t_std):
    """Model space → seconds; NaN where λt+1 ≤ 0 (dataset.py:97-115)."""
    t = np.asarray(e, dtype=np.float64) * t_std + t_mean
    if abs(lam) < 1e-9:
        return np.exp(t) - shift
    base = lam * t + 1.0
    with np.errstate(invalid="ignore"):
        out = np.power(base, 1.0 / lam) - shift
    return np.where(base > 0, out, np.nan)


def boxcox_encode(y, lam, shift, t_mean, t_std):
    y = np.asarray(y, dtype=np.float64) + shift
    t = np.log(y) if abs(lam) < 1e-9 else (np.power(y, lam) - 1.0) / lam
    return (t - t_mean) / t_std


def _decode_grad(e, lam, shift, t_mean, t_std):
    # costmodel.py:358-373 (clamped at 1e-12, zero slope beyond)
    t = e * t_std + t_mean
    if abs(lam) < 1e-9:
        return np.exp(t) - shift, t_std * np.exp(t)
    base = lam * t + 1.0
    ok = base > 1e-12
    base = np.where(ok, base, 1e-12)
    return (np.power(base, 1.0 / lam) - shift,
            np.where(ok, t_std * np.power(base, 1.0 / lam - 1.0), 0.0))


def loss_and_grad(pred, y, mode="hybrid", lam_h=1e-3, offset=0.0,
                  space="transformed", norm=None):
    """(value, dvalue/dpred) — costmodel.py:376-423.  norm = (λ, shift,
    t_mean, t_std) for the original-space relative term."""
    n = pred.size
    d = pred - y
    if mode == "mse":
        return float(np.mean(d * d)), 2.0 * d / n
    if space == "original":
        y0 = boxcox_decode(y, *norm)
        p0, dp0 = _decode_grad(pred, *norm)
        r = p0 - y0
        rv, rg = float(np.mean(np.abs(r) / y0)), np.sign(r) * dp0 / (y0 * n)
    else:
        den = y + offset
        rv, rg = float(np.mean(np.abs(d) / den)), np.sign(d) / (den * n)
    if mode == "mape":
        return rv, rg
    return float(np.mean(d * d)) + lam_h * rv, 2.0 * d / n + lam_h * rg
