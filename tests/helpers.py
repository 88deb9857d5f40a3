"""Shared test helpers: seeded fp32-representable inputs (the reference's own generator,
rng.hpp:12-24), config draws modelled on the reference's tests, and the parity metrics.

Parity metric: rel_err(a, b) = |a-b| / max(1, |a|, |b|) (gradcheck_util.hpp:19-21).
"""
from __future__ import annotations

import numpy as np

from oracle.oracle import Cfg

REL_TOL = 1e-5  # fp32 tolerance stated by the north star for distances/outputs/gradients


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))


def max_rel(a, b) -> float:
    if np.asarray(a).size == 0:
        return 0.0
    return float(rel_err(a, b).max())


def f32(x):
    """Round to fp32 and back: the oracle (fp64) and the kernels (fp32) see equal values."""
    return np.asarray(x, np.float32).astype(np.float64)


def video(chk, t, h, w, f, seed, lo=-1.0, hi=1.0, integer=False):
    v = chk.uniform(seed, lo, hi, t * h * w * f).reshape(t, h, w, f)
    if integer:
        v = np.floor(v)
    return f32(v)


def flow(chk, t, h, w, seed, mag, integer=False):
    fl = chk.uniform(seed, -mag, mag, t * h * w * 2).reshape(t, h, w, 2)
    if integer:
        fl = np.round(fl)
    return f32(fl)


def draw_cfg(rng, t, *, ws=(1, 3, 5), ps=(1, 3), s1=(1.0, 0.5), max_topl=4, hole_free=False):
    ws_ = int(rng.choice(ws))
    wt = int(rng.integers(0, 3)) if t > 1 else 0
    wt = min(wt, t - 1)
    ps_ = int(rng.choice(ps))
    s0 = int(rng.integers(1, 3))
    if hole_free:
        s0 = max(s0, ps_ // 2 + 1)
    min_frames = min(t, wt + 1)
    topl = 1 + int(rng.integers(0, max(1, min(max_topl, min_frames * ws_ * ws_))))
    return Cfg(ws=ws_, wt=wt, ps=ps_, stride0=s0, stride1=float(rng.choice(s1)), topl=topl,
               metric=str(rng.choice(["ip", "l2"])))


def tie_rows(oracle_sims_lplus1, topl, tol=1e-4):
    """Rows whose oracle ranking among the first topl+1 entries has an adjacent gap below
    tol*max(1,|s|): fp32 may legitimately reorder them (gradcheck_util.hpp:61-69)."""
    s = np.asarray(oracle_sims_lplus1)
    k = min(s.shape[1], topl + 1)
    gaps = s[:, : k - 1] - s[:, 1:k]
    scale = np.maximum(1.0, np.abs(s[:, : k - 1]))
    return np.any(gaps < tol * scale, axis=1)
