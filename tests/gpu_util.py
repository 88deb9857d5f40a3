"""Helpers for the -m gpu parity tests: move numpy fixtures to the device, run the CUDA path
through the C-ABI (paper_2309_16849_b200.snls), and compare with the oracle."""
from __future__ import annotations

import numpy as np

from oracle.oracle import Cfg
from tests.helpers import REL_TOL, max_rel


def snls_mod():
    from paper_2309_16849_b200 import snls

    return snls


def dev(x, dtype=None):
    import torch

    a = np.ascontiguousarray(x)
    if dtype is None:
        dtype = torch.int32 if a.dtype.kind in "iu" else torch.float32
    return torch.tensor(a, device="cuda", dtype=dtype)


def host(t):
    return t.detach().cpu().numpy().astype(np.float64) if t is not None else None


def scfg(c: Cfg):
    S = snls_mod()
    return S.SearchConfig(ws=c.ws, wt=c.wt, ps=c.ps, stride0=c.stride0, stride1=c.stride1,
                          topl=c.topl, metric=c.metric, softmax_scale=c.softmax_scale)


def gpu_search(q, k, ff, bf, cfg: Cfg, mode=0, generic=False, weights=False):
    S = snls_mod()
    ctx = S.context()
    ctx.force_generic(generic)
    try:
        r = S.shifted_nls_forward(dev(q), dev(k), None if ff is None else dev(ff),
                                  None if bf is None else dev(bf), scfg(cfg), mode=mode,
                                  want_weights=weights, ctx=ctx)
    finally:
        ctx.force_generic(False)
    return r


def rel_chains(chains_abs, cfg: Cfg, t, h, w, offsets=None):
    """Reference chains hold absolute link positions; the device tape holds them relative
    to the query pixel (snls_cuda.h)."""
    c = np.array(chains_abs, np.float64, copy=True)
    if c.size == 0:
        return c
    rows = c.shape[0]
    # only links k < |dt|-1 are written by the reference; the rest stay zero
    used = np.zeros(c.shape[:3], bool)
    if offsets is not None:
        m = np.abs(np.rint(offsets[..., 0])).astype(int) - 1
        used = np.arange(c.shape[2])[None, None, :] < m[..., None]
    nh, nw = (h - 1) // cfg.stride0 + 1, (w - 1) // cfg.stride0 + 1
    r = np.arange(rows)
    qx = (r % nw) * cfg.stride0
    qy = ((r // nw) % nh) * cfg.stride0
    c[..., 0] -= np.where(used, qy[:, None, None], 0)
    c[..., 1] -= np.where(used, qx[:, None, None], 0)
    return c


def compare_search(res, sims_ref, offs_ref, cfg: Cfg, sims_lplus1=None, exact=False,
                   exact_ties=False):
    """Selected values within REL_TOL everywhere; offsets equal on rows whose oracle ranking
    has no near-tie (exact ties must still resolve by scan order); with `exact` (integer
    inputs) everything must match bit for bit.  Returns the number of excluded rows."""
    sims = host(res.sims)
    offs = host(res.offsets)
    if exact:
        assert np.array_equal(sims, sims_ref), "sims differ on integer-valued inputs"
        assert np.array_equal(offs, offs_ref), "offsets differ on integer-valued inputs"
        return 0
    assert max_rel(sims, sims_ref) <= REL_TOL, max_rel(sims, sims_ref)
    s = np.asarray(sims_lplus1 if sims_lplus1 is not None else sims_ref)
    k = min(s.shape[1], cfg.topl + 1)
    gaps = s[:, : k - 1] - s[:, 1:k]
    scale = np.maximum(1.0, np.abs(s[:, : k - 1]))
    # Exact fp64 ties are kept (must resolve by scan order) only when the tied candidates are
    # the same computation (ps == 1 border reflection); with ps > 1 a reflected window can
    # hold a permutation of the same terms, which ties in fp64 by luck but not in fp32.
    lo = 0.0 if exact_ties else -1.0
    near = np.any((gaps > lo) & (gaps < 1e-4 * scale), axis=1)
    keep = ~near
    d = np.abs(offs[keep] - offs_ref[keep]) / np.maximum(1.0, np.abs(offs_ref[keep]))
    assert d.size == 0 or d.max() <= 1e-6, (d.max(), np.argwhere(d > 1e-6)[:5])
    return int(near.sum())
