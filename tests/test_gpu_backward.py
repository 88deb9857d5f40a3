"""GPU parity: shifted_nls_backward (dQ, dK, dFflow, dBflow) against the oracle's analytic
gradients (which the reference validates against finite differences, test_gradcheck.cpp),
stage-isolated on the reference's own tape."""
import os

import numpy as np
import pytest

from oracle.oracle import Cfg
from tests.gpu_util import dev, host, rel_chains, scfg, snls_mod
from tests.helpers import REL_TOL, draw_cfg, f32, flow, max_rel, video

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return z, Cfg(**eval(str(z["cfg"])))


def gpu_bwd(q, k, cfg, offsets, chains_abs, grad):
    S = snls_mod()
    t, h, w, _ = q.shape
    res = S.SearchResult(sims=dev(np.zeros(offsets.shape[:2])), offsets=dev(offsets),
                         chains=dev(rel_chains(chains_abs, cfg, t, h, w, offsets)) if cfg.wt > 1 else None,
                         cfg=scfg(cfg))
    return [host(x) for x in S.shifted_nls_backward(dev(grad), res, dev(q), dev(k))]


def centers_from(offsets32, cfg, t, h, w):
    """The reference tape (absolute fp64 centres) that the fp32 device tape encodes."""
    rows = offsets32.shape[0]
    nh, nw = (h - 1) // cfg.stride0 + 1, (w - 1) // cfg.stride0 + 1
    r = np.arange(rows)
    base = np.stack([r // (nh * nw), ((r // nw) % nh) * cfg.stride0, (r % nw) * cfg.stride0], -1)
    return base[:, None, :].astype(np.float64) + offsets32.astype(np.float32).astype(np.float64)


def abs_chains(chains_abs64, cfg, t, h, w, offsets):
    """fp64 reference chains -> fp32 relative device chains -> back to absolute fp64."""
    rel = rel_chains(chains_abs64, cfg, t, h, w, offsets).astype(np.float32).astype(np.float64)
    return rel_chains_inverse(rel, chains_abs64, cfg, t, h, w, offsets)


def rel_chains_inverse(rel, chains_abs64, cfg, t, h, w, offsets):
    out = rel.copy()
    if out.size == 0:
        return out
    back = rel_chains(np.zeros_like(chains_abs64), cfg, t, h, w, offsets)  # = -q on used links
    out[..., 0] -= back[..., 0]
    out[..., 1] -= back[..., 1]
    return out


@pytest.mark.parametrize("name", ["c2_mini", "c4_mini", "stride_half", "zero_flow"])
def test_golden_backward(name, port):
    """Stage-isolated on the reference's own tape.  The device tape is fp32 (offsets, relative
    chain links); identical inputs for the backward therefore means the same fp32 tape on
    both sides, and every gradient must then agree to REL_TOL.  Against the reference's fp64
    tape the flow gradients additionally carry the tape rounding (d(dS/dy)/dy ~ 2*sum(dk/dy)^2
    times ~2e-7 px): that distance is bounded separately at 1e-4."""
    z, cfg = load(name)
    t, h, w, _ = z["q"].shape
    dq, dk, dff, dbf = gpu_bwd(z["q"], z["k"], cfg, z["offsets"], z["chains"], z["grad_sims"])
    same = port.search_bwd(z["q"], z["k"], cfg, centers_from(z["offsets"], cfg, t, h, w),
                           abs_chains(z["chains"], cfg, t, h, w, z["offsets"]),
                           z["grad_sims"].astype(np.float64))
    for got, key in ((dq, "dq"), (dk, "dk"), (dff, "dfflow"), (dbf, "dbflow")):
        assert max_rel(got, same[key]) <= REL_TOL, (key, max_rel(got, same[key]))
        bound = REL_TOL if key in ("dq", "dk") else 1e-4
        assert max_rel(got, z[key]) <= bound, (key, max_rel(got, z[key]))


def test_random_backward_vs_oracle(port):
    rng = np.random.default_rng(100)
    done = 0
    for i in range(30):
        t = int(rng.integers(1, 4))
        h, w, f = int(rng.integers(5, 10)), int(rng.integers(5, 10)), int(rng.choice([1, 2, 4]))
        cfg = draw_cfg(rng, t, ws=(1, 3, 5), ps=(1, 3))
        q, k = video(port, t, h, w, f, 50000 + i), video(port, t, h, w, f, 51000 + i)
        ff, bf = flow(port, t, h, w, 52000 + i, 1.5), flow(port, t, h, w, 53000 + i, 1.5)
        try:
            fw = port.search_fwd(q, k, ff, bf, cfg)
        except Exception:
            continue
        g = f32(port.uniform(54000 + i, -1, 1, fw["sims"].size).reshape(fw["sims"].shape))
        want = port.search_bwd(q, k, cfg, fw["centers"], fw["chains"], g)
        got = gpu_bwd(q, k, cfg, fw["offsets"], fw["chains"], g)
        for a, key in zip(got, ("dq", "dk", "dfflow", "dbflow")):
            assert max_rel(a, want[key]) <= REL_TOL, (i, key, max_rel(a, want[key]))
        done += 1
    assert done >= 20


def test_zero_upstream_and_window_of_one(port):
    """test_gradcheck.cpp:24-65: zero upstream -> zero grads; ws=1 ip -> dQ = K, dK = Q."""
    S = snls_mod()
    q, k = video(port, 2, 6, 6, 2, 7), video(port, 2, 6, 6, 2, 8)
    ff, bf = flow(port, 2, 6, 6, 9, 1.0), flow(port, 2, 6, 6, 10, 1.0)
    cfg = S.SearchConfig(ws=3, wt=1, topl=2)
    r = S.shifted_nls_forward(dev(q), dev(k), dev(ff), dev(bf), cfg)
    for x in S.shifted_nls_backward(dev(np.zeros(r.sims.shape)), r, dev(q), dev(k)):
        assert np.all(host(x) == 0)
    q, k = video(port, 1, 5, 5, 3, 17), video(port, 1, 5, 5, 3, 18)
    cfg = S.SearchConfig(ws=1, wt=0, ps=1, topl=1, metric="ip")
    r = S.nls_forward(dev(q), dev(k), cfg)
    dq, dk, _, _ = S.shifted_nls_backward(dev(np.ones(r.sims.shape)), r, dev(q), dev(k))
    assert np.array_equal(host(dq), k) and np.array_equal(host(dk), q)


def test_backward_from_gpu_forward_tape(port):
    """End to end on the device tape (offsets + relative chains) of a wt=2 search."""
    S = snls_mod()
    z, cfg = load("c2_mini")
    q, k = dev(z["q"]), dev(z["k"])
    r = S.shifted_nls_forward(q, k, dev(z["fflow"]), dev(z["bflow"]), scfg(cfg))
    same = np.all(np.abs(host(r.offsets) - z["offsets"]) < 1e-5)
    if not same:
        pytest.skip("fp32 reordered a near-tie; covered stage-isolated")
    got = [host(x) for x in S.shifted_nls_backward(dev(z["grad_sims"]), r, q, k)]
    for a, key in zip(got, ("dq", "dk", "dfflow", "dbflow")):
        assert max_rel(a, z[key]) <= REL_TOL, key
