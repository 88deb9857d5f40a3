"""The two-pass patch wpsum (csrc/aggregate.cu wpsum_patch_kernel + wpsum_combine_kernel: the
plan for ps 5 / 7 at F 32 / 64) against the oracle's wpsum (aggregate.cpp:124-203), with the
offsets drawn directly: fractional shifts reaching past every border (reflected taps), frame
offsets of -1 / 0 / +1, every stride that keeps the output hole-free, the write-set counts
bit-exact, and a frame range equal to the same frames of the whole-clip call."""
import numpy as np
import pytest

from oracle.oracle import Cfg
from tests.gpu_util import dev, host, scfg, snls_mod
from tests.helpers import REL_TOL, f32, max_rel, video

pytestmark = pytest.mark.gpu

CASES = [(ps, f, s0) for ps in (5, 7) for f in (32, 64) for s0 in ((3, 4) if ps == 5 else (4, 5))]


def _selection(t, h, w, cfg, seed):
    rng = np.random.default_rng(seed)
    nh, nw = (h - 1) // cfg.stride0 + 1, (w - 1) // cfg.stride0 + 1
    rows = t * nh * nw
    qt = np.repeat(np.arange(t), nh * nw)[:, None]
    dt = rng.integers(-1, 2, size=(rows, cfg.topl))
    dt = np.clip(qt + dt, 0, t - 1) - qt
    offs = np.stack([dt, rng.uniform(-6, 6, (rows, cfg.topl)), rng.uniform(-6, 6, (rows, cfg.topl))], -1)
    wts = rng.uniform(0.0, 1.0, (rows, cfg.topl))
    return f32(wts / wts.sum(1, keepdims=True)), f32(offs)


@pytest.mark.parametrize("ps,f,s0", CASES, ids=[f"p{p}f{f}s{s}" for p, f, s in CASES])
def test_patch_wpsum_vs_oracle(port, ps, f, s0):
    S = snls_mod()
    t, h, w = 4, 29, 26
    cfg = Cfg(ws=5, wt=1, ps=ps, stride0=s0, topl=6, metric="l2", softmax_scale=1.0)
    v = video(port, t, h, w, f, 40 + ps + f + s0)
    wts, offs = _selection(t, h, w, cfg, 7 * ps + s0)
    out, cnt = S.wpsum(dev(v), dev(wts), dev(offs), scfg(cfg))
    want, wcnt = port.wpsum(v, wts, offs, cfg)
    assert np.array_equal(host(cnt), wcnt)
    err = max_rel(host(out), want)
    print(f"[patch wpsum p{ps} f{f} s{s0}] max rel {err:.2e}")
    assert err <= REL_TOL
    # a frame range gives exactly those frames of the whole-clip result
    nq = ((h - 1) // s0 + 1) * ((w - 1) // s0 + 1)
    o2, c2 = S.wpsum(dev(v), dev(wts[nq:3 * nq]), dev(offs[nq:3 * nq]), scfg(cfg), frames=(1, 3))
    assert np.array_equal(host(o2), host(out)[1:3])
    assert np.array_equal(host(c2), host(cnt)[1:3])


@pytest.mark.parametrize("ps,f,s0", CASES, ids=[f"p{p}f{f}s{s}" for p, f, s in CASES])
def test_pairs_wpsum_backward_vs_oracle(port, ps, f, s0):
    """wpsum_backward's channel-pair kernel (wpsum_bwd_pairs: ps 5/7 at F 32/64) against the
    oracle (aggregate.cpp:351-460): dV and dW, borders and cell completion in play."""
    S = snls_mod()
    t, h, w = 4, 29, 26
    cfg = Cfg(ws=5, wt=1, ps=ps, stride0=s0, topl=6, metric="l2", softmax_scale=1.0)
    v = video(port, t, h, w, f, 60 + ps + f + s0)
    wts, offs = _selection(t, h, w, cfg, 11 * ps + s0)
    _, cnt = S.wpsum(dev(v), dev(wts), dev(offs), scfg(cfg))
    go = video(port, t, h, w, f, 90 + s0)
    dv, dw = S.wpsum_backward(dev(go), cnt, dev(v), dev(wts), dev(offs), scfg(cfg))
    wdv, wdw = port.wpsum_bwd(go, host(cnt), v, wts, offs, cfg, deterministic=False)
    edv, edw = max_rel(host(dv), wdv), max_rel(host(dw), wdw)
    print(f"[pairs wpsum bwd p{ps} f{f} s{s0}] dV {edv:.2e} dW {edw:.2e}")
    assert edv <= REL_TOL and edw <= REL_TOL
