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


TRAIN = [(5, 32, 3, "l2"), (7, 32, 4, "ip"), (5, 64, 4, "ip"), (7, 64, 5, "l2")]


@pytest.mark.parametrize("ps,f,s0,metric", TRAIN, ids=[f"p{p}f{f}s{s}{m}" for p, f, s, m in TRAIN])
def test_train_backward_interleaved_vs_separate_and_oracle(port, ps, f, s0, metric):
    """snls_train_bwd's interleaved launch (search + wpsum backward blocks side by side,
    search_bwd.cu train_bwd_interleaved) equals the two operators called separately and the
    oracle's backward operators (search.cpp:499-711, aggregate.cpp:351-460)."""
    from tests.helpers import flow

    S = snls_mod()
    t, h, w = 4, 21, 19
    cfg = Cfg(ws=5, wt=1, ps=ps, stride0=s0, topl=5, metric=metric, softmax_scale=0.05)
    q, k, v = (video(port, t, h, w, f, 300 + i + ps + f) for i in range(3))
    ff, bf = flow(port, t, h, w, 310 + ps, 1.5), flow(port, t, h, w, 311 + ps, 1.5)
    r = S.shifted_nls_forward(dev(q), dev(k), dev(ff), dev(bf), scfg(cfg), want_weights=True)
    cen, ch = S.search_tape64(r, dev(ff), dev(bf))
    rows, L = r.sims.shape
    g = f32(port.uniform(320, -1, 1, rows * L).reshape(rows, L))
    _, cnt = S.wpsum(dev(v), r.weights, r.offsets, scfg(cfg))
    go = video(port, t, h, w, f, 330)
    got = [host(x) for x in S.train_backward(dev(g), dev(go), cnt, r, dev(q), dev(k), dev(v), tape64=(cen, ch))]
    dq, dk, dff, dbf = [host(x) for x in S.shifted_nls_backward(dev(g), r, dev(q), dev(k), tape64=(cen, ch))]
    dv, dw = [host(x) for x in S.wpsum_backward(dev(go), cnt, dev(v), r.weights, r.offsets, scfg(cfg))]
    for a, b, name in zip(got, (dq, dk, dv, dff, dbf, dw), ("dq", "dk", "dv", "dff", "dbf", "dw")):
        assert max_rel(a, b) <= REL_TOL, (name, max_rel(a, b))
    sb = port.search_bwd(q, k, cfg, cen.cpu().numpy(), None if ch is None else ch.cpu().numpy(), g)
    wdv, wdw = port.wpsum_bwd(go, host(cnt), v, host(r.weights), host(r.offsets), cfg)
    for a, b, name in zip(got, (sb["dq"], sb["dk"], wdv, sb["dfflow"], sb["dbflow"], wdw),
                          ("dq", "dk", "dv", "dff", "dbf", "dw")):
        err = max_rel(a, b)
        print(f"[train bwd p{ps} f{f} s{s0} {metric}] {name} {err:.2e}")
        assert err <= REL_TOL, (name, err)


DET = [(3, 32, 2), (3, 8, 2), (5, 64, 3), (7, 32, 4), (9, 16, 5), (3, 96, 3), (1, 3, 1)]


@pytest.mark.parametrize("ps,f,s0", DET, ids=[f"p{p}f{f}s{s}" for p, f, s in DET])
def test_wpsum_backward_deterministic(port, ps, f, s0):
    """wpsum_backward in the reference's deterministic mode (aggregate.cpp:439-450; here int64
    fixed point): bitwise identical on repeated runs and within 1e-5 of the oracle -- through
    each kernel family (channel pairs, one channel per lane with 1 / 3 slices, the generic
    per-entry kernel at ps 9)."""
    S = snls_mod()
    t, h, w = 3, 23, 21
    cfg = Cfg(ws=3, wt=1, ps=ps, stride0=s0, topl=4, metric="l2", softmax_scale=1.0)
    v = video(port, t, h, w, f, 500 + ps + f)
    wts, offs = _selection(t, h, w, cfg, 13 * ps + s0)
    _, cnt = S.wpsum(dev(v), dev(wts), dev(offs), scfg(cfg))
    go = video(port, t, h, w, f, 510 + s0)
    a = [host(x) for x in S.wpsum_backward(dev(go), cnt, dev(v), dev(wts), dev(offs), scfg(cfg),
                                           deterministic=True)]
    b = [host(x) for x in S.wpsum_backward(dev(go), cnt, dev(v), dev(wts), dev(offs), scfg(cfg),
                                           deterministic=True)]
    assert all(np.array_equal(x, y) for x, y in zip(a, b)), "deterministic wpsum_backward differs"
    wdv, wdw = port.wpsum_bwd(go, host(cnt), v, wts, offs, cfg, deterministic=True)
    edv, edw = max_rel(a[0], wdv), max_rel(a[1], wdw)
    print(f"[det wpsum bwd p{ps} f{f} s{s0}] dV {edv:.2e} dW {edw:.2e}")
    assert edv <= REL_TOL and edw <= REL_TOL


def test_train_backward_deterministic_is_bitwise_reproducible(port):
    """snls_train_bwd with SNLS_BWD_DETERMINISTIC: every gradient (dQ, dK, dV, dW, flows)
    bitwise identical across runs (both operators in fixed-point mode)."""
    from tests.helpers import flow

    S = snls_mod()
    t, h, w, f = 4, 21, 19, 64
    cfg = Cfg(ws=5, wt=2, ps=7, stride0=4, topl=5, metric="ip", softmax_scale=0.05)
    q, k, v = (video(port, t, h, w, f, 600 + i) for i in range(3))
    ff, bf = flow(port, t, h, w, 610, 1.5), flow(port, t, h, w, 611, 1.5)
    r = S.shifted_nls_forward(dev(q), dev(k), dev(ff), dev(bf), scfg(cfg), want_weights=True)
    cen, ch = S.search_tape64(r, dev(ff), dev(bf))
    rows, L = r.sims.shape
    g = dev(f32(port.uniform(620, -1, 1, rows * L).reshape(rows, L)))
    _, cnt = S.wpsum(dev(v), r.weights, r.offsets, scfg(cfg))
    go = dev(video(port, t, h, w, f, 630))
    runs = [[host(x) for x in S.train_backward(g, go, cnt, r, dev(q), dev(k), dev(v), tape64=(cen, ch),
                                               deterministic=True)] for _ in range(2)]
    for x, y, name in zip(runs[0], runs[1], ("dq", "dk", "dv", "dff", "dbf", "dw")):
        assert np.array_equal(x, y), f"deterministic train_backward {name} differs"
    # the interleaved deterministic launch = the two deterministic operators called separately
    dq, dk, dff, dbf = [host(x) for x in S.shifted_nls_backward(g, r, dev(q), dev(k), tape64=(cen, ch),
                                                                 deterministic=True)]
    dv, dw = [host(x) for x in S.wpsum_backward(go, cnt, dev(v), r.weights, r.offsets, scfg(cfg),
                                                deterministic=True)]
    for a, b, name in zip(runs[0], (dq, dk, dv, dff, dbf, dw), ("dq", "dk", "dv", "dff", "dbf", "dw")):
        assert np.array_equal(a, b), (name, max_rel(a, b))
