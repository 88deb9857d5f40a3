"""GPU parity: softmax_rows, wpsum (deterministic gather), gather_stack and wpsum backward
against the oracle (test_aggregate.cpp, test_gradcheck.cpp:162-196, acceptance crits 7/8)."""
import os

import numpy as np
import pytest

from oracle.oracle import Cfg
from tests.gpu_util import compare_search, dev, host, oracle_ranked, scfg, snls_mod
from tests.helpers import REL_TOL, draw_cfg, f32, flow, max_rel, video

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return z, Cfg(**eval(str(z["cfg"])))


@pytest.mark.parametrize("name", ["c2_mini", "c4_mini", "stride_half", "zero_flow"])
def test_golden_aggregate_stage_isolated(name):
    """Same weights and offsets as the reference -> wpsum, counts, gather_stack, backward."""
    S = snls_mod()
    z, cfg = load(name)
    if "wpsum" not in z:
        pytest.skip("no aggregation in this fixture")
    v, w, o = dev(z["v"]), dev(z["weights"]), dev(z["offsets"])
    out, counts = S.wpsum(v, w, o, scfg(cfg))
    assert np.array_equal(host(counts), z["counts"])
    assert max_rel(host(out), z["wpsum"]) <= REL_TOL
    assert max_rel(host(S.gather_stack(v, w, o, scfg(cfg))), z["stack"]) <= REL_TOL
    dv, dw = S.wpsum_backward(dev(z["grad_out"]), counts, v, w, o, scfg(cfg))
    assert max_rel(host(dv), z["dv"]) <= REL_TOL
    assert max_rel(host(dw), z["dweights"]) <= REL_TOL


def test_softmax_cases():
    """test_aggregate.cpp:71-125"""
    S = snls_mod()
    w = host(S.softmax_rows(dev(np.array([[-5.0], [0.0], [7.5]])), 10.0))
    assert np.all(w == 1.0)
    w = host(S.softmax_rows(dev(np.array([[0.0, 0.0]])), 3.7))
    assert np.allclose(w, 0.5, atol=1e-7)
    w = host(S.softmax_rows(dev(np.array([[2.0, 1.0, 0.0]])), 1.0))
    e2, e1 = np.exp(2.0), np.exp(1.0)
    assert max_rel(w[0], np.array([e2, e1, 1.0]) / (e2 + e1 + 1.0)) <= 1e-6
    from oracle.oracle import Checker

    s = f32(Checker("port").uniform(5, -40, 40, 50).reshape(10, 5))
    w = host(S.softmax_rows(dev(s), -10.0))
    assert np.all(w >= 0) and np.all(np.abs(w.sum(1) - 1) <= 1e-6)
    with pytest.raises(S.DomainError, match="non-finite"):
        S.softmax_rows(dev(np.array([[np.inf, 0.0]])), 1.0)


def test_identity_reproduces_video_exactly(port):
    """test_aggregate.cpp:127-146 and the gather_stack identity slice (278-297)."""
    S = snls_mod()
    v = video(port, 2, 6, 7, 2, 11)
    rows = 2 * 6 * 7
    cfg = S.SearchConfig(ws=3, ps=1, stride0=1, topl=1)
    out, counts = S.wpsum(dev(v), dev(np.ones((rows, 1))), dev(np.zeros((rows, 1, 3))), cfg)
    assert np.array_equal(host(out), v) and np.all(host(counts) == 1)
    st = S.gather_stack(dev(v), dev(np.ones((rows, 1))), dev(np.zeros((rows, 1, 3))), cfg)
    assert np.array_equal(host(st)[0], v)


def test_random_aggregation_vs_oracle(port):
    """Random searches feed realistic offsets (test_aggregate.cpp:44-67, 328-350)."""
    S = snls_mod()
    rng = np.random.default_rng(9300)
    for i in range(25):
        t = int(rng.integers(1, 4))
        h, w, f = int(rng.integers(5, 12)), int(rng.integers(5, 12)), int(rng.choice([1, 2, 4, 8]))
        cfg = draw_cfg(rng, t, ws=(3, 5), ps=(1, 3, 5), hole_free=True, max_topl=3)
        v, q = video(port, t, h, w, f, 700000 + i), video(port, t, h, w, f, 800000 + i)
        ff, bf = flow(port, t, h, w, 900 + i, 1.5), flow(port, t, h, w, 950 + i, 1.5)
        sr = port.search_fwd(q, v, ff, bf, cfg)
        wts = port.softmax_rows(sr["sims"], 1.0)
        want, counts = port.wpsum(v, wts, sr["offsets"], cfg)
        out, gc = S.wpsum(dev(v), dev(wts), dev(sr["offsets"]), scfg(cfg))
        assert np.array_equal(host(gc), counts) and np.all(counts >= 1)
        assert max_rel(host(out), want) <= REL_TOL
        st = host(S.gather_stack(dev(v), dev(wts), dev(sr["offsets"]), scfg(cfg)))
        assert max_rel(st, port.gather_stack(v, wts, sr["offsets"], cfg)) <= REL_TOL
        # criterion 8: sum over L / count reproduces wpsum
        assert max_rel(st.sum(0) / counts[..., None], host(out)) <= 1e-5
        go = f32(port.uniform(1000 + i, -1, 1, v.size).reshape(v.shape))
        dv, dw = S.wpsum_backward(dev(go), gc, dev(v), dev(wts), dev(sr["offsets"]), scfg(cfg))
        wdv, wdw = port.wpsum_bwd(go, counts, v, wts, sr["offsets"], cfg)
        assert max_rel(host(dv), wdv) <= REL_TOL and max_rel(host(dw), wdw) <= REL_TOL


def test_linearity_convexity_and_holes(port):
    S = snls_mod()
    z, cfg = load("c4_mini")
    v, w, o = z["v"].astype(np.float64), dev(z["weights"]), dev(z["offsets"])
    v2 = video(port, *v.shape, 42)
    a, _ = S.wpsum(dev(v), w, o, scfg(cfg))
    b, _ = S.wpsum(dev(v2), w, o, scfg(cfg))
    m, _ = S.wpsum(dev(f32(1.7 * v - 0.6 * v2)), w, o, scfg(cfg))
    assert max_rel(host(m), 1.7 * host(a) - 0.6 * host(b)) <= 1e-5
    # ps = 1: convex blends stay inside [min, max]  (test_aggregate.cpp:222-247)
    c = Cfg(ws=3, wt=1, ps=1, stride0=2, topl=3)
    q = video(port, 2, 9, 9, 2, 52)
    vv = video(port, 2, 9, 9, 2, 53)
    zf = np.zeros((2, 9, 9, 2))
    sr = port.search_fwd(q, vv, zf, zf, c)
    out, _ = S.wpsum(dev(vv), dev(port.softmax_rows(sr["sims"], 1.0)), dev(sr["offsets"]), scfg(c))
    assert host(out).min() >= vv.min() - 1e-6 and host(out).max() <= vv.max() + 1e-6
    with pytest.raises(S.ConfigError, match="hole-free"):
        S.wpsum(dev(np.zeros((1, 6, 6, 1))), dev(np.ones((36, 1))), dev(np.zeros((36, 1, 3))),
                S.SearchConfig(ws=3, ps=3, stride0=1, topl=1))
    bad = np.zeros((36, 1, 3))
    bad[3, 0, 0] = 5.0  # dt leaves the clip
    with pytest.raises(S.DomainError, match="offsets leave the clip"):
        S.wpsum(dev(np.zeros((1, 6, 6, 1))), dev(np.ones((36, 1))), dev(bad),
                S.SearchConfig(ws=3, ps=1, stride0=1, topl=1))


def test_wpsum_backward_zero_and_identity(port):
    """test_gradcheck.cpp:162-188"""
    S = snls_mod()
    v = video(port, 1, 6, 6, 2, 27)
    cfg = S.SearchConfig(ws=3, ps=1, stride0=1, topl=1)
    w, o = dev(np.ones((36, 1))), dev(np.zeros((36, 1, 3)))
    _, counts = S.wpsum(dev(v), w, o, cfg)
    dv, dw = S.wpsum_backward(dev(np.zeros_like(v)), counts, dev(v), w, o, cfg)
    assert np.all(host(dv) == 0) and np.all(host(dw) == 0)
    g = video(port, 1, 6, 6, 2, 28)
    dv, _ = S.wpsum_backward(dev(g), counts, dev(v), w, o, cfg)
    assert np.array_equal(host(dv), g)


def test_end_to_end_search_softmax_wpsum(port):
    """GPU search -> fused softmax -> GPU wpsum against the oracle chain (c4 miniature)."""
    S = snls_mod()
    z, cfg = load("c4_mini")
    q, k, v = dev(z["q"]), dev(z["k"]), dev(z["v"])
    r = S.shifted_nls_forward(q, k, dev(z["fflow"]), dev(z["bflow"]), scfg(cfg), want_weights=True)
    out, counts = S.wpsum(v, r.weights, r.offsets, scfg(cfg))
    assert np.array_equal(host(counts), z["counts"])
    # the device picks the reference's candidates on every row (compare_search), so the whole
    # chain -- fp32 sims, fused softmax, gather -- must hold the north star's 1e-5
    ranked = oracle_ranked(port, z["q"], z["k"], z["fflow"], z["bflow"], cfg)
    st = compare_search(r, ranked, cfg, z["q"], z["k"], label=" c4_mini e2e")
    assert st["mismatched"] == 0
    err = max_rel(host(out), z["wpsum"])
    assert err <= REL_TOL, err
