"""GPU parity: the sm_100a search forward (tiled stride1==1 path and generic path) against the
oracle, through the C-ABI.  Cases follow the reference's own suites (test_search.cpp,
acceptance.cpp crit 1/2) plus the BASELINE configs' fixtures (tests/golden)."""
import os

import numpy as np
import pytest

from oracle.oracle import Cfg
from tests.gpu_util import (compare_search, dev, gpu_search, host, oracle_ranked, rel_chains,
                            scfg, snls_mod)
from tests.helpers import REL_TOL, draw_cfg, f32, flow, max_rel, video

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return z, Cfg(**eval(str(z["cfg"])))


def test_c1_integer_is_bit_exact():
    """BASELINE configs[0] on 8-bit integer-valued videos: every fp32 sum is exact, so sims
    and offsets (incl. the exact border-reflection ties) must equal the reference bitwise."""
    z, cfg = load("c1_integer")
    for generic in (False, True):
        r = gpu_search(z["q"], z["k"], z["fflow"], z["bflow"], cfg, generic=generic)
        compare_search(r, z, cfg, exact=True)


@pytest.mark.parametrize("plan", ["tiled", "stream", "generic"])
def test_c1_uniform_offsets_bit_exact_on_every_row(plan):
    """BASELINE configs[0] itself (U[0,255) videos, integer flows): north_star and SURVEY 8d
    ask for bit-exact top-k indices, ties broken by the reference's index order -- asserted
    on all 12,288 rows, no near-tie exclusion (the reference's exact border-reflection ties
    included, search.cpp:187-197)."""
    S = snls_mod()
    z, cfg = load("c1_uniform")
    ctx = S.context()
    ctx.set_search_kernel("stream" if plan == "stream" else "tiled")
    try:
        r = gpu_search(z["q"], z["k"], z["fflow"], z["bflow"], cfg, generic=plan == "generic")
    finally:
        ctx.set_search_kernel("auto")
    assert np.array_equal(host(r.offsets), z["offsets"]), "c1 offsets differ from the reference"
    assert max_rel(host(r.sims), z["sims"]) <= REL_TOL
    st = compare_search(r, z, cfg, z["q"], z["k"], exact_ties=True, max_skip=0.0, label=" c1")
    assert st["mismatched"] == 0


@pytest.mark.parametrize("name", ["c2_mini", "c4_mini", "stride_half", "zero_flow"])
@pytest.mark.parametrize("generic", [False, True])
def test_golden_search(port, name, generic):
    z, cfg = load(name)
    r = gpu_search(z["q"], z["k"], z["fflow"], z["bflow"], cfg, generic=generic, weights=True)
    ranked = oracle_ranked(port, z["q"], z["k"], z["fflow"], z["bflow"], cfg)
    assert np.array_equal(ranked["sims"][:, :cfg.topl], z["sims"])  # port == reference golden
    compare_search(r, ranked, cfg, z["q"], z["k"], label=f" {name}")
    if cfg.wt > 1:
        t, h, w, _ = z["q"].shape
        ok = np.all(np.abs(host(r.offsets) - z["offsets"]) < 1e-4, axis=(1, 2))
        want = rel_chains(z["chains"], cfg, t, h, w, z["offsets"])[ok]
        got = host(r.chains)[ok]
        assert max_rel(got, want) <= REL_TOL
    if "weights" in z:
        assert max_rel(host(r.weights), z["weights"]) <= REL_TOL


def test_tiled_path_taken_for_baseline_shapes():
    S = snls_mod()
    z, cfg = load("c4_mini")
    ctx = S.context()
    gpu_search(z["q"], z["k"], z["fflow"], z["bflow"], cfg)
    assert ctx.last_search_path() == 1
    gpu_search(z["q"], z["k"], z["fflow"], z["bflow"], cfg, generic=True)
    assert ctx.last_search_path() == 0


def test_random_configs_vs_oracle(port):
    """fused / full-grid / generic / tiled all agree with the oracle (test_search.cpp:317-347)."""
    rng = np.random.default_rng(67)
    for i in range(40):
        t = int(rng.integers(1, 5))
        h, w = int(rng.integers(4, 14)), int(rng.integers(4, 14))
        f = int(rng.choice([1, 2, 3, 4, 8, 16]))
        cfg = draw_cfg(rng, t, ws=(1, 3, 5, 9), ps=(1, 3), s1=(1.0, 1.0, 0.5))
        q, k = video(port, t, h, w, f, 3000 + i), video(port, t, h, w, f, 4000 + i)
        ff, bf = flow(port, t, h, w, 5000 + i, 1.5), flow(port, t, h, w, 6000 + i, 1.5)
        try:
            ref = oracle_ranked(port, q, k, ff, bf, cfg)
        except Exception:
            continue
        for mode, generic in ((0, False), (0, True), (1, False)):
            r = gpu_search(q, k, ff, bf, cfg, mode=mode, generic=generic)
            compare_search(r, ref, cfg, q, k, label=f" random#{i} mode{mode} generic{int(generic)}")


def test_zero_flow_equals_plain_search_bitwise(port):
    """Criterion 1 (acceptance.cpp:109-140): zero flows reduce to nls_forward, bitwise."""
    S = snls_mod()
    rng = np.random.default_rng(11)
    for i in range(20):
        t = int(rng.integers(1, 4))
        h, w, f = int(rng.integers(3, 11)), int(rng.integers(3, 11)), int(rng.choice([1, 3, 4, 8]))
        cfg = draw_cfg(rng, t, ws=(1, 3, 5), ps=(1, 3))
        q, k = dev(video(port, t, h, w, f, 100000 + i)), dev(video(port, t, h, w, f, 200000 + i))
        zf = dev(np.zeros((t, h, w, 2)))
        try:
            a = S.shifted_nls_forward(q, k, zf, zf, scfg(cfg))
        except S.ConfigError:
            continue
        b = S.nls_forward(q, k, scfg(cfg))
        assert np.array_equal(host(a.sims), host(b.sims))
        assert np.array_equal(host(a.offsets), host(b.offsets))


def test_window_of_one_inner_product():
    """test_search.cpp:89-110"""
    S = snls_mod()
    from oracle.oracle import Checker

    P = Checker("port")
    q, k = video(P, 2, 4, 5, 3, 7), video(P, 2, 4, 5, 3, 8)
    r = S.nls_forward(dev(q), dev(k), S.SearchConfig(ws=1, wt=0, ps=1, topl=1, metric="ip"))
    dot = (q * k).sum(-1).reshape(-1)
    assert max_rel(host(r.sims)[:, 0], dot) <= 1e-6
    assert np.all(host(r.offsets) == 0)


def test_self_match_and_constructed_shift(port):
    """test_search.cpp:112-137 and 208-243"""
    S = snls_mod()
    q = video(port, 2, 6, 6, 2, 17)
    for ws in (3, 5):
        r = S.nls_forward(dev(q), dev(q), S.SearchConfig(ws=ws, ps=1, topl=1, metric="l2"))
        assert np.all(host(r.sims) == 0.0)
    base = video(port, 1, 8, 12, 2, 47, 0.0, 255.0)
    k = np.roll(base, 5, axis=2)
    zb = np.zeros((1, 8, 12, 2))
    for fx in (5.0, 4.0):
        ff = np.zeros((1, 8, 12, 2))
        ff[..., 1] = fx
        r = S.shifted_nls_forward(dev(base), dev(k), dev(ff), dev(zb),
                                  S.SearchConfig(ws=3, ps=1, topl=1, metric="l2"))
        sims, offs = host(r.sims).reshape(8, 12), host(r.offsets).reshape(8, 12, 3)
        for y in range(1, 7):
            for x in range(1, 6):
                assert sims[y, x] == 0.0 and offs[y, x, 2] == 5.0


def test_full_frame_window_is_global_argmax(port):
    """Criterion 2 (acceptance.cpp:142-200): ws = 2*max(h,w)-1 covers the frame."""
    rng = np.random.default_rng(13)
    for i in range(6):
        t, h, w, f = 1 + i % 2, int(rng.integers(4, 9)), int(rng.integers(4, 9)), 1 + i % 3
        q, k = video(port, t, h, w, f, 300000 + i), video(port, t, h, w, f, 400000 + i)
        cfg = Cfg(ws=2 * max(h, w) - 1, wt=0, ps=1, topl=1, metric="l2" if i % 2 else "ip")
        ref = port.search_fwd(q, k, np.zeros((t, h, w, 2)), np.zeros((t, h, w, 2)), cfg)
        r = gpu_search(q, k, None, None, cfg)
        assert max_rel(host(r.sims), ref["sims"]) <= 1e-6
        assert np.array_equal(host(r.offsets), ref["offsets"])


def test_determinism_across_runs():
    z, cfg = load("c4_mini")
    a = gpu_search(z["q"], z["k"], z["fflow"], z["bflow"], cfg, weights=True)
    b = gpu_search(z["q"], z["k"], z["fflow"], z["bflow"], cfg, weights=True)
    for x, y in ((a.sims, b.sims), (a.offsets, b.offsets), (a.weights, b.weights)):
        assert np.array_equal(host(x), host(y))


def test_replay_reproduces_sims():
    S = snls_mod()
    z, cfg = load("c2_mini")
    q, k = dev(z["q"]), dev(z["k"])
    r = S.shifted_nls_forward(q, k, dev(z["fflow"]), dev(z["bflow"]), scfg(cfg))
    rep = S.replay_similarities(r, q, k)
    assert max_rel(host(rep), host(r.sims)) <= REL_TOL


def test_top_l_selection_and_ties():
    """test_search.cpp:245-315"""
    S = snls_mod()
    sel, soff = S.top_l(dev(np.array([[3.0, 1.0, 2.0]])),
                        dev(np.array([[[0, 0, 0], [0, 1, 1], [0, 2, 2]]], np.float32)), 2)
    assert host(sel).tolist() == [[3.0, 2.0]] and host(soff)[0, 1, 2] == 2.0
    off = np.zeros((1, 4, 3), np.float32)
    off[0, :, 2] = np.arange(4)
    sel, soff = S.top_l(dev(np.full((1, 4), 5.0)), dev(off), 2)
    assert host(soff)[0, :, 2].tolist() == [0.0, 1.0]
    from oracle.oracle import Checker

    P = Checker("port")
    full = f32(P.uniform(57, -10, 10, 20 * 50).reshape(20, 50))
    offs = np.zeros((20, 50, 3))
    offs[:, :, 2] = np.arange(50)
    want_s, want_o = P.top_l(full, offs, 7)
    sel, soff = S.top_l(dev(full), dev(offs), 7)
    assert np.array_equal(host(sel), want_s) and np.array_equal(host(soff), want_o)
    with pytest.raises(S.ConfigError):
        S.top_l(dev(np.ones((1, 2))), dev(np.zeros((1, 2, 3))), 3)
    with pytest.raises(S.DomainError, match="fewer than L"):
        S.top_l(dev(np.array([[1.0, -np.inf]])), dev(np.zeros((1, 2, 3))), 2)


def test_search_grid_matches_oracle(port):
    S = snls_mod()
    z, cfg = load("c4_mini")
    grid, goff = S.search_grid(dev(z["q"]), dev(z["k"]), dev(z["fflow"]), dev(z["bflow"]), scfg(cfg))
    want, woff = port.search_full_grid(z["q"], z["k"], z["fflow"], z["bflow"], cfg)
    g = host(grid)
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(g), fin)
    assert max_rel(g[fin], want[fin]) <= REL_TOL


def test_errors_match_reference_contract(port):
    S = snls_mod()
    q = dev(video(port, 2, 6, 6, 1, 127))
    ff = dev(flow(port, 2, 6, 6, 129, 1.0))
    with pytest.raises(S.ConfigError, match="topl exceeds the valid window entries"):
        S.shifted_nls_forward(q, q, ff, ff, S.SearchConfig(ws=3, wt=1, ps=1, topl=27))
    with pytest.raises(S.ConfigError, match="ws must be odd"):
        S.shifted_nls_forward(q, q, ff, ff, S.SearchConfig(ws=4))
    bad = video(port, 2, 6, 6, 2, 1)
    bad[0, 0, 0, 0] = np.nan
    with pytest.raises(S.DomainError, match="search fflow: flow holds a non-finite value"):
        S.shifted_nls_forward(q, q, dev(bad), ff, S.SearchConfig(ws=3, ps=1, topl=1))
    with pytest.raises(S.DomainError, match="flow shape"):
        S.shifted_nls_forward(q, q, dev(np.zeros((2, 6, 5, 2))), ff, S.SearchConfig(ws=3))


@pytest.mark.parametrize("plan", ["tiled", "stream", "generic"])
def test_degenerate_shapes_and_far_flows(port, plan):
    """Edge cases the reference's reflect/shift code handles (tensor.cpp:23-29 period-2(n-1)
    mirror for ANY magnitude, n == 1 -> 0; search.cpp:72-122): 1-pixel frames, frames
    smaller than the window, stride0 beyond the frame, flows far outside the frame (many
    reflection folds), through every search plan, against the oracle."""
    S = snls_mod()
    cases = [  # (t, h, w, f, ws, wt, ps, s0, topl, flow magnitude)
        (2, 1, 1, 4, 3, 1, 1, 1, 2, 0.7),
        (3, 1, 7, 4, 5, 1, 3, 2, 3, 3.0),
        (2, 5, 4, 32, 11, 1, 3, 9, 4, 60.0),
        (4, 9, 11, 32, 11, 3, 3, 2, 16, 200.0),
        (3, 12, 10, 64, 9, 2, 7, 4, 10, 37.5),
        (2, 3, 3, 64, 9, 1, 3, 1, 5, 1e3),
    ]
    ctx = S.context()
    for i, (t, h, w, f, ws, wt, ps, s0, topl, mag) in enumerate(cases):
        cfg = Cfg(ws=ws, wt=wt, ps=ps, stride0=s0, topl=topl, metric="l2" if i % 2 else "ip",
                  softmax_scale=0.01)
        q, k = video(port, t, h, w, f, 910 + i), video(port, t, h, w, f, 920 + i)
        ff, bf = flow(port, t, h, w, 930 + i, mag), flow(port, t, h, w, 940 + i, mag)
        ref = oracle_ranked(port, q, k, ff, bf, cfg)
        ctx.set_search_kernel("stream" if plan == "stream" else "tiled")
        try:
            r = gpu_search(q, k, ff, bf, cfg, generic=plan == "generic")
        finally:
            ctx.set_search_kernel("auto")
        compare_search(r, ref, cfg, q, k, label=f" {plan} case{i}")


REPLAY_SHAPES = [  # (t, h, w, f, cfg): c4 / c5 / c2 lane layouts, both metrics, plus generic-only
    (5, 23, 21, 32, Cfg(ws=11, wt=3, ps=3, stride0=2, topl=16, metric="l2")),
    (4, 19, 22, 64, Cfg(ws=9, wt=2, ps=3, stride0=2, topl=10, metric="l2")),
    (4, 20, 18, 64, Cfg(ws=9, wt=2, ps=7, stride0=4, topl=10, metric="ip")),
    (3, 13, 15, 16, Cfg(ws=5, wt=1, ps=3, stride0=2, topl=6, metric="ip")),
    (3, 12, 11, 8, Cfg(ws=9, wt=1, ps=1, stride0=1, topl=10, metric="l2")),
    (3, 11, 12, 4, Cfg(ws=5, wt=1, ps=3, stride0=2, stride1=0.5, topl=5, metric="l2")),  # generic
]


@pytest.mark.parametrize("plan", ["tiled", "stream", "generic"])
@pytest.mark.parametrize("i", range(len(REPLAY_SHAPES)))
def test_replay_is_bitwise_the_forward_of_every_plan(port, plan, i):
    """replay_similarities from the fp64 tape (search.cpp:470-493; test_search.cpp:539-553:
    'replay reproduces the selected similarities exactly') through each plan's own per-slot
    arithmetic equals that plan's forward BIT FOR BIT -- on the reference's own tape too."""
    S = snls_mod()
    t, h, w, f, cfg = REPLAY_SHAPES[i]
    q, k = video(port, t, h, w, f, 9100 + i), video(port, t, h, w, f, 9200 + i)
    ff, bf = flow(port, t, h, w, 9300 + i, 2.0), flow(port, t, h, w, 9400 + i, 2.0)
    ctx = S.context()
    ctx.set_search_kernel("stream" if plan == "stream" else "tiled")
    ctx.force_generic(plan == "generic")
    try:
        dq, dk, dff, dbf = dev(q), dev(k), dev(ff), dev(bf)
        r = S.shifted_nls_forward(dq, dk, dff, dbf, scfg(cfg), ctx=ctx)
        cen, _ = S.search_tape64(r, dff, dbf, ctx=ctx)
        got = S.replay_similarities(r, dq, dk, ctx=ctx, centers=cen)  # 'auto': the plan just used
    finally:
        ctx.set_search_kernel("auto")
        ctx.force_generic(False)
    assert np.array_equal(host(got), host(r.sims)), (ctx.last_search_path(), np.abs(host(got) - host(r.sims)).max())
    # and the oracle's replay of the same tape agrees to the fp32 tolerance
    want = port.replay(q, k, cfg, cen.cpu().numpy())
    assert max_rel(host(got), want) <= REL_TOL
