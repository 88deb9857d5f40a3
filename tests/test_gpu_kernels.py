"""GPU parity of every production register plan (the kernels the bench runs) at the BASELINE
configs' ws / ps / wt / F / metric, on frames small enough for the oracle and with borders
in play: the region-row tiled plan and the query-stationary streaming plan must each match
the oracle (search_fwd + fused softmax), and each plan's full-grid mode must equal its fused
mode bit for bit (test_search.cpp:317-347)."""
import numpy as np
import pytest

from oracle.oracle import Cfg
from tests.gpu_util import compare_search, dev, host, oracle_ranked, scfg, snls_mod
from tests.helpers import REL_TOL, flow, max_rel, video

pytestmark = pytest.mark.gpu

# (name, T, H, W, F, cfg) -- BASELINE configs[1], [3], [4] shapes with reduced frames
SHAPES = [
    ("c2", 5, 30, 28, 64, Cfg(ws=9, wt=2, ps=7, stride0=4, topl=10, metric="ip",
                              softmax_scale=1.0 / 3136)),
    ("c4", 6, 34, 30, 32, Cfg(ws=11, wt=3, ps=3, stride0=2, topl=16, metric="l2",
                              softmax_scale=1.0 / 288)),
    ("c5", 5, 28, 34, 64, Cfg(ws=9, wt=2, ps=3, stride0=2, topl=10, metric="l2",
                              softmax_scale=1.0 / 576)),
]

_cache = {}


def case(port, name, t, h, w, f, cfg):
    if name not in _cache:
        seed = {"c2": 11, "c4": 100, "c5": 500}[name]
        q = video(port, t, h, w, f, seed)
        k = q if name != "c2" else video(port, t, h, w, f, seed + 1)
        ff, bf = flow(port, t, h, w, seed + 3, 2.0), flow(port, t, h, w, seed + 4, 2.0)
        ref = oracle_ranked(port, q, k, ff, bf, cfg)
        wts = port.softmax_rows(ref["sims"][:, :cfg.topl], cfg.softmax_scale)
        _cache[name] = (q, k, ff, bf, ref, wts)
    return _cache[name]


@pytest.mark.parametrize("kernel,path", [("tiled", 1), ("stream", 3)])
@pytest.mark.parametrize("name,t,h,w,f,cfg", SHAPES, ids=[s[0] for s in SHAPES])
def test_register_plan_vs_oracle(port, kernel, path, name, t, h, w, f, cfg):
    S = snls_mod()
    q, k, ff, bf, ref, wts = case(port, name, t, h, w, f, cfg)
    ctx = S.context()
    ctx.set_search_kernel(kernel)
    try:
        args = (dev(q), dev(k), dev(ff), dev(bf), scfg(cfg))
        r = S.shifted_nls_forward(*args, want_weights=True, ctx=ctx)
        assert ctx.last_search_path() == path
        compare_search(r, ref, cfg, q, k, label=f" {name} {kernel}")
        assert max_rel(host(r.weights), wts) <= REL_TOL
        g = S.shifted_nls_forward(*args, mode=1, want_weights=True, ctx=ctx)
        for x, y in ((r.sims, g.sims), (r.offsets, g.offsets), (r.weights, g.weights)):
            assert np.array_equal(host(x), host(y)), "full grid != fused for this plan"
        again = S.shifted_nls_forward(*args, want_weights=True, ctx=ctx)
        assert np.array_equal(host(again.sims), host(r.sims))
        assert np.array_equal(host(again.offsets), host(r.offsets))
    finally:
        ctx.set_search_kernel("auto")


@pytest.mark.parametrize("name,t,h,w,f,cfg", SHAPES, ids=[s[0] for s in SHAPES])
def test_wpsum_at_baseline_shapes_stage_isolated(port, name, t, h, w, f, cfg):
    """wpsum / gather_stack at the BASELINE F / ps / stride0 (c5: F = 64 runs the query-centric
    kernel as two channel slices) against the oracle on the device's own selection."""
    S = snls_mod()
    q, k, ff, bf, ref, wts = case(port, name, t, h, w, f, cfg)
    v = video(port, t, h, w, f, 777)
    r = S.shifted_nls_forward(dev(q), dev(k), dev(ff), dev(bf), scfg(cfg), want_weights=True)
    out, cnt = S.wpsum(dev(v), r.weights, r.offsets, scfg(cfg))
    want, wcnt = port.wpsum(v, host(r.weights), host(r.offsets), cfg)
    assert np.array_equal(host(cnt), wcnt)
    assert max_rel(host(out), want) <= REL_TOL
    st = S.gather_stack(dev(v), r.weights, r.offsets, scfg(cfg))
    assert max_rel(host(st), port.gather_stack(v, host(r.weights), host(r.offsets), cfg)) <= REL_TOL


# every instantiated tiled kernel (search_tiled.cu launch_search_tiled): (ps, ws) x F x metric,
# i.e. each lane width G, each arithmetic path (float4 packed / float2 packed pairs, Q patch in
# shared memory) and both accumulation branches, on frames with borders in play
MATRIX = [(ps, ws, f, m)
          for ps, ws in ((3, 11), (3, 9), (7, 9), (1, 9), (3, 5), (1, 5))
          for f in ((16, 32, 64) if ps == 7 else (4, 8, 16, 32, 64))
          for m in ("ip", "l2")]


@pytest.mark.parametrize("ps,ws,f,metric", MATRIX, ids=[f"p{p}w{w}f{f}{m}" for p, w, f, m in MATRIX])
def test_tiled_plan_matrix_vs_oracle(port, ps, ws, f, metric):
    S = snls_mod()
    t, h, w = 3, 13, 15
    cfg = Cfg(ws=ws, wt=1, ps=ps, stride0=2, topl=min(10, ws * ws), metric=metric,
              softmax_scale=1.0 / (ps * ps * f))
    seed = 7000 + 97 * ps + 13 * ws + f + (1 if metric == "l2" else 0)
    q, k = video(port, t, h, w, f, seed), video(port, t, h, w, f, seed + 1)
    ff, bf = flow(port, t, h, w, seed + 2, 2.0), flow(port, t, h, w, seed + 3, 2.0)
    ref = oracle_ranked(port, q, k, ff, bf, cfg)
    ctx = S.context()
    ctx.set_search_kernel("tiled")
    try:
        r = S.shifted_nls_forward(dev(q), dev(k), dev(ff), dev(bf), scfg(cfg), ctx=ctx)
        assert ctx.last_search_path() == 1, "expected the tiled kernel for this shape"
    finally:
        ctx.set_search_kernel("auto")
    compare_search(r, ref, cfg, q, k, label=f" p{ps}w{ws}f{f}{metric}")


def test_c2_stride1_search_row(port):
    """SURVEY 8d's search-only c2 row at stride0 = 1 (every pixel a query), reduced frames."""
    S = snls_mod()
    cfg = Cfg(ws=9, wt=2, ps=7, stride0=1, topl=10, metric="ip", softmax_scale=1.0 / 3136)
    t, h, w, f = 5, 12, 14, 64
    q, k = video(port, t, h, w, f, 11), video(port, t, h, w, f, 12)
    ff, bf = flow(port, t, h, w, 14, 2.0), flow(port, t, h, w, 15, 2.0)
    ref = oracle_ranked(port, q, k, ff, bf, cfg)
    ctx = S.context()
    r = S.shifted_nls_forward(dev(q), dev(k), dev(ff), dev(bf), scfg(cfg), ctx=ctx)
    assert ctx.last_search_path() == 1
    compare_search(r, ref, cfg, q, k, label=" c2 stride0=1")


EXACT = [(11, 3, 32, "l2", 16), (11, 3, 32, "l2", 17), (11, 3, 32, "l2", 40), (11, 3, 32, "l2", 100),
         (9, 7, 64, "ip", 10), (9, 3, 64, "l2", 10), (9, 7, 32, "l2", 10), (11, 3, 16, "ip", 16)]


@pytest.mark.parametrize("ws,ps,f,metric,topl", EXACT, ids=[f"w{a}p{b}f{c}{d}k{e}" for a, b, c, d, e in EXACT])
def test_topl_sizes_bit_exact_on_integer_inputs(port, ws, ps, f, metric, topl):
    """L up to the register lists' 16 entries runs the tiled kernel, above it the generic one;
    on integer-valued videos and flows every sum is exact in fp32, so sims and offsets must
    equal the oracle bit for bit -- including the many exact ties, resolved by scan order
    (search.cpp:187-197) -- in the fused and the full-grid mode."""
    S = snls_mod()
    t, h, w = 3, 12, 13
    cfg = Cfg(ws=ws, wt=1, ps=ps, stride0=2, topl=topl, metric=metric, softmax_scale=1.0 / (ps * ps * f))
    seed = 8000 + 7 * topl + ps * 131 + f
    q = video(port, t, h, w, f, seed, lo=0.0, hi=16.0, integer=True)
    k = video(port, t, h, w, f, seed + 1, lo=0.0, hi=16.0, integer=True)
    ff = flow(port, t, h, w, seed + 2, 2.0, integer=True)
    bf = flow(port, t, h, w, seed + 3, 2.0, integer=True)
    ref = port.search_fwd(q, k, ff, bf, cfg)
    ctx = S.context()
    for mode in (0, 1):
        r = S.shifted_nls_forward(dev(q), dev(k), dev(ff), dev(bf), scfg(cfg), ctx=ctx, mode=mode)
        if mode == 0:
            assert ctx.last_search_path() == (1 if topl <= 16 else 0)
        compare_search(r, ref, cfg, exact=True)


@pytest.mark.parametrize("band", [1, 3, 5])
def test_band_raster_is_bitwise_the_plain_raster(port, band):
    """The temporally blocked CTA raster (common.cuh band_row; c5's default) only reorders
    independent queries: sims, offsets, weights and the full grid are bitwise the plain
    raster's.  Shapes with nw a multiple of the CTA's query count (the remap's condition)."""
    S = snls_mod()
    cases = [(5, 19, 32, 32, Cfg(ws=11, wt=3, ps=3, stride0=2, topl=16, metric="l2", softmax_scale=1 / 288)),
             (4, 17, 16, 64, Cfg(ws=9, wt=2, ps=3, stride0=1, topl=10, metric="l2", softmax_scale=1 / 576))]
    ctx = S.context()
    for t, h, w, f, cfg in cases:
        v = dev(video(port, t, h, w, f, 4400 + f))
        ff, bf = dev(flow(port, t, h, w, 4500, 2.0)), dev(flow(port, t, h, w, 4501, 2.0))
        outs = []
        for b in (0, band):
            ctx.set_search_band(b)
            try:
                r = S.shifted_nls_forward(v, v, ff, bf, scfg(cfg), want_weights=True, ctx=ctx)
                g = S.shifted_nls_forward(v, v, ff, bf, scfg(cfg), mode=1, ctx=ctx)
            finally:
                ctx.set_search_band(-1)
            outs.append([host(x) for x in (r.sims, r.offsets, r.weights, g.sims)])
        for x, y in zip(*outs):
            assert np.array_equal(x, y)


# query grids whose sides divide the CTA tile (the 4 x 4 / 2 x 2 query-tile raster of the tiled
# plan, search_tiled.cu SNLS_TILE2D*) -- the shapes above mostly take the linear raster
TILE_SHAPES = [
    ("c4-tile", 4, 16, 24, 32, Cfg(ws=11, wt=3, ps=3, stride0=2, topl=16, metric="l2", softmax_scale=1.0 / 288)),
    ("c2-tile", 3, 32, 32, 64, Cfg(ws=9, wt=2, ps=7, stride0=4, topl=10, metric="ip", softmax_scale=1.0 / 3136)),
    ("c5-tile", 3, 16, 16, 64, Cfg(ws=9, wt=2, ps=3, stride0=2, topl=10, metric="l2", softmax_scale=1.0 / 576)),
]


@pytest.mark.parametrize("name,t,h,w,f,cfg", TILE_SHAPES, ids=[s[0] for s in TILE_SHAPES])
def test_query_tile_raster_vs_oracle(port, name, t, h, w, f, cfg):
    S = snls_mod()
    q = video(port, t, h, w, f, 910)
    k = q if name != "c2-tile" else video(port, t, h, w, f, 911)
    ff, bf = flow(port, t, h, w, 912, 2.0), flow(port, t, h, w, 913, 2.0)
    ref = oracle_ranked(port, q, k, ff, bf, cfg)
    r = S.shifted_nls_forward(dev(q), dev(k), dev(ff), dev(bf), scfg(cfg), want_weights=True)
    st = compare_search(r, ref, cfg, q, k, label=f" {name}")
    assert st["mismatched"] == 0 or st["mismatched"] <= 0.01 * st["rows"]
    wts = port.softmax_rows(ref["sims"][:, :cfg.topl], cfg.softmax_scale)
    assert max_rel(host(r.weights), wts) <= REL_TOL
