"""GPU checks at the BASELINE configs' FULL sizes (c2 and c4; the oracle cannot run these in
seconds), through size-independent properties of the operators:

* determinism: the forward (search + fused softmax + wpsum) is bitwise reproducible;
* adjointness of wpsum: out is linear in V and in the weights, so for any upstream G
  <G, wpsum(V)> = <V, dV(G)> = <W, dW(G)>  (wpsum_backward is the exact transpose);
* Euler's identity for the search backward: for the inner product sims are linear in Q and in
  K, so sum(dQ * Q) = sum(dK * K) = sum(g * sims); for negated squared L2 they are
  homogeneous of degree 2 in (Q, K) jointly, so sum(dQ * Q) + sum(dK * K) = 2 sum(g * sims);
* bit-exact agreement of the fused and the full-grid modes at full size.
Tolerances: fp32 accumulations over ~1e8 terms -- relative 1e-4 of the summed magnitudes."""
import numpy as np
import pytest

from tests.gpu_util import snls_mod

pytestmark = pytest.mark.gpu

FULL = {
    "c4": dict(T=10, H=256, W=256, F=32, cfg=dict(ws=11, wt=3, ps=3, stride0=2, topl=16, metric="l2",
                                                  softmax_scale=1 / 288), seed=100),
    "c2": dict(T=5, H=128, W=128, F=64, cfg=dict(ws=9, wt=2, ps=7, stride0=4, topl=10, metric="ip",
                                                 softmax_scale=1 / 3136), seed=11),
}


def _inputs(S, w):
    import torch

    T, H, W, F = w["T"], w["H"], w["W"], w["F"]
    v = torch.from_numpy(S.uniform_fill(w["seed"], -1, 1, T * H * W * F).reshape(T, H, W, F)).cuda()
    ff = torch.from_numpy(S.uniform_fill(w["seed"] + 100, -2, 2, T * H * W * 2).reshape(T, H, W, 2)).cuda()
    bf = torch.from_numpy(S.uniform_fill(w["seed"] + 200, -2, 2, T * H * W * 2).reshape(T, H, W, 2)).cuda()
    return v, ff, bf


def _dot(a, b):
    return float((a.double() * b.double()).sum())


def _scale(a, b):
    return float((a.double() * b.double()).abs().sum())


@pytest.mark.parametrize("name", sorted(FULL))
def test_fullsize_properties(name):
    import torch

    S = snls_mod()
    w = FULL[name]
    cfg = S.SearchConfig(**w["cfg"])
    v, ff, bf = _inputs(S, w)
    r = S.shifted_nls_forward(v, v, ff, bf, cfg, want_weights=True)
    out, cnt = S.wpsum(v, r.weights, r.offsets, cfg)
    # determinism and fused == full grid, bitwise
    r2 = S.shifted_nls_forward(v, v, ff, bf, cfg, want_weights=True)
    out2, _ = S.wpsum(v, r2.weights, r2.offsets, cfg)
    assert torch.equal(r.sims, r2.sims) and torch.equal(r.offsets, r2.offsets) and torch.equal(out, out2)
    g = S.shifted_nls_forward(v, v, ff, bf, cfg, mode=S.MODE_FULLGRID, want_weights=True)
    assert torch.equal(r.sims, g.sims) and torch.equal(r.offsets, g.offsets)
    # wpsum adjoint in V and in W
    G = torch.from_numpy(S.uniform_fill(w["seed"] + 300, -1, 1, v.numel()).reshape(v.shape)).cuda()
    dv, dw = S.wpsum_backward(G, cnt, v, r.weights, r.offsets, cfg)
    lhs = _dot(G, out)
    for rhs, sc in ((_dot(v, dv), _scale(v, dv)), (_dot(r.weights, dw), _scale(r.weights, dw))):
        assert abs(lhs - rhs) <= 1e-4 * max(sc, 1.0), (lhs, rhs, sc)
    # Euler identity for the search backward (Q = K = V aliased as in run_benchmark)
    gs = torch.from_numpy(S.uniform_fill(w["seed"] + 400, -1, 1, r.sims.numel()).reshape(r.sims.shape)).cuda()
    dq, dk, _, _ = S.shifted_nls_backward(gs, r, v, v)
    gsum = _dot(gs, r.sims)
    got = _dot(dq, v) + _dot(dk, v)
    want = 2.0 * gsum  # ip: 1 (Q) + 1 (K); l2: degree 2 jointly
    sc = _scale(dq, v) + _scale(dk, v)
    assert abs(got - want) <= 1e-4 * max(sc, 1.0), (got, want, sc)
