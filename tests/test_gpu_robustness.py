"""Robustness at the C boundary: huge finite flows (Middlebury's unknown-flow
marker is ~1e9-1e10) must neither fault nor corrupt, misaligned tensor pointers are rejected
before any vector load, the device error latch is read-and-cleared atomically, and a zero or
negative noise sigma aligns the clean clip as harness.cpp:95 does."""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import Cfg
from tests.gpu_util import compare_search, dev, host, oracle_ranked, scfg, snls_mod
from tests.helpers import REL_TOL, f32, max_rel, video

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("plan", ["tiled", "stream", "generic"])
def test_far_flow_inside_int_range_is_exact(port, plan):
    """Shifts of ~1.5e9 px (inside the reference's int range, below the +-(2^31 - 2^24)
    clamp) still match the oracle exactly: forward and wpsum."""
    S = snls_mod()
    t, h, w, f = 3, 12, 13, 32
    cfg = Cfg(ws=5, wt=1, ps=3, stride0=2, topl=4, metric="l2", softmax_scale=1.0 / 288)
    q, k = video(port, t, h, w, f, 71), video(port, t, h, w, f, 72)
    ff = f32(np.full((t, h, w, 2), 1.5e9) + port.uniform(73, 0, 1, t * h * w * 2).reshape(t, h, w, 2))
    bf = f32(np.full((t, h, w, 2), -1.5e9) + port.uniform(74, 0, 1, t * h * w * 2).reshape(t, h, w, 2))
    ref = oracle_ranked(port, q, k, ff, bf, cfg)
    ctx = S.context()
    ctx.set_search_kernel("stream" if plan == "stream" else "tiled")
    ctx.force_generic(plan == "generic")
    try:
        r = S.shifted_nls_forward(dev(q), dev(k), dev(ff), dev(bf), scfg(cfg), want_weights=True, ctx=ctx)
    finally:
        ctx.set_search_kernel("auto")
        ctx.force_generic(False)
    compare_search(r, ref, cfg, q, k, label=f" far-flow {plan}")
    v = video(port, t, h, w, f, 75)
    out, cnt = S.wpsum(dev(v), r.weights, r.offsets, scfg(cfg))
    want, wc = port.wpsum(v, host(r.weights), host(r.offsets), cfg)
    assert np.array_equal(host(cnt), wc)
    # offsets of 1.5e9 hold only ~128 px of fp32 resolution: compare against the oracle on
    # the device's own (fp32) offsets, which both sides then read identically
    assert max_rel(host(out), want) <= REL_TOL


def test_non_representable_flow_does_not_fault(port):
    """1e10 px (beyond int32; the reference's own conversion is undefined there): the kernels
    must finish without a device fault and the context must stay usable."""
    S = snls_mod()
    t, h, w, f = 2, 10, 10, 4
    cfg = S.SearchConfig(ws=3, wt=1, ps=3, stride0=2, topl=2)
    q = dev(video(port, t, h, w, f, 81))
    ff = dev(np.full((t, h, w, 2), 1e10))
    r = S.shifted_nls_forward(q, q, ff, ff, cfg, want_weights=True)
    out, cnt = S.wpsum(q, r.weights, r.offsets, cfg)
    S.shifted_nls_backward(dev(np.ones(r.sims.shape)), r, q, q)
    import torch

    torch.cuda.synchronize()
    assert np.all(np.isfinite(host(r.sims)))
    # the context still works afterwards
    r2 = S.nls_forward(q, q, cfg)
    assert np.all(np.isfinite(host(r2.sims)))


def test_misaligned_pointers_are_rejected(port):
    import torch

    S = snls_mod()
    base = dev(video(port, 1, 6, 6, 5, 91).reshape(-1))
    view = base[1:1 + 6 * 6 * 4].view(1, 6, 6, 4)  # contiguous, 4 bytes past alignment
    cfg = S.SearchConfig(ws=3, ps=1, topl=1)
    with pytest.raises(S.SnlsError, match="aligned"):
        S.nls_forward(view, view, cfg)
    # and at the C-ABI itself (no Python check in between)
    L = S.lib()
    c = S._cfg(cfg)
    sims = torch.empty((36, 1), device="cuda")
    offs = torch.empty((36, 1, 3), device="cuda")
    rc = L.snls_search_fwd(S.context().h, C.byref(c), S._Dims(1, 6, 6, 4), C.c_void_p(view.data_ptr()),
                           C.c_void_p(view.data_ptr()), None, None, 0, C.c_void_p(sims.data_ptr()),
                           C.c_void_p(offs.data_ptr()), None, None)
    assert rc == 4 and b"aligned" in L.snls_last_error()
    torch.cuda.synchronize()  # no sticky fault


def test_latch_is_taken_once(port):
    S = snls_mod()
    with pytest.raises(S.DomainError, match="non-finite"):
        S.softmax_rows(dev(np.array([[np.inf, 0.0]])), 1.0)
    S.context().sync_check()  # cleared by the take: a second check is clean
    w = host(S.softmax_rows(dev(np.array([[1.0, 0.0]])), 1.0))
    assert abs(w.sum() - 1.0) < 1e-6


def test_align_frames_nonpositive_sigma_uses_clean(port):
    S = snls_mod()
    t, h, w, f = 3, 12, 12, 3
    clean = np.floor(port.uniform(5, 0, 256, t * h * w * f)).reshape(t, h, w, f).astype(np.float32)
    cfg = S.SearchConfig(ws=5, wt=0, ps=3, stride0=2, topl=1, metric="l2", softmax_scale=1.0)
    a = S.align_frames(clean, cfg, flow_source=0, sigma=0.0, seed=1)
    b = S.align_frames(clean, cfg, flow_source=0, sigma=-3.0, seed=1)
    assert np.array_equal(a["aligned"], b["aligned"])
    assert np.array_equal(a["frame_psnr"], b["frame_psnr"])
