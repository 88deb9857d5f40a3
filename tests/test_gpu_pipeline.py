"""GPU: the host-buffer pipeline (snls_pipeline_run) -- chunked H2D / kernels / D2H overlap --
returns exactly the device-resident path's results (same kernels, same per-row arithmetic),
for every chunk size, aliased and distinct Q/K/V, and zero flows; errors keep the
reference's types and messages."""
import numpy as np
import pytest

from oracle.oracle import Checker
from tests.gpu_util import dev, host, snls_mod
from tests.helpers import flow, video

pytestmark = pytest.mark.gpu


def _host_out(S, T, H, W, F, cfg):
    rows = S.query_grid(T, H, W, cfg.stride0)[0]
    L = cfg.topl
    return (np.zeros((rows, L), np.float32), np.zeros((rows, L, 3), np.float32),
            np.zeros((rows, L), np.float32), np.zeros((T, H, W, F), np.float32),
            np.zeros((T, H, W), np.int32))


@pytest.mark.parametrize("chunk", [1, 2, 3, 9])
@pytest.mark.parametrize("alias", [True, False])
def test_pipeline_equals_device_path(chunk, alias):
    S = snls_mod()
    P = Checker("port")
    T, H, W, F = 9, 22, 20, 32
    cfg = S.SearchConfig(ws=11, wt=3, ps=3, stride0=2, topl=16, metric="l2", softmax_scale=1 / 288)
    q = video(P, T, H, W, F, 41).astype(np.float32)
    k = q if alias else video(P, T, H, W, F, 42).astype(np.float32)
    v = q if alias else video(P, T, H, W, F, 43).astype(np.float32)
    ff = flow(P, T, H, W, 44, 2.0).astype(np.float32)
    bf = flow(P, T, H, W, 45, 2.0).astype(np.float32)
    r = S.shifted_nls_forward(dev(q), dev(k), dev(ff), dev(bf), cfg, want_weights=True)
    want_out, want_cnt = S.wpsum(dev(v), r.weights, r.offsets, cfg)
    sims, offs, wts, out, cnt = _host_out(S, T, H, W, F, cfg)
    pipe = S.Pipeline(cfg, (T, H, W, F), chunk_frames=chunk)
    pipe.run(q, k, v, ff, bf, sims=sims, offsets=offs, weights=wts, out=out, counts=cnt)
    assert np.array_equal(sims, host(r.sims))
    assert np.array_equal(offs, host(r.offsets))
    assert np.array_equal(wts, host(r.weights))
    assert np.array_equal(out, host(want_out))
    assert np.array_equal(cnt, host(want_cnt))
    # a second run on the same pipeline (buffers reused) is identical
    out2 = np.zeros_like(out)
    pipe.run(q, k, v, ff, bf, out=out2)
    assert np.array_equal(out2, out)


def test_pipeline_zero_flows_and_pinned_buffers():
    import torch

    S = snls_mod()
    P = Checker("port")
    T, H, W, F = 4, 16, 18, 64
    cfg = S.SearchConfig(ws=9, wt=2, ps=3, stride0=2, topl=10, metric="l2", softmax_scale=1 / 576)
    q = torch.from_numpy(video(P, T, H, W, F, 51).astype(np.float32)).pin_memory()
    r = S.nls_forward(q.cuda(), q.cuda(), cfg, want_weights=True)
    want_out, _ = S.wpsum(q.cuda(), r.weights, r.offsets, cfg)
    sims, offs, wts, out, cnt = _host_out(S, T, H, W, F, cfg)
    out_p = torch.zeros(out.shape).pin_memory()
    pipe = S.Pipeline(cfg, (T, H, W, F), chunk_frames=2)
    pipe.run(q, q, q, None, None, sims=sims, offsets=offs, out=out_p)
    assert np.array_equal(sims, host(r.sims))
    assert np.array_equal(out_p.numpy(), host(want_out))


def test_pipeline_errors():
    S = snls_mod()
    P = Checker("port")
    T, H, W, F = 2, 8, 8, 8
    q = video(P, T, H, W, F, 61).astype(np.float32)
    ff = flow(P, T, H, W, 62, 1.0).astype(np.float32)
    with pytest.raises(S.ConfigError, match="ws must be odd"):
        S.Pipeline(S.SearchConfig(ws=4), (T, H, W, F))
    # T = 2, wt = 1: every query sees 2 of 3 frames -> 18 < 20 valid entries
    pipe = S.Pipeline(S.SearchConfig(ws=3, wt=1, ps=1, topl=20), (T, H, W, F))
    with pytest.raises(S.ConfigError, match="topl exceeds the valid window entries"):
        pipe.run(q, q, q, ff, ff)
    bad = ff.copy()
    bad[1, 2, 3, 0] = np.inf
    pipe = S.Pipeline(S.SearchConfig(ws=3, wt=1, ps=1, topl=2), (T, H, W, F))
    with pytest.raises(S.DomainError, match="search fflow: flow holds a non-finite value"):
        pipe.run(q, q, q, bad, ff)


def test_pipeline_streaming_submit_wait():
    """Two clips in flight (submit/submit/wait/wait, then more than two submits in a row):
    every clip's results equal the synchronous path's."""
    S = snls_mod()
    P = Checker("port")
    T, H, W, F = 5, 18, 20, 32
    cfg = S.SearchConfig(ws=11, wt=3, ps=3, stride0=2, topl=16, metric="l2", softmax_scale=1 / 288)
    clips = [video(P, T, H, W, F, 70 + i).astype(np.float32) for i in range(5)]
    flows = [flow(P, T, H, W, 80 + i, 2.0).astype(np.float32) for i in range(5)]
    pipe = S.Pipeline(cfg, (T, H, W, F), chunk_frames=1)
    want = []
    for c, fl in zip(clips, flows):
        sims, offs, wts, out, cnt = _host_out(S, T, H, W, F, cfg)
        pipe.run(c, c, c, fl, fl, sims=sims, out=out)
        want.append((sims, out))
    got = [_host_out(S, T, H, W, F, cfg) for _ in clips]
    for i, (c, fl) in enumerate(zip(clips, flows)):  # a third submit waits for the oldest
        pipe.submit(c, c, c, fl, fl, sims=got[i][0], out=got[i][3])
    pipe.wait()
    pipe.wait()
    for (ws, wo), g in zip(want, got):
        assert np.array_equal(g[0], ws) and np.array_equal(g[3], wo)
