"""GPU: the frame-range entry points behind frame sharding.  A rank's slab (owned frames plus
the wt-frame halo) searched/aggregated with frames=(t0, t1) must reproduce the unsharded
device results for those frames bit for bit (same kernels, same per-query arithmetic)."""
import numpy as np
import pytest

from oracle.oracle import Checker
from paper_2309_16849_b200 import shard
from tests.gpu_util import dev, host, snls_mod
from tests.helpers import flow, video

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("F,ps,ws,wt", [(8, 3, 5, 2), (32, 3, 11, 3), (16, 1, 9, 1)])
def test_slab_equals_unsharded(F, ps, ws, wt):
    S = snls_mod()
    P = Checker("port")
    T, H, W = 9, 20, 18
    cfg = S.SearchConfig(ws=ws, wt=wt, ps=ps, stride0=2, topl=6, metric="l2", softmax_scale=0.05)
    v = video(P, T, H, W, F, 11)
    ff, bf = flow(P, T, H, W, 12, 1.5), flow(P, T, H, W, 13, 1.5)
    full = S.shifted_nls_forward(dev(v), dev(v), dev(ff), dev(bf), cfg, want_weights=True)
    fout, fcnt = S.wpsum(dev(v), full.weights, full.offsets, cfg)
    nq = ((H - 1) // 2 + 1) * ((W - 1) // 2 + 1)
    for world in (2, 3):
        for rank in range(world):
            p = shard.plan(T, world, rank, wt)
            slab = lambda x: dev(x[p.lo:p.hi])  # noqa: E731
            res, out, cnt = shard.search_aggregate_shard(slab(v), slab(v), slab(v), slab(ff), slab(bf), p, cfg)
            rows = slice(p.a * nq, p.b * nq)
            assert np.array_equal(host(res.sims), host(full.sims)[rows])
            assert np.array_equal(host(res.offsets), host(full.offsets)[rows])
            assert np.array_equal(host(res.weights), host(full.weights)[rows])
            assert np.array_equal(host(out), host(fout)[p.a:p.b])
            assert np.array_equal(host(cnt), host(fcnt)[p.a:p.b])


@pytest.mark.parametrize("world", [2, 3, 4])
def test_overlapped_interior_then_edges_equals_unsharded(world):
    """The overlapped step (interior frames first, then the halo-dependent edge frames, each
    through the frame-range entry points) reproduces the unsharded rows bit for bit; the
    slabs are prefilled as the exchange would leave them."""
    import torch

    S = snls_mod()
    P = Checker("port")
    T, H, W, F = 11, 18, 20, 32
    cfg = S.SearchConfig(ws=9, wt=2, ps=3, stride0=2, topl=10, metric="l2", softmax_scale=1 / 288)
    v = video(P, T, H, W, F, 21)
    ff, bf = flow(P, T, H, W, 22, 2.0), flow(P, T, H, W, 23, 2.0)
    full = S.shifted_nls_forward(dev(v), dev(v), dev(ff), dev(bf), cfg, want_weights=True)
    fout, fcnt = S.wpsum(dev(v), full.weights, full.offsets, cfg)
    nq = ((H - 1) // 2 + 1) * ((W - 1) // 2 + 1)
    for rank in range(world):
        p = shard.plan(T, world, rank, cfg.wt)
        n = (p.b - p.a) * nq
        o = (torch.empty((n, 10), device="cuda"), torch.empty((n, 10, 3), device="cuda"), None,
             torch.empty((n, 10), device="cuda"), torch.empty((p.b - p.a, H, W, F), device="cuda"),
             torch.empty((p.b - p.a, H, W), device="cuda", dtype=torch.int32))
        sl = lambda x: dev(x[p.lo:p.hi])  # noqa: E731
        vs = sl(v)
        shard.search_aggregate_overlapped(vs, vs, vs, sl(ff), sl(bf), p, cfg, o, split=True)
        rows = slice(p.a * nq, p.b * nq)
        assert np.array_equal(host(o[0]), host(full.sims)[rows])
        assert np.array_equal(host(o[1]), host(full.offsets)[rows])
        assert np.array_equal(host(o[3]), host(full.weights)[rows])
        assert np.array_equal(host(o[4]), host(fout)[p.a:p.b])
        assert np.array_equal(host(o[5]), host(fcnt)[p.a:p.b])


@pytest.mark.parametrize("world", [2, 3])
def test_frame_range_backward_plus_reverse_halo_equals_unsharded(world):
    """Each rank runs wpsum_backward + shifted_nls_backward on its slab for its own rows
    (frame-range entry points); adding every rank's slab gradients into the clip -- what
    snls_reverse_halo_add does over NCCL -- gives the unsharded device gradients (fp32
    atomics in a different order: REL_TOL)."""
    import torch

    from tests.helpers import REL_TOL, max_rel

    S = snls_mod()
    P = Checker("port")
    T, H, W, F = 9, 18, 16, 32
    cfg = S.SearchConfig(ws=9, wt=2, ps=3, stride0=2, topl=10, metric="l2", softmax_scale=1 / 288)
    v = dev(video(P, T, H, W, F, 31))
    ff, bf = dev(flow(P, T, H, W, 32, 2.0)), dev(flow(P, T, H, W, 33, 2.0))
    nq = ((H - 1) // 2 + 1) * ((W - 1) // 2 + 1)
    gs = dev(P.uniform(34, -1, 1, T * nq * 10).reshape(T * nq, 10))
    go = dev(P.uniform(35, -1, 1, T * H * W * F).reshape(T, H, W, F))
    full = S.shifted_nls_forward(v, v, ff, bf, cfg, want_weights=True)
    _, cnt = S.wpsum(v, full.weights, full.offsets, cfg)
    want_dv, want_dw = S.wpsum_backward(go, cnt, v, full.weights, full.offsets, cfg)
    want = S.shifted_nls_backward(gs, full, v, v)
    acc = [torch.zeros_like(x) for x in (want[0], want[1], want_dv, want[2], want[3])]
    for rank in range(world):
        p = shard.plan(T, world, rank, cfg.wt)
        sv, sff, sbf = v[p.lo:p.hi].contiguous(), ff[p.lo:p.hi].contiguous(), bf[p.lo:p.hi].contiguous()
        res = S.shifted_nls_forward(sv, sv, sff, sbf, cfg, want_weights=True, frames=(p.t0, p.t1))
        _, c = S.wpsum(sv, res.weights, res.offsets, cfg, frames=(p.t0, p.t1))
        rows = slice(p.a * nq, p.b * nq)
        out = shard.backward_shard(gs[rows].contiguous(), go[p.a:p.b].contiguous(), res, c, sv, sv, sv,
                                   p, cfg)
        dq, dk, dv, dff, dbf, dw = out
        assert max_rel(host(dw), host(want_dw)[rows]) <= REL_TOL
        for a_, g in zip(acc, (dq, dk, dv, dff, dbf)):
            a_[p.lo:p.hi] += g
    for a_, w in zip(acc, (want[0], want[1], want_dv, want[2], want[3])):
        assert max_rel(host(a_), host(w)) <= REL_TOL


def test_nccl_communicator_world1_selfcheck():
    """The C-ABI's own NCCL communicator on the lease's single GPU: ncclCommInitRank over a
    fresh id, ncclCommCount == 1, a grouped ncclSend/ncclRecv to itself moves the bytes, the
    halo exchange and reverse halo are no-ops at world 1 (no peers), and the overlapped step
    through the communicator equals the plain step."""
    import torch

    S = snls_mod()
    P = Checker("port")
    comm = shard.Comm(shard.Comm.unique_id(), 0, 1)
    info = comm.info()
    assert info["nranks"] == 1 and info["nccl_version"] > 0
    src = torch.arange(1 << 20, device="cuda", dtype=torch.float32)
    dst = torch.zeros_like(src)
    comm.loopback(src, dst)
    torch.cuda.synchronize()
    assert torch.equal(src, dst)
    T, H, W, F = 6, 16, 16, 32
    cfg = S.SearchConfig(ws=9, wt=2, ps=3, stride0=2, topl=10, metric="l2", softmax_scale=1 / 288)
    v = dev(video(P, T, H, W, F, 41))
    ff, bf = dev(flow(P, T, H, W, 42, 2.0)), dev(flow(P, T, H, W, 43, 2.0))
    p = shard.plan(T, 1, 0, cfg.wt)
    assert shard.transfers(p) == []
    nq = ((H - 1) // 2 + 1) * ((W - 1) // 2 + 1)
    o = (torch.empty((T * nq, 10), device="cuda"), torch.empty((T * nq, 10, 3), device="cuda"), None,
         torch.empty((T * nq, 10), device="cuda"), torch.empty((T, H, W, F), device="cuda"),
         torch.empty((T, H, W), device="cuda", dtype=torch.int32))
    shard.search_aggregate_overlapped(v, v, v, ff, bf, p, cfg, o, comm=comm, split=True)
    full = S.shifted_nls_forward(v, v, ff, bf, cfg, want_weights=True)
    fout, _ = S.wpsum(v, full.weights, full.offsets, cfg)
    assert torch.equal(o[0], full.sims) and torch.equal(o[4], fout)
    g = torch.ones_like(v)
    comm.reverse_add([g], p)
    torch.cuda.synchronize()
    assert torch.equal(g, torch.ones_like(v))
    comm.close()
