"""CPU (gloo, world size 2 and 3): frame sharding with a wt-frame halo.

Each rank owns a contiguous frame range, assembles its slab [a-wt, b+wt) ∩ [0, T) through
the shard plan of the C-ABI (snls_shard_plan / snls_shard_transfers) moved by a gloo
stand-in of the NCCL exchange (tests/shard_gloo.py), and computes its rows on the slab.  With the oracle as the compute the
sharded rows must equal the unsharded ones BIT FOR BIT: that pins the halo plan, the
exchange and the frame-range semantics the CUDA entry points (snls_*_frames) implement."""
import os
import socket

import numpy as np
import pytest

from paper_2309_16849_b200 import shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plan_partitions_and_transfers_pair_up():
    for T in (5, 8, 13, 64):
        for world in (1, 2, 3, 4, 8):
            if world > T:
                continue
            for wt in (0, 1, 2, 3):
                plans = [shard.plan(T, world, r, wt) for r in range(world)]
                owned = sorted(f for p in plans for f in range(p.a, p.b))
                assert owned == list(range(T))
                for p in plans:
                    assert p.lo == max(0, p.a - wt) and p.hi == min(T, p.b + wt)
                    for peer, rng, kind in shard.transfers(p):
                        other = {(q, r2, k2) for q, r2, k2 in shard.transfers(plans[peer])}
                        assert (p.rank, rng, "send" if kind == "recv" else "recv") in other
                    # the halo is exactly the slab minus the owned frames
                    recv = sorted(f for _, (lo, hi), k in shard.transfers(p) if k == "recv"
                                  for f in range(lo, hi))
                    assert recv == [f for f in range(p.lo, p.hi) if not p.a <= f < p.b]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, T, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle.oracle import Cfg, Checker
    from paper_2309_16849_b200 import shard as SH
    from tests import shard_gloo as G

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    P = Checker("port")
    H = W = 10
    F = 4
    cfg = Cfg(ws=3, wt=2, ps=3, stride0=2, stride1=1.0, topl=3, metric="l2", softmax_scale=0.1)
    # every rank can generate only its own frames (per-frame seeds)
    def frame(t, seed, lo, hi, c):
        return P.uniform(seed * 1000 + t, lo, hi, H * W * c).reshape(H, W, c)
    p = SH.plan(T, world, rank, cfg.wt)
    own_v = torch.tensor(np.stack([frame(t, 500, -1, 1, F) for t in range(p.a, p.b)]).astype(np.float32))
    own_ff = torch.tensor(np.stack([frame(t, 501, -1.5, 1.5, 2) for t in range(p.a, p.b)]).astype(np.float32))
    own_bf = torch.tensor(np.stack([frame(t, 502, -1.5, 1.5, 2) for t in range(p.a, p.b)]).astype(np.float32))
    v = G.exchange(own_v, p).double().numpy()
    ff = G.exchange(own_ff, p).double().numpy()
    bf = G.exchange(own_bf, p).double().numpy()
    res = P.search_fwd(v, v, ff, bf, cfg)          # Q = K = V, slab as a clip
    nq = ((H - 1) // cfg.stride0 + 1) * ((W - 1) // cfg.stride0 + 1)
    rows = slice(p.t0 * nq, p.t1 * nq)
    wts = P.softmax_rows(res["sims"], cfg.softmax_scale)
    out, counts = P.wpsum(v, wts, res["offsets"], cfg)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), slab=v, sims=res["sims"][rows],
             offsets=res["offsets"][rows], out=out[p.t0:p.t1], counts=counts[p.t0:p.t1],
             a=p.a, b=p.b, lo=p.lo, hi=p.hi)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,T", [(2, 7), (3, 8)])
def test_gloo_halo_exchange_matches_unsharded_oracle(tmp_path, world, T):
    import torch.multiprocessing as mp

    from oracle.oracle import Cfg, Checker

    mp.spawn(_worker, args=(world, _free_port(), T, str(tmp_path)), nprocs=world, join=True)
    P = Checker("port")
    H = W = 10
    F = 4
    cfg = Cfg(ws=3, wt=2, ps=3, stride0=2, stride1=1.0, topl=3, metric="l2", softmax_scale=0.1)

    def frame(t, seed, lo, hi, c):
        return P.uniform(seed * 1000 + t, lo, hi, H * W * c).reshape(H, W, c)
    v = np.stack([frame(t, 500, -1, 1, F) for t in range(T)]).astype(np.float32).astype(np.float64)
    ff = np.stack([frame(t, 501, -1.5, 1.5, 2) for t in range(T)]).astype(np.float32).astype(np.float64)
    bf = np.stack([frame(t, 502, -1.5, 1.5, 2) for t in range(T)]).astype(np.float32).astype(np.float64)
    full = P.search_fwd(v, v, ff, bf, cfg)
    wts = P.softmax_rows(full["sims"], cfg.softmax_scale)
    fout, fcounts = P.wpsum(v, wts, full["offsets"], cfg)
    nq = 25
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        a, b, lo, hi = int(z["a"]), int(z["b"]), int(z["lo"]), int(z["hi"])
        assert np.array_equal(z["slab"], v[lo:hi])                    # halo frames arrived intact
        assert np.array_equal(z["sims"], full["sims"][a * nq:b * nq])   # bitwise, not approx
        assert np.array_equal(z["offsets"], full["offsets"][a * nq:b * nq])
        assert np.array_equal(z["out"], fout[a:b]) and np.array_equal(z["counts"], fcounts[a:b])


def test_interior_range_needs_no_halo():
    for T in (6, 9, 64):
        for world in (2, 3, 8):
            if world > T:
                continue
            for wt in (1, 2, 3):
                for r in range(world):
                    p = shard.plan(T, world, r, wt)
                    ia, ib = shard.interior_range(p)
                    assert p.a <= ia <= ib <= p.b
                    for qt in range(ia, ib):  # every frame a query can read is owned
                        assert p.a <= qt - wt and qt + wt < p.b


def _async_worker(rank, world, port, T, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2309_16849_b200 import shard as SH
    from tests import shard_gloo as G

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    p = SH.plan(T, world, rank, 2)
    full = torch.arange(T * 6, dtype=torch.float32).reshape(T, 3, 2) + 0.5
    slab = torch.full((p.hi - p.lo, 3, 2), -1.0)
    slab[p.t0:p.t1] = full[p.a:p.b]
    flow = torch.full((p.hi - p.lo, 3, 2), -2.0)
    flow[p.t0:p.t1] = -full[p.a:p.b]
    G.exchange_inplace([slab, flow], p)
    np.savez(os.path.join(out_dir, f"a{rank}.npz"), slab=slab.numpy(), flow=flow.numpy(),
             want=full[p.lo:p.hi].numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,T", [(2, 6), (3, 7), (4, 9)])
def test_gloo_inplace_async_exchange(tmp_path, world, T):
    import torch.multiprocessing as mp

    mp.spawn(_async_worker, args=(world, _free_port(), T, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        z = np.load(tmp_path / f"a{r}.npz")
        assert np.array_equal(z["slab"], z["want"]) and np.array_equal(z["flow"], -z["want"])


def _bwd_worker(rank, world, port, T, out_dir):
    """Sharded backward through the oracle on each slab (owned rows only: zero upstream
    gradient elsewhere), then the reverse halo exchange."""
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle.oracle import Cfg, Checker
    from paper_2309_16849_b200 import shard as SH
    from tests import shard_gloo as G

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    P = Checker("port")
    H = W = 10
    F = 4
    cfg = Cfg(ws=3, wt=2, ps=3, stride0=2, stride1=1.0, topl=3, metric="l2", softmax_scale=0.1)
    v, ff, bf, gs, go = _bwd_inputs(P, T, H, W, F)
    p = SH.plan(T, world, rank, cfg.wt)
    nq = 25
    sv, sff, sbf = v[p.lo:p.hi], ff[p.lo:p.hi], bf[p.lo:p.hi]
    res = P.search_fwd(sv, sv, sff, sbf, cfg)
    wts = P.softmax_rows(res["sims"], cfg.softmax_scale)
    _, counts = P.wpsum(sv, wts, res["offsets"], cfg)
    g_s = np.zeros_like(res["sims"])
    g_s[p.t0 * nq:p.t1 * nq] = gs[p.a * nq:p.b * nq]
    g_o = np.zeros_like(sv)
    g_o[p.t0:p.t1] = go[p.a:p.b]
    # the owned frames' counts are the unsharded counts; halo frames carry zero gradient
    dv, _ = P.wpsum_bwd(g_o, counts, sv, wts, res["offsets"], cfg)
    gb = P.search_bwd(sv, sv, cfg, res["centers"], res["chains"], g_s)
    grads = [torch.tensor(x) for x in (gb["dk"], dv, gb["dfflow"], gb["dbflow"])]
    G.reverse_exchange_add(grads, p)
    np.savez(os.path.join(out_dir, f"b{rank}.npz"), dq=gb["dq"][p.t0:p.t1],
             **{n: g[p.t0:p.t1].numpy() for n, g in zip(("dk", "dv", "dff", "dbf"), grads)},
             a=p.a, b=p.b)
    dist.barrier()
    dist.destroy_process_group()


def _bwd_inputs(P, T, H, W, F):
    def frame(t, seed, lo, hi, c):
        return P.uniform(seed * 1000 + t, lo, hi, H * W * c).reshape(H, W, c)
    f32 = lambda x: x.astype(np.float32).astype(np.float64)  # noqa: E731
    v = f32(np.stack([frame(t, 500, -1, 1, F) for t in range(T)]))
    ff = f32(np.stack([frame(t, 501, -1.5, 1.5, 2) for t in range(T)]))
    bf = f32(np.stack([frame(t, 502, -1.5, 1.5, 2) for t in range(T)]))
    gs = f32(P.uniform(503, -1, 1, T * 25 * 3).reshape(T * 25, 3))
    go = f32(P.uniform(504, -1, 1, T * H * W * F).reshape(T, H, W, F))
    return v, ff, bf, gs, go


@pytest.mark.parametrize("world,T", [(2, 7), (3, 8)])
def test_gloo_reverse_halo_backward_matches_unsharded_oracle(tmp_path, world, T):
    import torch.multiprocessing as mp

    from oracle.oracle import Cfg, Checker

    mp.spawn(_bwd_worker, args=(world, _free_port(), T, str(tmp_path)), nprocs=world, join=True)
    P = Checker("port")
    cfg = Cfg(ws=3, wt=2, ps=3, stride0=2, stride1=1.0, topl=3, metric="l2", softmax_scale=0.1)
    v, ff, bf, gs, go = _bwd_inputs(P, T, 10, 10, 4)
    res = P.search_fwd(v, v, ff, bf, cfg)
    wts = P.softmax_rows(res["sims"], cfg.softmax_scale)
    _, counts = P.wpsum(v, wts, res["offsets"], cfg)
    dv, _ = P.wpsum_bwd(go, counts, v, wts, res["offsets"], cfg)
    gb = P.search_bwd(v, v, cfg, res["centers"], res["chains"], gs)
    want = {"dq": gb["dq"], "dk": gb["dk"], "dv": dv, "dff": gb["dfflow"], "dbf": gb["dbflow"]}
    for r in range(world):
        z = np.load(tmp_path / f"b{r}.npz")
        a, b = int(z["a"]), int(z["b"])
        for n, w in want.items():  # fp64, summation order differs: tight tolerance
            assert np.allclose(z[n], w[a:b], rtol=1e-12, atol=1e-12), n


def _py_plan(T, world, rank, wt):
    """Independent restatement of the plan for checking the C-ABI's."""
    per, rem = divmod(T, world)
    a = rank * per + min(rank, rem)
    b = a + per + (1 if rank < rem else 0)
    return a, b, max(0, a - wt), min(T, b + wt)


def test_c_abi_plan_matches_independent_restatement():
    for T in (1, 5, 8, 13, 64):
        for world in (1, 2, 3, 4, 8):
            if world > T:
                with pytest.raises(Exception, match="at least one frame"):
                    shard.plan(T, world, 0, 2)
                continue
            for wt in (0, 1, 2, 3):
                for r in range(world):
                    p = shard.plan(T, world, r, wt)
                    assert (p.a, p.b, p.lo, p.hi) == _py_plan(T, world, r, wt)
                    want = []
                    for peer in range(world):
                        if peer == r:
                            continue
                        pa, pb, _, _ = _py_plan(T, world, peer, wt)
                        lo, hi = max(p.lo, pa), min(p.hi, pb)
                        if lo < hi:
                            want.append((peer, (lo, hi), "recv"))
                        _, _, qlo, qhi = _py_plan(T, world, peer, wt)
                        lo, hi = max(qlo, p.a), min(qhi, p.b)
                        if lo < hi:
                            want.append((peer, (lo, hi), "send"))
                    assert shard.transfers(p) == want


def test_comm_api_is_exported():
    from paper_2309_16849_b200 import snls as S

    L = S.lib()
    for name in ("snls_comm_unique_id", "snls_comm_init", "snls_comm_destroy", "snls_comm_info",
                 "snls_halo_exchange_async", "snls_halo_wait", "snls_reverse_halo_add",
                 "snls_comm_loopback", "snls_shard_plan", "snls_shard_transfers"):
        assert hasattr(L, name), name
