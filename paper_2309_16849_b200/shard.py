"""Frame sharding of one video across ranks (BASELINE configs[4]).

A query at frame t only reads key/value frames t-wt .. t+wt and the flow frames between
(search.cpp:84-101, 300), and wpsum writes only into the query's own frame
(aggregate.cpp:197-198).  So rank r owns query frames [a, b) and needs the slab
[lo, hi) = [a-wt, b+wt) ∩ [0, T) of K/V/flows: the wt-frame halo on each side comes from the
neighbouring owners by point-to-point send/recv -- NCCL over NVLink on GPUs, gloo in the
CPU tests -- and no other collective touches the data path.  Searching the slab with query
rows restricted to [a-lo, b-lo) (snls_search_fwd_frames) gives exactly the rows the
unsharded search gives: frames outside the slab are either off the clip or out of reach.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ShardPlan:
    rank: int
    world: int
    T: int
    wt: int
    a: int   # owned query frames [a, b)
    b: int
    lo: int  # slab frames [lo, hi)
    hi: int

    @property
    def t0(self) -> int:  # owned frames inside the slab
        return self.a - self.lo

    @property
    def t1(self) -> int:
        return self.b - self.lo


def owned_range(T: int, world: int, rank: int):
    """Balanced contiguous split of T frames over `world` ranks."""
    per, rem = divmod(T, world)
    a = rank * per + min(rank, rem)
    return a, a + per + (1 if rank < rem else 0)


def plan(T: int, world: int, rank: int, wt: int) -> ShardPlan:
    if world > T:
        raise ValueError("frame sharding needs at least one frame per rank")
    a, b = owned_range(T, world, rank)
    return ShardPlan(rank, world, T, wt, a, b, max(0, a - wt), min(T, b + wt))


def transfers(p: ShardPlan):
    """(peer, frame range, 'send'|'recv') messages of rank p.rank, peers in ascending order.
    A peer's frames that fall in my slab are received; my frames inside a peer's slab are sent.
    Works for any shard length (halo may span several owners when b - a < wt)."""
    out = []
    for peer in range(p.world):
        if peer == p.rank:
            continue
        pa, pb = owned_range(p.T, p.world, peer)
        # frames I need from `peer`
        lo, hi = max(p.lo, pa), min(p.hi, pb)
        if lo < hi:
            out.append((peer, (lo, hi), "recv"))
        # frames `peer` needs from me
        q = plan(p.T, p.world, peer, p.wt)
        lo, hi = max(q.lo, p.a), min(q.hi, p.b)
        if lo < hi:
            out.append((peer, (lo, hi), "send"))
    return out


def exchange(local, p: ShardPlan, group=None):
    """Assemble the slab [lo, hi) from `local` (the owned frames [a, b), frame-major tensor)
    with one batched send/recv per (peer, direction).  Returns the slab tensor."""
    import torch
    import torch.distributed as dist

    shape = (p.hi - p.lo,) + tuple(local.shape[1:])
    slab = torch.empty(shape, dtype=local.dtype, device=local.device)
    slab[p.a - p.lo:p.b - p.lo].copy_(local)
    ops = []
    for peer, (lo, hi), kind in transfers(p):
        if kind == "recv":
            ops.append(dist.P2POp(dist.irecv, slab[lo - p.lo:hi - p.lo], peer, group))
        else:
            ops.append(dist.P2POp(dist.isend, local[lo - p.a:hi - p.a].contiguous(), peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return slab


def exchange_async(slabs, p: ShardPlan, group=None):
    """Fill the halo frames of persistent slab tensors in place: every tensor in `slabs` is a
    frame-major [lo, hi) slab whose owned frames [a, b) are already in place; one batched
    send/recv per (peer, direction, tensor) is started and the work handles are returned
    (NCCL: wait() only orders the caller's stream after the transfer, so work enqueued
    before it -- the interior frames -- overlaps the exchange)."""
    import torch.distributed as dist

    ops = []
    for slab in slabs:
        for peer, (lo, hi), kind in transfers(p):
            view = slab[lo - p.lo:hi - p.lo]
            ops.append(dist.P2POp(dist.irecv if kind == "recv" else dist.isend, view, peer, group))
    return dist.batch_isend_irecv(ops) if ops else []


def interior_range(p: ShardPlan):
    """Owned query frames whose key/value/flow frames all lie in the owned range (no halo
    needed): [a + wt, b - wt) -- chain links read fflow qt..qt+dt-1 and bflow qt..qt+dt+1
    (search.cpp:84-101), wpsum reads v at qt + dt (aggregate.cpp:108)."""
    lo = min(p.a + p.wt, p.b)
    hi = max(p.b - p.wt, lo)
    return lo, hi


def search_aggregate_overlapped(slab_q, slab_k, slab_v, slab_ff, slab_bf, p: ShardPlan, cfg, out,
                                ctx=None, group=None, world=1, split=None):
    """One frame-sharded step with the halo exchange overlapped: start the exchange of the
    K/V/flow halo, search + aggregate the interior frames (no halo needed) meanwhile, wait,
    then do the edge frames.  `out` = (sims, offsets, chains, weights, video, counts) for
    the owned frames; the slabs are persistent [lo, hi) tensors with the owned frames in
    place (Q only needs its owned frames)."""
    from . import snls as S

    sims, offs, chains, wts, vout, counts = out
    uniq = []  # aliased slabs (Q = K = V) are exchanged once
    for x in (slab_k, slab_v, slab_ff, slab_bf):
        if all(x is not u for u in uniq):
            uniq.append(x)
    reqs = exchange_async(uniq, p, group) if world > 1 else []
    nq = sims.shape[0] // (p.b - p.a)

    def run(f0, f1):  # owned query frames [f0, f1)
        if f0 >= f1:
            return
        r0, r1 = (f0 - p.a) * nq, (f1 - p.a) * nq
        o = (sims[r0:r1], offs[r0:r1], None if chains is None else chains[r0:r1], wts[r0:r1])
        S.shifted_nls_forward(slab_q, slab_k, slab_ff, slab_bf, cfg, ctx=ctx, check=False, out=o,
                              frames=(f0 - p.lo, f1 - p.lo))
        S.wpsum(slab_v, wts[r0:r1], offs[r0:r1], cfg, ctx=ctx, check=False,
                out=(vout[f0 - p.a:f1 - p.a], counts[f0 - p.a:f1 - p.a]), frames=(f0 - p.lo, f1 - p.lo))

    split = world > 1 if split is None else split
    ia, ib = interior_range(p) if split else (p.a, p.b)
    run(ia, ib)
    for r in reqs:
        r.wait()
    run(p.a, ia)
    run(ib, p.b)


def reverse_exchange_add(slab_grads, p: ShardPlan, group=None):
    """The backward's halo step: gradients a rank accumulated into its
    halo frames (dK / dV / dFlow land in frames qt + dt, search.cpp:584-666;
    aggregate.cpp:412-460) belong to the owners of those frames.  Every halo range received
    in the forward is sent back; every range sent in the forward comes back from that peer
    as a partial sum and is added into the owned frames.  In place on the slab tensors;
    afterwards each rank's owned frames [t0, t1) hold the full gradient."""
    import torch
    import torch.distributed as dist

    ops, pending = [], []
    for g in slab_grads:
        for peer, (lo, hi), kind in transfers(p):
            view = g[lo - p.lo:hi - p.lo]
            if kind == "recv":  # my partial sums for the peer's frames go back to it
                ops.append(dist.P2POp(dist.isend, view.contiguous(), peer, group))
            else:  # the peer's partial sums for my frames
                buf = torch.empty_like(view)
                ops.append(dist.P2POp(dist.irecv, buf, peer, group))
                pending.append((view, buf))
    for r in (dist.batch_isend_irecv(ops) if ops else []):
        r.wait()
    for view, buf in pending:
        view.add_(buf)


def backward_shard(grad_sims, grad_out, res, counts, slab_q, slab_k, slab_v, p: ShardPlan, cfg,
                   ctx=None, group=None, world=1):
    """wpsum_backward + shifted_nls_backward for the owned rows/frames of a frame shard
    (frame-range entry points on the slab), then the reverse halo exchange.  Returns
    slab-shaped (dq, dk, dv, dfflow, dbflow) whose owned frames hold the full gradient
    (Q's halo frames carry nothing: queries read only their own frame), and dweights."""
    from . import snls as S

    fr = (p.t0, p.t1)
    dv, dw = S.wpsum_backward(grad_out, counts, slab_v, res.weights, res.offsets, cfg, ctx=ctx,
                              check=False, frames=fr)
    dq, dk, dff, dbf = S.shifted_nls_backward(grad_sims, res, slab_q, slab_k, ctx=ctx, check=False,
                                              frames=fr)
    if world > 1:
        reverse_exchange_add([dk, dv, dff, dbf], p, group)
    return dq, dk, dv, dff, dbf, dw


def search_aggregate_shard(q_local, k_slab, v_slab, ff_slab, bf_slab, p: ShardPlan, cfg, ctx=None,
                           check=True):
    """Search + fused softmax + wpsum for the owned frames on the device (C-ABI frame-range
    entry points).  q_local holds the owned frames only; Q's halo is never read."""
    import torch

    from . import snls as S

    q_slab = q_local
    if q_local.shape[0] != k_slab.shape[0]:
        q_slab = torch.zeros_like(k_slab)
        q_slab[p.t0:p.t1].copy_(q_local)
    res = S.shifted_nls_forward(q_slab, k_slab, ff_slab, bf_slab, cfg, want_weights=True,
                                frames=(p.t0, p.t1), ctx=ctx, check=check)
    out, counts = S.wpsum(v_slab, res.weights, res.offsets, cfg, frames=(p.t0, p.t1), ctx=ctx,
                          check=check)
    return res, out, counts
