"""Frame sharding of one video across GPUs (BASELINE configs[4]):
a thin ctypes wrapper over the C-ABI's shard plan and NCCL halo exchange
(csrc/comm.cu, include/snls_cuda.h) -- no torch.distributed on the data path.

A query at frame t only reads key/value frames t-wt .. t+wt and the flow frames between
(search.cpp:84-101, 300), and wpsum writes only into the query's own frame
(aggregate.cpp:197-198).  So rank r owns query frames [a, b) and needs the slab
[lo, hi) = [a-wt, b+wt) ∩ [0, T) of K/V/flows: the wt-frame halo on each side comes from the
neighbouring owners by ncclSend/ncclRecv over NVLink.  Searching the slab with query rows
restricted to [a-lo, b-lo) (snls_search_fwd_frames) gives exactly the rows the unsharded
search gives: frames outside the slab are either off the clip or out of reach.

torch tensors are only the device buffers here; torch.distributed is used once, as the
out-of-band channel that hands rank 0's NCCL id to the other ranks (Comm.create).
The CPU tests run the same plan with a gloo stand-in exchange (tests/shard_gloo.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import snls as S


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


def _lib():
    L = S.lib()
    if not getattr(L, "_snls_comm_types", False):
        I, P = C.c_int, C.c_void_p
        L.snls_shard_plan.argtypes = [I, I, I, I, C.POINTER(I)]
        L.snls_shard_transfers.argtypes = [I, I, I, I, I] + [C.POINTER(I)] * 5
        L.snls_comm_unique_id.argtypes = [P]
        L.snls_comm_init.argtypes = [P, P, I, I, C.POINTER(P)]
        L.snls_comm_destroy.argtypes = [P]
        L.snls_comm_info.argtypes = [P, C.POINTER(I), C.POINTER(I)]
        L.snls_halo_exchange_async.argtypes = [P, I, I, I, C.POINTER(P), C.POINTER(C.c_int64)]
        L.snls_halo_wait.argtypes = [P]
        L.snls_reverse_halo_add.argtypes = [P, I, I, I, C.POINTER(P), C.POINTER(C.c_int64)]
        L.snls_comm_loopback.argtypes = [P, P, P, C.c_uint64]
        L._snls_comm_types = True
    return L


def plan(T: int, world: int, rank: int, wt: int) -> ShardPlan:
    """snls_shard_plan: balanced contiguous split; slab = owned frames +- wt, clipped."""
    out = (C.c_int * 4)()
    S._raise(_lib().snls_shard_plan(T, world, rank, wt, out))
    return ShardPlan(rank, world, T, wt, out[0], out[1], out[2], out[3])


def owned_range(T: int, world: int, rank: int):
    p = plan(T, world, rank, 0)
    return p.a, p.b


def transfers(p: ShardPlan):
    """(peer, (lo, hi), 'recv'|'send') messages of rank p.rank (snls_shard_transfers): a
    peer's frames inside my slab are received, my frames inside a peer's slab are sent;
    peers ascending, recv before send.  Any shard length (a halo may span several owners)."""
    cap = 4 * p.world + 4
    arr = [(C.c_int * cap)() for _ in range(4)]
    n = C.c_int()
    S._raise(_lib().snls_shard_transfers(p.T, p.world, p.rank, p.wt, cap, *arr, C.byref(n)))
    return [(arr[0][i], (arr[1][i], arr[2][i]), "recv" if arr[3][i] else "send") for i in range(n.value)]


def interior_range(p: ShardPlan):
    """Owned query frames whose key/value/flow frames all lie in the owned range (no halo
    needed): [a + wt, b - wt) -- chain links read fflow qt..qt+dt-1 and bflow qt..qt+dt+1
    (search.cpp:84-101), wpsum reads v at qt + dt (aggregate.cpp:108)."""
    lo = min(p.a + p.wt, p.b)
    hi = max(p.b - p.wt, lo)
    return lo, hi


class Comm:
    """An NCCL communicator of the C-ABI (snls_comm) bound to a context's device/stream."""

    def __init__(self, unique_id: bytes, rank: int, world: int, ctx=None):
        import torch

        self.ctx = ctx or S.context(torch.cuda.current_device())
        self.rank, self.world = rank, world
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        S._raise(_lib().snls_comm_init(self.ctx.h, buf, rank, world, C.byref(h)))
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        S._raise(_lib().snls_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def create(cls, rank: int, world: int, ctx=None):
        """Rank 0 makes the id; torch.distributed (already initialised) carries it to the
        other ranks -- the only use of torch.distributed here (control plane)."""
        uid = cls.unique_id() if rank == 0 else None
        if world > 1:
            import torch.distributed as dist

            box = [uid]
            dist.broadcast_object_list(box, src=0)
            uid = box[0]
        return cls(uid, rank, world, ctx)

    def info(self):
        n, v = C.c_int(), C.c_int()
        S._raise(_lib().snls_comm_info(self.h, C.byref(n), C.byref(v)))
        return {"nranks": n.value, "nccl_version": v.value}

    def close(self):
        if getattr(self, "h", None):
            _lib().snls_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _arrays(tensors, per_frame):
        n = len(tensors)
        ptrs = (C.c_void_p * max(n, 1))(*[S._ptr(t).value for t in tensors])
        sizes = (C.c_int64 * max(n, 1))(*[per_frame(t) for t in tensors])
        return n, ptrs, sizes

    def exchange_async(self, slabs, p: ShardPlan):
        """snls_halo_exchange_async on persistent [lo, hi) slabs (owned frames in place)."""
        n, ptrs, sizes = self._arrays(slabs, lambda t: t[0].numel() * t.element_size())
        S._raise(_lib().snls_halo_exchange_async(self.h, p.T, p.wt, n, ptrs, sizes))

    def wait(self):
        S._raise(_lib().snls_halo_wait(self.h))

    def reverse_add(self, slab_grads, p: ShardPlan):
        """snls_reverse_halo_add: halo partial gradients to their owners, owned frames += the
        peers' partial sums (in place)."""
        n, ptrs, sizes = self._arrays(slab_grads, lambda t: t[0].numel())
        S._raise(_lib().snls_reverse_halo_add(self.h, p.T, p.wt, n, ptrs, sizes))

    def loopback(self, src, dst):
        S._raise(_lib().snls_comm_loopback(self.h, S._ptr(src), S._ptr(dst),
                                           src.numel() * src.element_size()))


def search_aggregate_overlapped(slab_q, slab_k, slab_v, slab_ff, slab_bf, p: ShardPlan, cfg, out,
                                ctx=None, comm: Comm | None = None, split=None):
    """One frame-sharded step with the halo exchange overlapped: start the NCCL exchange of
    the K/V/flow halo, search + aggregate the interior frames (no halo needed) meanwhile,
    join, then do the edge frames.  `out` = (sims, offsets, chains, weights, video, counts)
    for the owned frames; the slabs are persistent [lo, hi) tensors with the owned frames in
    place (Q only needs its owned frames)."""
    sims, offs, chains, wts, vout, counts = out
    uniq = []  # aliased slabs (Q = K = V) are exchanged once
    for x in (slab_k, slab_v, slab_ff, slab_bf):
        if all(x is not u for u in uniq):
            uniq.append(x)
    if comm is not None:
        comm.exchange_async(uniq, p)
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

    split = comm is not None if split is None else split
    ia, ib = interior_range(p) if split else (p.a, p.b)
    run(ia, ib)
    if comm is not None:
        comm.wait()
    run(p.a, ia)
    run(ib, p.b)


def backward_shard(grad_sims, grad_out, res, counts, slab_q, slab_k, slab_v, p: ShardPlan, cfg,
                   ctx=None, comm: Comm | None = None):
    """wpsum_backward + shifted_nls_backward for the owned rows/frames of a frame shard
    (frame-range entry points on the slab), then the reverse halo (snls_reverse_halo_add).
    Returns slab-shaped (dq, dk, dv, dfflow, dbflow) whose owned frames hold the full
    gradient (Q's halo frames carry nothing: queries read only their own frame), and dW."""
    fr = (p.t0, p.t1)
    dv, dw = S.wpsum_backward(grad_out, counts, slab_v, res.weights, res.offsets, cfg, ctx=ctx,
                              check=False, frames=fr)
    dq, dk, dff, dbf = S.shifted_nls_backward(grad_sims, res, slab_q, slab_k, ctx=ctx, check=False,
                                              frames=fr)
    if comm is not None and p.world > 1:
        comm.reverse_add([dk, dv, dff, dbf], p)
    return dq, dk, dv, dff, dbf, dw


def search_aggregate_shard(q_local, k_slab, v_slab, ff_slab, bf_slab, p: ShardPlan, cfg, ctx=None,
                           check=True):
    """Search + fused softmax + wpsum for the owned frames on the device (C-ABI frame-range
    entry points).  q_local holds the owned frames only; Q's halo is never read."""
    import torch

    q_slab = q_local
    if q_local.shape[0] != k_slab.shape[0]:
        q_slab = torch.zeros_like(k_slab)
        q_slab[p.t0:p.t1].copy_(q_local)
    res = S.shifted_nls_forward(q_slab, k_slab, ff_slab, bf_slab, cfg, want_weights=True,
                                frames=(p.t0, p.t1), ctx=ctx, check=check)
    out, counts = S.wpsum(v_slab, res.weights, res.offsets, cfg, frames=(p.t0, p.t1), ctx=ctx,
                          check=check)
    return res, out, counts
