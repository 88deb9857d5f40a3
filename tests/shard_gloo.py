"""TEST HARNESS ONLY -- a gloo stand-in for the NCCL halo exchange of
paper_2309_16849_b200/shard.py (snls_halo_exchange_async / snls_reverse_halo_add), so the
multi-rank frame-sharding logic runs on CPU tensors here: the same message plan
(shard.transfers, i.e. snls_shard_transfers) moved with torch.distributed point-to-point
calls over gloo.  The product path on GPUs is the C-ABI's NCCL exchange."""
from __future__ import annotations

from paper_2309_16849_b200.shard import ShardPlan, transfers


def exchange(local, p: ShardPlan, group=None):
    """Assemble the slab [lo, hi) from `local` (owned frames [a, b))."""
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
    for req in (dist.batch_isend_irecv(ops) if ops else []):
        req.wait()
    return slab


def exchange_inplace(slabs, p: ShardPlan, group=None):
    """Fill the halo frames of persistent [lo, hi) slabs in place (snls_halo_exchange_async)."""
    import torch.distributed as dist

    ops = []
    for slab in slabs:
        for peer, (lo, hi), kind in transfers(p):
            view = slab[lo - p.lo:hi - p.lo]
            ops.append(dist.P2POp(dist.irecv if kind == "recv" else dist.isend, view, peer, group))
    for req in (dist.batch_isend_irecv(ops) if ops else []):
        req.wait()


def reverse_exchange_add(slab_grads, p: ShardPlan, group=None):
    """snls_reverse_halo_add's semantics: halo partials go to their owners, owned frames +=
    the peers' partial sums."""
    import torch
    import torch.distributed as dist

    ops, pending = [], []
    for g in slab_grads:
        for peer, (lo, hi), kind in transfers(p):
            view = g[lo - p.lo:hi - p.lo]
            if kind == "recv":
                ops.append(dist.P2POp(dist.isend, view.contiguous(), peer, group))
            else:
                buf = torch.empty_like(view)
                ops.append(dist.P2POp(dist.irecv, buf, peer, group))
                pending.append((view, buf))
    for r in (dist.batch_isend_irecv(ops) if ops else []):
        r.wait()
    for view, buf in pending:
        view.add_(buf)
