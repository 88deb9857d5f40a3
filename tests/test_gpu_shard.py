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
