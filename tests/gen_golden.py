"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libsnls_ref.so: the
unmodified /root/reference sources compiled by oracle/Makefile).

    python tests/gen_golden.py

Each fixture stores its inputs (fp32-representable, from the reference's UniformStream) and
the reference's fp64 outputs.  tests/test_oracle.py pins the plain-C restatement against
them bit for bit; the GPU tests compare the CUDA path against them at the stated tolerance.
The fixtures are committed because /root/reference does not exist on the GPU box.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Cfg, Checker  # noqa: E402
from tests.helpers import f32, flow, video  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def cfg_dict(c: Cfg):
    return dict(ws=c.ws, wt=c.wt, ps=c.ps, stride0=c.stride0, stride1=c.stride1, topl=c.topl,
                metric=c.metric, softmax_scale=c.softmax_scale)


def save(name, cfg, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, cfg=np.array(repr(cfg_dict(cfg))), **arrays)
    print(path, os.path.getsize(path))


def search_case(R, name, t, h, w, f, cfg, seeds, *, lo=-1.0, hi=1.0, integer=False, fmag=1.5,
                int_flow=False, aggregate=True, backward=True, zero_flow=False):
    q = video(R, t, h, w, f, seeds[0], lo, hi, integer)
    k = video(R, t, h, w, f, seeds[1], lo, hi, integer)
    if zero_flow:
        ff = np.zeros((t, h, w, 2))
        bf = np.zeros((t, h, w, 2))
    else:
        ff = flow(R, t, h, w, seeds[2], fmag, int_flow)
        bf = flow(R, t, h, w, seeds[3], fmag, int_flow)
    res = R.search_fwd(q, k, ff, bf, cfg)
    arrays = dict(q=q.astype(np.float32), k=k.astype(np.float32), fflow=ff.astype(np.float32),
                  bflow=bf.astype(np.float32), sims=res["sims"], offsets=res["offsets"],
                  chains=res["chains"])
    # one extra rank, to let parity tests exclude tie-adjacent rows (gradcheck_util.hpp:61-69)
    if cfg.topl < cfg.window_slots():
        c2 = Cfg(**{**cfg_dict(cfg), "topl": cfg.topl + 1})
        try:
            arrays["sims_lplus1"] = R.search_fwd(q, k, ff, bf, c2)["sims"]
        except Exception:
            pass
    if aggregate and cfg.hole_free():
        v = video(R, t, h, w, f, seeds[4], lo, hi, integer)
        wts = R.softmax_rows(res["sims"], cfg.softmax_scale)
        out, counts = R.wpsum(v, wts, res["offsets"], cfg)
        stack = R.gather_stack(v, wts, res["offsets"], cfg)
        arrays.update(v=v.astype(np.float32), weights=wts, wpsum=out, counts=counts, stack=stack)
        if backward:
            go = f32(R.uniform(seeds[5], -1, 1, v.size).reshape(v.shape))
            dv, dw = R.wpsum_bwd(go, counts, v, wts, res["offsets"], cfg)
            arrays.update(grad_out=go.astype(np.float32), dv=dv, dweights=dw)
    if backward:
        gs = f32(R.uniform(seeds[6], -1, 1, res["sims"].size).reshape(res["sims"].shape))
        g = R.search_bwd(q, k, cfg, res["centers"], res["chains"], gs)
        arrays.update(grad_sims=gs.astype(np.float32), dq=g["dq"], dk=g["dk"],
                      dfflow=g["dfflow"], dbflow=g["dbflow"])
    save(name, cfg, **arrays)


def main():
    os.makedirs(OUT, exist_ok=True)
    R = Checker("reference")
    # BASELINE configs[0]: 3x64x64x3, integer flow, ws9 wt1 ps1 k10 L2 (seeds 1-4)
    c1 = Cfg(ws=9, wt=1, ps=1, stride0=1, stride1=1.0, topl=10, metric="l2")
    search_case(R, "c1_integer", 3, 64, 64, 3, c1, (1, 2, 3, 4, 5, 6, 7), lo=0.0, hi=256.0,
                integer=True, fmag=2.0, int_flow=True, aggregate=False, backward=False)
    search_case(R, "c1_uniform", 3, 64, 64, 3, c1, (1, 2, 3, 4, 5, 6, 7), lo=0.0, hi=255.0,
                fmag=2.0, int_flow=True, aggregate=False, backward=False)
    # c2-shaped miniature: fractional flow, ip, ps7 at the hole-free stride, wt2 chains
    search_case(R, "c2_mini", 5, 16, 16, 8,
                Cfg(ws=5, wt=2, ps=7, stride0=4, stride1=1.0, topl=10, metric="ip",
                    softmax_scale=1.0 / (49 * 8)), (11, 12, 13, 14, 15, 16, 17), fmag=2.0)
    # c4-shaped miniature: L2, ps3, stride0 2, wt3 (two-link chains)
    search_case(R, "c4_mini", 7, 18, 18, 8,
                Cfg(ws=5, wt=3, ps=3, stride0=2, stride1=1.0, topl=6, metric="l2",
                    softmax_scale=1.0 / (9 * 8)), (100, 200, 300, 301, 302, 303, 304), fmag=1.5)
    # fractional key stride (generic path)
    search_case(R, "stride_half", 3, 10, 9, 2,
                Cfg(ws=5, wt=1, ps=3, stride0=2, stride1=0.5, topl=3, metric="l2"),
                (21, 22, 23, 24, 25, 26, 27))
    # zero flow (crit 1) and the window-of-one identity
    search_case(R, "zero_flow", 2, 7, 6, 3,
                Cfg(ws=3, wt=1, ps=3, stride0=2, stride1=1.0, topl=4, metric="ip"),
                (31, 32, 33, 34, 35, 36, 37), zero_flow=True)
    # known answers from the reference's unit tests
    reflect = np.array([[i, n, R.reflect_index(i, n)] for n in (1, 2, 5, 7)
                        for i in range(-12, 13)], np.int64)
    sm = R.softmax_rows(np.array([[2.0, 1.0, 0.0]]), 1.0)
    ramp = np.arange(16, dtype=np.float64).reshape(1, 4, 4, 1)
    save("known_answers", Cfg(), reflect=reflect, softmax_210=sm, ramp=ramp)


if __name__ == "__main__":
    main()
