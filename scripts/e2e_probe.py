"""Decompose the c4 e2e step: H2D alone, D2H alone, chunked compute alone, full pipeline."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
from paper_2309_16849_b200 import snls as S

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
vid, ff, bf = bench.make_inputs(S, wl, 0)
cfg = S.SearchConfig(ws=wl["ws"], wt=wl["wt"], ps=wl["ps"], stride0=wl["stride0"], topl=wl["topl"],
                     metric=wl["metric"], softmax_scale=wl["beta"])
vp, fp_, bp = (torch.from_numpy(x).pin_memory() for x in (vid, ff, bf))
vd, fd, bd = vp.cuda(), fp_.cuda(), bp.cuda()
T = wl["T"]
rows = S.query_grid(T, wl["H"], wl["W"], wl["stride0"])[0]
L = wl["topl"]
sims = torch.empty((rows, L), device="cuda"); offs = torch.empty((rows, L, 3), device="cuda")
wts = torch.empty((rows, L), device="cuda"); out = torch.empty_like(vd)
cnt = torch.empty(vd.shape[:3], device="cuda", dtype=torch.int32)
sp, op_, oo = torch.empty((rows, L)).pin_memory(), torch.empty((rows, L, 3)).pin_memory(), torch.empty(vd.shape).pin_memory()
ctx = S.context()
nq = rows // T

def timeit(fn, n=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n

def h2d():
    vd.copy_(vp, non_blocking=True); fd.copy_(fp_, non_blocking=True); bd.copy_(bp, non_blocking=True)
def d2h():
    sp.copy_(sims, non_blocking=True); op_.copy_(offs, non_blocking=True); oo.copy_(out, non_blocking=True)
def whole():
    S.shifted_nls_forward(vd, vd, fd, bd, cfg, ctx=ctx, check=False, out=(sims, offs, None, wts))
    S.wpsum(vd, wts, offs, cfg, ctx=ctx, check=False, out=(out, cnt))
def chunked(c):
    def f():
        for a in range(0, T, c):
            b = min(T, a + c)
            r0, r1 = a * nq, b * nq
            S.shifted_nls_forward(vd, vd, fd, bd, cfg, ctx=ctx, check=False, frames=(a, b),
                                  out=(sims[r0:r1], offs[r0:r1], None, wts[r0:r1]))
            S.wpsum(vd, wts[r0:r1], offs[r0:r1], cfg, ctx=ctx, check=False, frames=(a, b),
                    out=(out[a:b], cnt[a:b]))
    return f
print("h2d ms", timeit(h2d), "GB/s", (vid.nbytes + ff.nbytes + bf.nbytes) / timeit(h2d) / 1e6)
print("d2h ms", timeit(d2h), "GB/s", (sp.numel() * 4 + op_.numel() * 4 + oo.numel() * 4) / timeit(d2h) / 1e6)
print("whole compute ms", timeit(whole))
for c in (1, 2, 5):
    print(f"chunked({c}) compute ms", timeit(chunked(c)))
for c in (1, 2):
    pipe = S.Pipeline(cfg, vid.shape, chunk_frames=c, ctx=ctx)
    print(f"pipeline({c}) ms", timeit(lambda: pipe.run(vp, vp, vp, fp_, bp, sims=sp, offsets=op_, out=oo)))

# device-resident, chunked over two streams (search of chunk i+1 overlaps wpsum/tail of i)
s2 = [torch.cuda.Stream(), torch.cuda.Stream()]
ctxs = [S.Context(0, s2[0]), S.Context(0, s2[1])]
def chunked2(c):
    def f():
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        for st in s2:
            st.wait_event(ev)
        for i, a in enumerate(range(0, T, c)):
            b = min(T, a + c)
            r0, r1 = a * nq, b * nq
            cx = ctxs[i % 2]
            S.shifted_nls_forward(vd, vd, fd, bd, cfg, ctx=cx, check=False, frames=(a, b),
                                  out=(sims[r0:r1], offs[r0:r1], None, wts[r0:r1]))
            S.wpsum(vd, wts[r0:r1], offs[r0:r1], cfg, ctx=cx, check=False, frames=(a, b),
                    out=(out[a:b], cnt[a:b]))
        for st in s2:
            e = torch.cuda.Event(); e.record(st); cur.wait_event(e)
    return f
for c in (1, 2, 5):
    print(f"chunked2({c}) compute ms", timeit(chunked2(c)))

# compute with the copy engines busy: does PCIe traffic slow the kernels?
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
vd2, fd2, bd2 = torch.empty_like(vd), torch.empty_like(fd), torch.empty_like(bd)
def busy_copies(n):
    with torch.cuda.stream(s_in):
        for _ in range(n):
            vd2.copy_(vp, non_blocking=True); fd2.copy_(fp_, non_blocking=True); bd2.copy_(bp, non_blocking=True)
    with torch.cuda.stream(s_out):
        for _ in range(n):
            sp.copy_(sims, non_blocking=True); op_.copy_(offs, non_blocking=True); oo.copy_(out, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
busy_copies(6)
a.record()
for _ in range(5):
    whole()
b.record(); torch.cuda.synchronize()
print("whole compute ms with concurrent H2D+D2H", a.elapsed_time(b) / 5)
