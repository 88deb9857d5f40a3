"""Probe: does running frame chunk c's wpsum on a second stream beside chunk c+1's search
shorten the c4 step?  (device-resident inputs; CUDA events; L2 flushed between steps)"""
import sys
import torch

sys.path.insert(0, ".")
from paper_2309_16849_b200 import snls as S  # noqa: E402

t, h, w, f = 10, 256, 256, 32
cfg = S.SearchConfig(ws=11, wt=3, ps=3, stride0=2, topl=16, metric="l2", softmax_scale=1.0 / 288)
g = torch.Generator(device="cuda").manual_seed(0)
v = torch.rand((t, h, w, f), device="cuda", generator=g) * 2 - 1
ff = torch.rand((t, h, w, 2), device="cuda", generator=g) * 4 - 2
bf = torch.rand((t, h, w, 2), device="cuda", generator=g) * 4 - 2
nq = ((h - 1) // 2 + 1) * ((w - 1) // 2 + 1)
rows, L = t * nq, cfg.topl
sims = torch.empty((rows, L), device="cuda"); offs = torch.empty((rows, L, 3), device="cuda")
ch = torch.empty((rows, L, max(cfg.wt - 1, 1), 6), device="cuda"); wts = torch.empty((rows, L), device="cuda")
out = torch.empty_like(v); cnt = torch.empty((t, h, w), dtype=torch.int32, device="cuda")
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
c1, c2 = S.Context(0, s1), S.Context(0, s2)
S.shifted_nls_forward(v, v, ff, bf, cfg, want_weights=True, ctx=c1)  # warm


def step(chunk):
    evs = []
    for a in range(0, t, chunk):
        b = min(t, a + chunk)
        r0, r1 = a * nq, b * nq
        o = (sims[r0:r1], offs[r0:r1], ch[r0:r1], wts[r0:r1])
        S.shifted_nls_forward(v, v, ff, bf, cfg, ctx=c1, check=False, out=o, want_weights=True, frames=(a, b))
        e = torch.cuda.Event(); e.record(s1); s2.wait_event(e)
        # wpsum of frames [a, b) needs the search rows of those frames only
        with torch.cuda.stream(s2):
            S.wpsum(v, wts[r0:r1], offs[r0:r1], cfg, ctx=c2, check=False, out=(out[a:b], cnt[a:b]), frames=(a, b))
    e = torch.cuda.Event(); e.record(s2); s1.wait_event(e)


for chunk in (10, 5, 2, 1):
    ts = []
    for i in range(13):
        flush.zero_(); torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record(s1); step(chunk); en.record(s1); torch.cuda.synchronize()
        if i >= 3:
            ts.append(st.elapsed_time(en))
    ts.sort()
    print(f"chunk {chunk}: median {ts[len(ts)//2]:.3f} ms  min {ts[0]:.3f}")
