"""Median device time of the search launch alone (no weights) for a bench workload:
python scripts/search_time.py c4  (A/B helper; SNLS_LIB_OVERRIDE selects a variant build)."""
import sys

sys.path.insert(0, ".")
import torch

import bench
from paper_2309_16849_b200 import snls as S

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
m = bench.work_model(wl)
vid, ff, bf = bench.make_inputs(S, wl, 0)
v, f, b = (torch.from_numpy(x).cuda() for x in (vid, ff, bf))
cfg = S.SearchConfig(ws=wl["ws"], wt=wl["wt"], ps=wl["ps"], stride0=wl["stride0"], topl=wl["topl"],
                     metric=wl["metric"], softmax_scale=wl["beta"])
rows, L = m["rows"], wl["topl"]
sims, offs = torch.empty((rows, L), device="cuda"), torch.empty((rows, L, 3), device="cuda")
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
ctx = S.context()
for _ in range(3):
    S.shifted_nls_forward(v, v, f, b, cfg, ctx=ctx, check=False, out=(sims, offs, None, None))
ts = []
for _ in range(20):
    flush.zero_()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    S.shifted_nls_forward(v, v, f, b, cfg, ctx=ctx, check=False, out=(sims, offs, None, None))
    e.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(e))
print(sys.argv[1:], "search ms", sorted(ts)[len(ts) // 2])
