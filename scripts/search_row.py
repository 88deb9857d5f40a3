"""Time the search kernel alone on SURVEY 8d's search-only row (c2 shapes at stride0 = 1:
81,920 queries) and report its FP32 roofline fraction (bench.py's work model)."""
import json
import sys

sys.path.insert(0, ".")
import torch

import bench
from paper_2309_16849_b200 import snls as S

wl = dict(bench.WORKLOADS["c2"], stride0=1)
m = bench.work_model(wl)
vid, ff, bf = bench.make_inputs(S, wl, 0)
v, f, b = (torch.from_numpy(x).cuda() for x in (vid, ff, bf))
cfg = S.SearchConfig(ws=wl["ws"], wt=wl["wt"], ps=wl["ps"], stride0=1, topl=wl["topl"], metric=wl["metric"],
                     softmax_scale=wl["beta"])
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
ms = sorted(ts)[len(ts) // 2]
peak = 148 * 128 * 2 * bench.peaks()[0].get("sm_max_mhz", 1965.0) * 1e6 / 1e12
ach = 2 * m["search_instr"] / (ms * 1e-3) / 1e12
print(json.dumps({"row": "c2 s0=1 search only", "rows": rows, "ms": ms, "search_instr": m["search_instr"],
                  "achieved_tflops": ach, "peak_tflops": peak, "frac": ach / peak}))
