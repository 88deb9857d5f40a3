"""One clip through snls_pipeline_run (synchronous) at several chunk sizes: host wall time
per call and (SNLS_PIPE_TRACE=1) the clip's timeline."""
import sys
import time

sys.path.insert(0, ".")
import torch

import bench
from paper_2309_16849_b200 import snls as S

w = sys.argv[1] if len(sys.argv) > 1 else "c4"
wl = bench.WORKLOADS[w]
vid, ff, bf = bench.make_inputs(S, wl, 0)
cfg = S.SearchConfig(ws=wl["ws"], wt=wl["wt"], ps=wl["ps"], stride0=wl["stride0"], topl=wl["topl"],
                     metric=wl["metric"], softmax_scale=wl["beta"])
rows, L = bench.work_model(wl)["rows"], wl["topl"]
vp, fp_, bp = (torch.from_numpy(x).pin_memory() for x in (vid, ff, bf))
sp, op_, oo = torch.empty((rows, L)).pin_memory(), torch.empty((rows, L, 3)).pin_memory(), torch.empty(vid.shape).pin_memory()
ctx = S.context()
for chunk in [int(c) for c in (sys.argv[2:] or ["1", "2", "5"])]:
    pipe = S.Pipeline(cfg, vid.shape, chunk_frames=chunk, ctx=ctx)
    for _ in range(3):
        pipe.run(vp, vp, vp, fp_, bp, sims=sp, offsets=op_, out=oo)
    ts = []
    for _ in range(10):
        a = time.perf_counter()
        pipe.run(vp, vp, vp, fp_, bp, sims=sp, offsets=op_, out=oo)
        ts.append((time.perf_counter() - a) * 1e3)
    ts.sort()
    print(f"{w} one clip, chunk {chunk}: median {ts[5]:.3f} ms, min {ts[0]:.3f} ms", flush=True)
