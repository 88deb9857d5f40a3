"""Host cost of the streaming pipeline: time spent inside Pipeline.submit / wait vs the wall
time per clip (is the e2e stream host-bound?).  python scripts/pipe_host_probe.py c2 1"""
import sys
import time

sys.path.insert(0, ".")
import torch

import bench
from paper_2309_16849_b200 import snls as S

w = sys.argv[1] if len(sys.argv) > 1 else "c2"
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 1
wl = bench.WORKLOADS[w]
vid, ff, bf = bench.make_inputs(S, wl, 0)
cfg = S.SearchConfig(ws=wl["ws"], wt=wl["wt"], ps=wl["ps"], stride0=wl["stride0"], topl=wl["topl"],
                     metric=wl["metric"], softmax_scale=wl["beta"])
rows, L = bench.work_model(wl)["rows"], wl["topl"]
vp, fp_, bp = (torch.from_numpy(x).pin_memory() for x in (vid, ff, bf))
outs = [(torch.empty((rows, L)).pin_memory(), torch.empty((rows, L, 3)).pin_memory(),
         torch.empty(vid.shape).pin_memory()) for _ in range(3)]
ctx = S.context()
pipe = S.Pipeline(cfg, vid.shape, chunk_frames=chunk, ctx=ctx)
for i in range(6):
    pipe.submit(vp, vp, vp, fp_, bp, sims=outs[i % 3][0], offsets=outs[i % 3][1], out=outs[i % 3][2])
for _ in range(3):
    pipe.wait()
n = 60
t_sub = t_wait = 0.0
t0 = time.perf_counter()
for i in range(n):
    a = time.perf_counter()
    pipe.submit(vp, vp, vp, fp_, bp, sims=outs[i % 3][0], offsets=outs[i % 3][1], out=outs[i % 3][2])
    t_sub += time.perf_counter() - a
for _ in range(3):
    a = time.perf_counter()
    pipe.wait()
    t_wait += time.perf_counter() - a
wall = time.perf_counter() - t0
print(f"{w} chunk {chunk}: wall {wall / n * 1e3:.3f} ms/clip, inside submit {t_sub / n * 1e3:.3f} ms/clip "
      f"(includes blocking on the oldest clip), final waits {t_wait * 1e3:.3f} ms")
# host enqueue cost alone: a pipeline with all slots free, one submit each
pipe2 = S.Pipeline(cfg, vid.shape, chunk_frames=chunk, ctx=ctx)
for i in range(3):
    pipe2.submit(vp, vp, vp, fp_, bp, sims=outs[i][0], offsets=outs[i][1], out=outs[i][2])
for _ in range(3):
    pipe2.wait()
torch.cuda.synchronize()
ts = []
for i in range(3):
    a = time.perf_counter()
    pipe2.submit(vp, vp, vp, fp_, bp, sims=outs[i][0], offsets=outs[i][1], out=outs[i][2])
    ts.append(time.perf_counter() - a)
for _ in range(3):
    pipe2.wait()
print(f"  enqueue (non-blocking submit) {min(ts) * 1e3:.3f} ms")
