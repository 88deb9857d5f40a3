"""How much could a shared-memory pre-reduction of the backward's dK / dV scatter save?
(north star: "backward kernels ... use shared-memory pre-reduction before atomics")

For the c3 step's own selection (Q = K = V self-search, the bench's inputs), count for each
CTA-sized group of consecutive query rows the raw-block pixels its (row, l) entries scatter
into: total contributions vs distinct (frame, y, x) pixels.  A shared tile can only merge the
repeats; the rest still needs one global reduction per pixel and channel."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2309_16849_b200 import snls as S  # noqa: E402

t, h, w, f = 5, 128, 128, 64
cfg = S.SearchConfig(ws=9, wt=2, ps=7, stride0=4, topl=10, metric="ip", softmax_scale=1.0 / 3136)
g = torch.Generator(device="cuda").manual_seed(11)
v = torch.rand((t, h, w, f), device="cuda", generator=g) * 2 - 1
ff = torch.rand((t, h, w, 2), device="cuda", generator=g) * 4 - 2
bf = torch.rand((t, h, w, 2), device="cuda", generator=g) * 4 - 2
r = S.shifted_nls_forward(v, v, ff, bf, cfg, want_weights=True)
offs = r.offsets.cpu().numpy()  # rows x L x 3 (dt, dy, dx)
nh, nw = (h - 1) // 4 + 1, (w - 1) // 4 + 1
rows = offs.shape[0]
qt = np.repeat(np.arange(t), nh * nw)
qy = np.tile(np.repeat(np.arange(nh) * 4, nw), t)
qx = np.tile(np.tile(np.arange(nw) * 4, nh), t)
P, HP = 7, 3
out = {}
for group in (2, 4, 8, 16, 32):
    tot, uniq = 0, 0
    for g0 in range(0, rows, group):
        pix = set()
        n = 0
        for rr in range(g0, min(rows, g0 + group)):
            for l in range(offs.shape[1]):
                kt = qt[rr] + int(round(offs[rr, l, 0]))
                by = qy[rr] - HP + int(np.floor(offs[rr, l, 1]))
                bx = qx[rr] - HP + int(np.floor(offs[rr, l, 2]))
                for i in range(P + 1):
                    for j in range(P + 1):
                        pix.add((kt, min(max(by + i, 0), h - 1), min(max(bx + j, 0), w - 1)))
                n += (P + 1) ** 2
        tot += n
        uniq += len(pix)
    out[group] = {"contributions": tot, "distinct_pixels": uniq, "reduction": round(tot / uniq, 3)}
    print(f"group of {group:2d} query rows: {tot} block-pixel contributions onto {uniq} distinct pixels "
          f"-> a perfect shared-memory pre-reduction removes {100 * (1 - uniq / tot):.1f}% of the reductions")
json.dump(out, open("gpurun_out/prereduce_potential.json", "w"), indent=1)

# per (query, key frame): neighbours in the frame, the union of their raw blocks and the
# bounding box a per-frame shared window would have to flush
frames_per_q, union_px, bbox_px, direct_px = [], 0, 0, 0
for rr in range(rows):
    by_frame = {}
    for l in range(offs.shape[1]):
        kt = qt[rr] + int(round(offs[rr, l, 0]))
        by = qy[rr] - HP + int(np.floor(offs[rr, l, 1]))
        bx = qx[rr] - HP + int(np.floor(offs[rr, l, 2]))
        by_frame.setdefault(kt, []).append((by, bx))
    frames_per_q.append(len(by_frame))
    for kt, blocks in by_frame.items():
        pix = set()
        for by, bx in blocks:
            for i in range(P + 1):
                for j in range(P + 1):
                    pix.add((by + i, bx + j))
        ys = [b[0] for b in blocks]
        xs = [b[1] for b in blocks]
        union_px += len(pix)
        bbox_px += (max(ys) - min(ys) + P + 1) * (max(xs) - min(xs) + P + 1)
        direct_px += len(blocks) * (P + 1) ** 2
print(f"per query: {np.mean(frames_per_q):.2f} key frames among its {offs.shape[1]} neighbours; "
      f"per (query, frame): direct {direct_px} px-reductions, union {union_px} "
      f"({100 * (1 - union_px / direct_px):.1f}% fewer), bounding boxes {bbox_px} "
      f"({100 * (1 - bbox_px / direct_px):.1f}% fewer)")
