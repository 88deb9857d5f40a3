"""Debug: tiled vs generic search on small random inputs, several (ws, ps, F)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2309_16849_b200 import snls as S
ctx = S.context(0)
rng = np.random.default_rng(0)
for (ws, ps, F, wt, T, H, W, s0) in [(5,3,8,0,1,12,12,1),(5,3,8,1,2,12,12,1),(5,3,16,0,1,12,12,1),(5,3,32,0,1,12,12,1),(5,1,8,0,1,12,12,1),(9,1,4,0,1,16,16,1),(11,3,32,0,1,20,20,1),(5,3,8,2,4,16,16,2)]:
    q = torch.tensor(rng.uniform(-1,1,(T,H,W,F)).astype(np.float32), device='cuda')
    k = torch.tensor(rng.uniform(-1,1,(T,H,W,F)).astype(np.float32), device='cuda')
    ff = torch.tensor(rng.uniform(-1.5,1.5,(T,H,W,2)).astype(np.float32), device='cuda')
    bf = torch.tensor(rng.uniform(-1.5,1.5,(T,H,W,2)).astype(np.float32), device='cuda')
    for flows in (False, True):
        cfg = S.SearchConfig(ws=ws, wt=wt, ps=ps, stride0=s0, topl=4, metric='l2')
        ctx.force_generic(True)
        g = S.shifted_nls_forward(q, k, ff if flows else None, bf if flows else None, cfg)
        ctx.force_generic(False)
        t = S.shifted_nls_forward(q, k, ff if flows else None, bf if flows else None, cfg)
        path = ctx.last_search_path()
        gs, ts = g.sims.cpu().numpy(), t.sims.cpu().numpy()
        d = np.abs(gs - ts).max()
        print(f"ws={ws} ps={ps} F={F} wt={wt} flows={flows} path={path} maxdiff={d:.3g}")
        if d > 1e-3:
            r = int(np.argmax(np.abs(gs - ts).max(1)))
            print("  row", r, "generic", gs[r], g.offsets.cpu().numpy()[r].tolist())
            print("  row", r, "tiled  ", ts[r], t.offsets.cpu().numpy()[r].tolist())
