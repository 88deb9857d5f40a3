"""Do H2D and D2H overlap (separate copy engines)?  Times each alone and both concurrently on
two streams, pinned host memory, for a c2 / c4 sized clip."""
import sys
import time

import torch

mb = float(sys.argv[1]) if len(sys.argv) > 1 else 21.0
n = int(mb * 1024 * 1024 / 4)
hi, ho = torch.empty(n).pin_memory(), torch.empty(n).pin_memory()
di, do = torch.empty(n, device="cuda"), torch.randn(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=20):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                di.copy_(hi, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                ho.copy_(do, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


run(True, True)
print(f"{mb:.0f} MB: h2d {run(True, False):.3f} ms, d2h {run(False, True):.3f} ms, both {run(True, True):.3f} ms")
