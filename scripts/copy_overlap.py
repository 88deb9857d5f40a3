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

# the pipeline's pattern: H2D in 5 frame-sized pieces (+ 10 small flow copies), D2H as one
# large copy, on two non-blocking streams
fi, ff_h, ff_d = 5, torch.empty(n // 32).pin_memory(), torch.empty(n // 32, device="cuda")


def run2(reps=20):
    torch.cuda.synchronize()
    t = time.perf_counter()
    step = n // fi
    for _ in range(reps):
        with torch.cuda.stream(s1):
            for f in range(fi):
                di[f * step:(f + 1) * step].copy_(hi[f * step:(f + 1) * step], non_blocking=True)
                ff_d.copy_(ff_h, non_blocking=True)
                ff_d.copy_(ff_h, non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


run2()
print(f"{mb:.0f} MB pipeline pattern (5 frame pieces + 10 flow copies H2D, one D2H): both {run2():.3f} ms")


def run3(pieces, flows, reps=20):
    torch.cuda.synchronize()
    t = time.perf_counter()
    step = n // pieces
    for _ in range(reps):
        with torch.cuda.stream(s1):
            for f in range(pieces):
                di[f * step:(f + 1) * step].copy_(hi[f * step:(f + 1) * step], non_blocking=True)
                for _ in range(flows):
                    ff_d.copy_(ff_h, non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


for pieces, flows in ((5, 0), (1, 2), (1, 0), (5, 2), (2, 0), (10, 0)):
    run3(pieces, flows)
    print(f"  H2D in {pieces} pieces + {flows} flow copies each, with one D2H: {run3(pieces, flows):.3f} ms")
