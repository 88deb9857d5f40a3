#!/usr/bin/env python
"""Benchmark: Shifted Non-Local Search forward (search + top-L + softmax + wpsum aggregate) on
B200, the BASELINE.json metric "search+aggregate queries/sec (ms/video) & %roofline".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4|c2|c3|c5]
                    [--videos-per-gpu V] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU)

`--gpus N` without a torchrun environment re-launches itself under torch.distributed.run
with N ranks (127.0.0.1 rendezvous); under torchrun WORLD_SIZE must equal N.
`--videos-per-gpu V` (c4): each rank processes V independent videos per step, so SURVEY 8e's
scaling ratio t(8 videos on 1 GPU) / t(1 video per GPU on 8) is `--gpus 1 --videos-per-gpu 8`
against `--gpus 8`.

Workload (default c4 = BASELINE configs[3]): one 10x256x256x32 video per GPU, ws 11, wt 3,
ps 3, k 16, L2, stride0 2, beta 1/288, fractional flows U[-2,2); Q = K = V as in the
reference's run_benchmark (harness.cpp:242-270).  Inputs come from the reference's own
generator UniformStream (seeds 100+b / 200+b / 300+b for video b = rank).
Multi-GPU: videos are independent -> shard by batch, no data-path collective ("weak").

A step = search (+ fused softmax epilogue) + wpsum on inputs resident in HBM; L2 (126 MB) is
flushed with a 512 MB memset between steps, outside the timed events.  `e2e` repeats the
step through the same public API from pinned HOST buffers with the H2D input copies and the
D2H read-back of the results (sims, offsets, aggregated video) inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "search+aggregate queries/sec (ms/video) & %roofline at 1/2/4/8 B200 vs CPU ref"
UNIT = "queries/s"

WORKLOADS = {
    # BASELINE configs[3]: batch=8 T=10 C=32 H=W=256 ws=11 wt=3 ps=3 k=16, one video per GPU
    "c4": dict(T=10, H=256, W=256, C=32, ws=11, wt=3, ps=3, topl=16, metric="l2", stride0=2,
               beta=1.0 / 288, vid_seed=100, ff_seed=200, bf_seed=300, flow_mag=2.0, pipe_chunk=5,
               name="c4: 10x256x256x32 per video, ws11 wt3 ps3 k16 L2 s0=2, one video/GPU"),
    # BASELINE configs[1]: T=5 C=64 H=W=128 ws=9 wt=2 ps=7 k=10 ip, stride0 4 (hole-free min)
    "c2": dict(T=5, H=128, W=128, C=64, ws=9, wt=2, ps=7, topl=10, metric="ip", stride0=4,
               beta=1.0 / 3136, vid_seed=11, ff_seed=14, bf_seed=15, flow_mag=2.0, pipe_chunk=5,
               name="c2: 5x128x128x64, ws9 wt2 ps7 k10 ip s0=4"),
    # BASELINE configs[2]: c2 shapes fwd + bwd (vid & flow grads); upstream gradients
    # U[-1,1) seeds 16 (sims) and 17 (wpsum output)
    "c3": dict(T=5, H=128, W=128, C=64, ws=9, wt=2, ps=7, topl=10, metric="ip", stride0=4,
               beta=1.0 / 3136, vid_seed=11, ff_seed=14, bf_seed=15, flow_mag=2.0, train=True,
               gs_seed=16, go_seed=17,
               name="c3: 5x128x128x64, ws9 wt2 ps7 k10 ip s0=4, fwd + bwd (dQ dK dV dW dFlow)"),
    # BASELINE configs[4]: single video T=64 C=64 H=W=512 ws=9 wt=2 ps=3 k=10, frame-sharded
    # across ranks with a wt-frame NCCL halo (per-frame seeds 500*1000+t)
    "c5": dict(T=64, H=512, W=512, C=64, ws=9, wt=2, ps=3, topl=10, metric="l2", stride0=2,
               beta=1.0 / 576, vid_seed=500, ff_seed=501, bf_seed=502, flow_mag=2.0,
               sharded=True, pipe_chunk=4,
               name="c5: one 64x512x512x64 video, ws9 wt2 ps3 k10 L2 s0=2, frame-sharded + halo"),
}


# ------------------------------------------------------------------------------------------
# Work model: FMA-pipe lane instructions (FFMA/FADD/FMUL = 1) and compulsory bytes
def work_model(wl):
    T, H, W, C = wl["T"], wl["H"], wl["W"], wl["C"]
    ws, wt, ps, s0, L = wl["ws"], wl["wt"], wl["ps"], wl["stride0"], wl["topl"]
    m = 2 if wl["metric"] == "l2" else 1
    nh, nw = (H - 1) // s0 + 1, (W - 1) // s0 + 1
    per_frame_q = nh * nw
    rows = T * per_frame_q
    sim = interp = chain = 0
    valid_slots = 0
    for qt in range(T):
        for dt in range(-wt, wt + 1):
            if 0 <= qt + dt < T:
                sim += per_frame_q * ws * ws * ps * ps * C * m
                interp += per_frame_q * (ws + ps - 1) ** 2 * C * 4
                chain += per_frame_q * 16 * max(abs(dt) - 1, 0)
                valid_slots += per_frame_q * ws * ws
    # wpsum: contributing units per pixel (footprint + cell completion, aggregate.cpp:156-188)
    half = ps // 2
    import numpy as np

    def units_1d(n, ng):
        cnt = np.zeros(n, np.int64)
        for y in range(n):
            c = sum(1 for py in range(-half, half + 1)
                    if 0 <= y - py <= (ng - 1) * s0 and (y - py) % s0 == 0)
            cnt[y] = c
        own = np.minimum((np.arange(n) + (s0 - 1) // 2) // s0, ng - 1) * s0
        far = np.abs(np.arange(n) - own) > half
        return cnt, far

    cy, fy = units_1d(H, nh)
    cx, fx = units_1d(W, nw)
    units = np.outer(cy, cx) + (fy[:, None] | fx[None, :])
    contrib = int(units.sum()) * T
    wpsum = contrib * L * C * 5 + T * H * W * C
    vid = T * H * W * C * 4
    flows = 2 * T * H * W * 2 * 4
    b_search = vid + flows + rows * L * (4 + 12 + 4)  # Q=K aliased; sims+offsets+weights
    b_wpsum = vid + rows * L * 16 + vid + T * H * W * 4
    return dict(rows=rows, search_instr=sim + interp + chain, search_sim=sim, search_interp=interp,
                wpsum_instr=wpsum, bytes_search=b_search, bytes_wpsum=b_wpsum,
                valid_slots_per_query=valid_slots / rows)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "MEASURED_PEAKS.json"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


# ------------------------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def make_frames(S, wl, t0, t1):
    """Frames [t0, t1) of the c5 video, flows and video from per-frame seeds."""
    import numpy as np

    H, W, C = wl["H"], wl["W"], wl["C"]
    vid = np.stack([S.uniform_fill(wl["vid_seed"] * 1000 + t, -1.0, 1.0, H * W * C).reshape(H, W, C)
                    for t in range(t0, t1)])
    m = wl["flow_mag"]
    ff = np.stack([S.uniform_fill(wl["ff_seed"] * 1000 + t, -m, m, H * W * 2).reshape(H, W, 2)
                   for t in range(t0, t1)])
    bf = np.stack([S.uniform_fill(wl["bf_seed"] * 1000 + t, -m, m, H * W * 2).reshape(H, W, 2)
                   for t in range(t0, t1)])
    return vid, ff, bf


def make_inputs(S, wl, b):
    import numpy as np

    T, H, W, C = wl["T"], wl["H"], wl["W"], wl["C"]
    vid = S.uniform_fill(wl["vid_seed"] + b, -1.0, 1.0, T * H * W * C).reshape(T, H, W, C)
    ff = S.uniform_fill(wl["ff_seed"] + b, -wl["flow_mag"], wl["flow_mag"], T * H * W * 2)
    bf = S.uniform_fill(wl["bf_seed"] + b, -wl["flow_mag"], wl["flow_mag"], T * H * W * 2)
    return vid, ff.reshape(T, H, W, 2), bf.reshape(T, H, W, 2)


def init_dist(world, local, backend):
    """One process per GPU; NCCL's INIT lines (communicator size) go to stderr as evidence of
    the N-rank communicator.  Returns the communicator description for the JSON line."""
    import torch
    import torch.distributed as dist

    if world <= 1:
        return None
    if backend == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()  # eager communicator creation (device_id) + one collective
    else:
        dist.init_process_group("gloo")
    n = dist.get_world_size()
    assert n == world, f"communicator has {n} ranks, WORLD_SIZE says {world}"
    print(f"[bench] rank {dist.get_rank()}: {backend} communicator nranks={n}", file=sys.stderr, flush=True)
    return {"backend": backend, "nranks": n}


def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    from paper_2309_16849_b200 import snls as S

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    comm_info = init_dist(world, local, "nccl")
    dev = torch.device("cuda", local)
    model = work_model(wl)
    rows = model["rows"]
    nvid = max(1, args.videos_per_gpu)
    if nvid > 1 and (wl.get("sharded") or wl.get("train")):
        raise SystemExit("--videos-per-gpu applies to the batch workloads (c4, c2)")
    cfg = S.SearchConfig(ws=wl["ws"], wt=wl["wt"], ps=wl["ps"], stride0=wl["stride0"],
                         stride1=1.0, topl=wl["topl"], metric=wl["metric"], softmax_scale=wl["beta"])
    sharded = wl.get("sharded", False)
    if sharded:  # frame sharding: own frames [a, b), halo frames from the neighbours (NCCL)
        from paper_2309_16849_b200 import shard as SH

        plan = SH.plan(wl["T"], world, rank, wl["wt"])
        vid_h, ff_h, bf_h = make_frames(S, wl, plan.a, plan.b)
        frames = (plan.t0, plan.t1)
        rows = (plan.b - plan.a) * (rows // wl["T"])
    else:
        # video b = rank * V + j (seeds 100+b / 200+b / 300+b)
        vid_h, ff_h, bf_h = make_inputs(S, wl, rank * nvid)
        frames = None
    own_vid = torch.from_numpy(vid_h).to(dev)
    own_ff = torch.from_numpy(ff_h).to(dev)
    own_bf = torch.from_numpy(bf_h).to(dev)
    vid, ff, bf = own_vid, own_ff, own_bf
    # the other videos of this rank (independent inputs, own output buffers)
    extra = []
    for j in range(1, nvid):
        vh, fh, bh = make_inputs(S, wl, rank * nvid + j)
        extra.append(tuple(torch.from_numpy(x).to(dev) for x in (vh, fh, bh)) +
                     (torch.empty((rows, wl["topl"]), device=dev), torch.empty((rows, wl["topl"], 3), device=dev),
                      torch.empty((rows, wl["topl"]), device=dev), torch.empty_like(own_vid),
                      torch.empty(own_vid.shape[:3], device=dev, dtype=torch.int32)))
    if sharded:  # persistent slabs [lo, hi): owned frames in place, halo frames refilled by
        # the in-place NCCL exchange every step (overlapped with the interior frames)
        def slab_of(own):
            sl = torch.zeros((plan.hi - plan.lo,) + tuple(own.shape[1:]), device=dev)
            sl[plan.t0:plan.t1].copy_(own)
            return sl
        vid, ff, bf = slab_of(own_vid), slab_of(own_ff), slab_of(own_bf)
    overlapped = sharded and world > 1
    stream = torch.cuda.current_stream(dev)
    ctx = S.context(local)
    # the halo moves over the C-ABI's own NCCL communicator (snls_halo_exchange_async); the
    # torch.distributed group above is control plane only (id broadcast, barriers, max)
    comm = SH.Comm.create(rank, world, ctx) if overlapped else None
    if comm is not None:
        ci = comm.info()
        comm_info["snls_halo_comm"] = ci
        print(f"[bench] rank {rank}: snls NCCL communicator nranks={ci['nranks']} "
              f"(NCCL {ci['nccl_version']})", file=sys.stderr, flush=True)
    ctx.set_search_kernel(args.search_kernel)
    L = wl["topl"]
    sims = torch.empty((rows, L), device=dev)
    offs = torch.empty((rows, L, 3), device=dev)
    wts = torch.empty((rows, L), device=dev)
    out = torch.empty_like(own_vid)
    counts = torch.empty(own_vid.shape[:3], device=dev, dtype=torch.int32)
    flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)
    train = wl.get("train", False)
    if train:  # the tape's chains and the two upstream gradients
        chains = torch.empty((rows, L, cfg.chain_stride(), 6), device=dev) if cfg.wt > 1 else None
        g_sims = torch.from_numpy(S.uniform_fill(wl["gs_seed"], -1, 1, rows * L).reshape(rows, L)).to(dev)
        g_out = torch.from_numpy(S.uniform_fill(wl["go_seed"], -1, 1, own_vid.numel())
                                 .reshape(own_vid.shape)).to(dev)
    bwd_ms = []

    def step():
        if overlapped:  # the data path's only communication: the wt-frame halo (NCCL P2P)
            SH.search_aggregate_overlapped(vid, vid, vid, ff, bf, plan, cfg, ctx=ctx, comm=comm,
                                           out=(sims, offs, None, wts, out, counts))
            ev_mid.record(stream)
            return
        res = S.shifted_nls_forward(vid, vid, ff, bf, cfg, ctx=ctx, check=False,
                                    out=(sims, offs, chains if train else None, wts), frames=frames)
        for (xv, xf, xb, xs, xo, xw, _, _) in extra:  # further videos of this rank: search
            S.shifted_nls_forward(xv, xv, xf, xb, cfg, ctx=ctx, check=False, out=(xs, xo, None, xw))
        ev_mid.record(stream)
        S.wpsum(vid, wts, offs, cfg, ctx=ctx, check=False, out=(out, counts), frames=frames)
        for (xv, _, _, _, xo, xw, xout, xcnt) in extra:  # ... and aggregation
            S.wpsum(xv, xw, xo, cfg, ctx=ctx, check=False, out=(xout, xcnt))
        if train:  # backward of the chain: dQ, dK, dV, dW, dFlow (snls_train_bwd) from the
            # reference-layout fp64 tape (snls_search_tape64: exact key positions, the flow
            # gradients' 1e-5 parity holds for Q = K = V self-similarity too)
            ev_bwd.record(stream)
            res.weights = wts
            t64 = S.search_tape64(res, ff, bf, ctx=ctx, check=False)
            S.train_backward(g_sims, g_out, counts, res, vid, vid, vid, ctx=ctx, check=False,
                             deterministic=args.deterministic, tape64=t64)

    # correctness gate before timing: device error latch must be clean
    ev_mid = torch.cuda.Event(enable_timing=True)
    ev_bwd = torch.cuda.Event(enable_timing=True)
    step()
    ctx.sync_check()
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launch_count()
    clocks = ClockSampler(local)
    clocks.start()
    evs = []
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        ev_mid = torch.cuda.Event(enable_timing=True)
        ev_bwd = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e2.record(stream)
        evs.append((e0, ev_mid, e2, ev_bwd))
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = ctx.launch_count() - launches0
    ctx.sync_check()
    step_ms = [a.elapsed_time(c) for a, _, c, _ in evs]
    search_ms = [a.elapsed_time(b) for a, b, _, _ in evs]
    wpsum_ms = [b.elapsed_time(bw if train else c) for _, b, c, bw in evs]
    bwd_ms = [bw.elapsed_time(c) for _, _, c, bw in evs] if train else []
    tot = sum(step_ms)
    tot_search = sum(search_ms)
    if world > 1:
        t = torch.tensor([tot, tot_search], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot, tot_search = float(t[0]), float(t[1])
    ms_per_step = tot / args.steps

    # ---- e2e: pinned host buffers, copies inside the timed region ----
    vid_p = torch.from_numpy(vid_h).pin_memory()
    ff_p, bf_p = torch.from_numpy(ff_h).pin_memory(), torch.from_numpy(bf_h).pin_memory()
    sims_p = torch.empty((rows, L)).pin_memory()
    offs_p = torch.empty((rows, L, 3)).pin_memory()
    out_p = torch.empty(vid_h.shape).pin_memory()
    use_pipe = not (sharded and world > 1) and not train
    if use_pipe:
        # the C-ABI host-buffer call (snls_pipeline_run): frame-chunked kernels overlapped
        # with the H2D input / D2H result copies; Q = K = V is one host buffer, copied once
        # frames per chunk, measured per workload for the streamed e2e (profiles/r01_plans.txt)
        chunk = args.pipe_chunk or wl.get("pipe_chunk", 1)
        pipe = S.Pipeline(cfg, vid_h.shape, chunk_frames=chunk, ctx=ctx)
        # one clip at a time (latency): per-frame chunks overlap the clip's own transfers best
        pipe1 = S.Pipeline(cfg, vid_h.shape, chunk_frames=1, ctx=ctx) if chunk != 1 else pipe

        def e2e_step():
            pipe1.run(vid_p, vid_p, vid_p, ff_p, bf_p, sims=sims_p, offsets=offs_p, out=out_p)
    else:
        vd, ffd, bfd = torch.empty_like(own_vid), torch.empty_like(own_ff), torch.empty_like(own_bf)

        def e2e_step():
            vd.copy_(vid_p, non_blocking=True)
            ffd.copy_(ff_p, non_blocking=True)
            bfd.copy_(bf_p, non_blocking=True)
            v2, f2, b2 = vd, ffd, bfd
            if overlapped:
                vid[plan.t0:plan.t1].copy_(vd)
                ff[plan.t0:plan.t1].copy_(ffd)
                bf[plan.t0:plan.t1].copy_(bfd)
                SH.search_aggregate_overlapped(vid, vid, vid, ff, bf, plan, cfg, ctx=ctx, comm=comm,
                                               out=(sims, offs, None, wts, out, counts))
                sims_p.copy_(sims, non_blocking=True)
                offs_p.copy_(offs, non_blocking=True)
                out_p.copy_(out, non_blocking=True)
                return
            res = S.shifted_nls_forward(v2, v2, f2, b2, cfg, ctx=ctx, check=False,
                                        out=(sims, offs, chains if train else None, wts), frames=frames)
            S.wpsum(v2, wts, offs, cfg, ctx=ctx, check=False, out=(out, counts), frames=frames)
            if train:
                res.weights = wts
                t64 = S.search_tape64(res, f2, b2, ctx=ctx, check=False)
                S.train_backward(g_sims, g_out, counts, res, v2, v2, v2, ctx=ctx, check=False,
                                 deterministic=args.deterministic, tape64=t64)
            sims_p.copy_(sims, non_blocking=True)
            offs_p.copy_(offs, non_blocking=True)
            out_p.copy_(out, non_blocking=True)

    # further videos of the rank go through the same call one after another: they copy the
    # same bytes as video 0, so e2e per step = V clips (timed per clip below, x V)
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # clips per e2e measurement: the stream's fill (first H2D) and drain (last D2H) are paid once
    # per measurement, so use the timed step count, capped at ~2 s of clips
    n_e2e = max(3, min(args.steps, int(2000.0 / max(ms_per_step, 1e-3))))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    a.record(stream)
    for _ in range(n_e2e):
        e2e_step()
    b.record(stream)
    torch.cuda.synchronize()
    e2e_wall_ms = (time.perf_counter() - w0) * 1e3 / n_e2e
    e2e_ms = a.elapsed_time(b) / n_e2e
    e2e_sync_ms = e2e_ms
    if use_pipe:
        # one-clip latency: snls_pipeline_run returns to the host between clips, so host
        # scheduling jitter lands in a mean; report the median clip instead
        per = []
        for _ in range(min(n_e2e, 30)):
            a.record(stream)
            e2e_step()
            b.record(stream)
            torch.cuda.synchronize()
            per.append(a.elapsed_time(b))
        e2e_sync_ms = sorted(per)[len(per) // 2]
    if use_pipe:
        # a stream of clips through snls_pipeline_submit / wait: every clip still copies its
        # inputs in and its results out, but the next clip's transfers overlap this one's
        # compute (three buffer slots; one set of host output buffers per clip in flight)
        NS = 3
        outs = [(sims_p, offs_p, out_p)] + [
            (torch.empty_like(sims_p).pin_memory(), torch.empty_like(offs_p).pin_memory(),
             torch.empty_like(out_p).pin_memory()) for _ in range(NS - 1)]
        for i in range(NS):
            pipe.submit(vid_p, vid_p, vid_p, ff_p, bf_p, sims=outs[i][0], offsets=outs[i][1], out=outs[i][2])
        for _ in range(NS):
            pipe.wait()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        a.record(stream)
        for i in range(n_e2e):
            pipe.submit(vid_p, vid_p, vid_p, ff_p, bf_p, sims=outs[i % NS][0], offsets=outs[i % NS][1],
                        out=outs[i % NS][2])
        for _ in range(NS):
            pipe.wait()
        b.record(stream)
        torch.cuda.synchronize()
        e2e_wall_ms = (time.perf_counter() - w0) * 1e3 / n_e2e
        e2e_ms = a.elapsed_time(b) / n_e2e
        assert torch.equal(outs[1][2], out_p) and torch.equal(outs[1][0], sims_p)
    e2e_ms *= nvid
    e2e_sync_ms *= nvid
    e2e_wall_ms *= nvid
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    ctx.sync_check()
    if use_pipe:
        # the pipeline's results are the device path's results (same kernels, same rows)
        assert torch.equal(sims_p, sims.cpu()) and torch.equal(out_p, out.cpu()), \
            "host-buffer pipeline disagrees with the device-resident step"
    h2d = (vid_h.nbytes + ff_h.nbytes + bf_h.nbytes) * nvid
    d2h = (sims_p.numel() * 4 + offs_p.numel() * 4 + out_p.numel() * 4) * nvid

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    total_rows = model["rows"] if sharded else rows * world * nvid
    P, peak_src = peaks()
    sm_max = float(P.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_peak_tflops = nsm * 128 * 2 * sm_max * 1e6 / 1e12
    t_search = tot_search / args.steps / 1e3
    share = rows / model["rows"]  # this rank's fraction of the video (frame sharding)
    achieved = 2.0 * model["search_instr"] * share * nvid / t_search / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(args.workload, {}).get("search_bytes_per_launch")
        except Exception:
            traffic = None
    result = {
        "metric": METRIC,
        "value": total_rows / (ms_per_step / 1e3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "ms_per_video": ms_per_step / nvid,
        "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic: reference UniformStream video U[-1,1) (Q=K=V) and flows U[-2,2)",
        "config": {"workload": wl["name"],
                   "videos_per_gpu": nvid if not sharded else f"1/{world} (frames {plan.a}..{plan.b - 1} on rank 0)",
                   "global_batch": nvid * world if not sharded else 1,
                   "queries_per_gpu": rows * nvid,
                   "parallelism": (f"frame-sharded x{world}, wt-frame halo via the C-ABI's NCCL send/recv"
                                   if sharded else f"batch-sharded x{world} (no collective)"),
                   "l2": "flushed (512 MB memset) between timed steps"},
        "comm": comm_info,
        "breakdown_ms": {("search_topl_softmax" if not overlapped else
                          "search_softmax_wpsum_with_halo_exchange"): tot_search / args.steps,
                         "wpsum": statistics.mean(wpsum_ms),
                         **({"backward": statistics.mean(bwd_ms)} if train else {})},
        "roofline": {"bound": "fp32", "kernel": "search_tiled_kernel",
                     "achieved": achieved, "peak": fp32_peak_tflops, "unit": "TFLOP/s",
                     "frac": achieved / fp32_peak_tflops, "traffic": traffic,
                     "algorithmic": f"{model['search_instr']:.4g} FMA-pipe instr/video x2 flop",
                     "peak_source": f"{nsm} SMs x 128 FP32 lanes x 2 x sm_max_mhz from {peak_src}",
                     "hbm_frac": model["bytes_search"] * share * nvid / t_search / 1e9 / float(P.get("hbm_gbs", 6650))},
        "e2e": {"value": total_rows / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
                "wall_ms_per_step": e2e_wall_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "sync_ms_per_step": e2e_sync_ms,
                "api": ("snls_pipeline_submit/wait (C-ABI, a stream of clips from pinned host "
                        f"buffers, {chunk} frame(s)/chunk, three clips in flight; "
                        "sync_ms_per_step = one clip at a time, snls_pipeline_run, 1 frame/chunk, median clip)") if use_pipe else
                       ("torch H2D + snls_halo_exchange_async (C-ABI NCCL) + snls_search_fwd_frames/"
                        "wpsum_fwd_frames + D2H" if overlapped else
                        "torch H2D + snls_search_fwd / snls_wpsum_fwd" +
                        (" / snls_train_bwd" if train else "") + " (C-ABI) + D2H")},
        "gpu_launches": launches,
        "clocks": clk,
        "wall_s_timed_loop": wall,
    }
    if world == 1 and not wl.get("sharded") and not wl.get("train"):
        result["e2e_cpp_api"] = cpp_api_e2e(wl)
    if world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(wl, budget_s=args.cpu_budget)
    print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------------------------------
def reference_sample(wl, crop):
    """The reference's own CPU path (oracle/_ref: unmodified sources, OpenMP, fp64) on a crop
    of the workload with identical per-query work (same ws/wt/ps/k/metric/stride0/C/T)."""
    import numpy as np

    from oracle.oracle import Cfg, Checker

    R = Checker("reference")
    T, C = wl["T"], wl["C"]
    H = W = crop
    v = R.uniform(wl["vid_seed"], -1, 1, T * H * W * C).astype(np.float32).astype(np.float64)
    v = v.reshape(T, H, W, C)
    ff = R.uniform(wl["ff_seed"], -2, 2, T * H * W * 2).astype(np.float32).astype(np.float64)
    bf = R.uniform(wl["bf_seed"], -2, 2, T * H * W * 2).astype(np.float32).astype(np.float64)
    ff, bf = ff.reshape(T, H, W, 2), bf.reshape(T, H, W, 2)
    cfg = Cfg(ws=wl["ws"], wt=wl["wt"], ps=wl["ps"], stride0=wl["stride0"], stride1=1.0,
              topl=wl["topl"], metric=wl["metric"], softmax_scale=wl["beta"])
    rows = T * ((H - 1) // cfg.stride0 + 1) * ((W - 1) // cfg.stride0 + 1)

    train = wl.get("train", False)
    if train:  # upstream gradients of the sims and of the aggregated video
        L = cfg.topl
        gs = R.uniform(wl["gs_seed"], -1, 1, rows * L).astype(np.float32).astype(np.float64)
        gs = gs.reshape(rows, L)
        go = R.uniform(wl["go_seed"], -1, 1, v.size).astype(np.float32).astype(np.float64)
        go = go.reshape(v.shape)

    def run():
        t0 = time.perf_counter()
        r = R.search_fwd(v, v, ff, bf, cfg)
        w = R.softmax_rows(r["sims"], cfg.softmax_scale)
        _, counts = R.wpsum(v, w, r["offsets"], cfg)
        if train:  # the reference's default (deterministic) backward
            R.wpsum_bwd(go, counts, v, w, r["offsets"], cfg)
            R.search_bwd(v, v, cfg, r["centers"], r["chains"], gs)
        return time.perf_counter() - t0

    return R, rows, run


def cpp_api_e2e(wl):
    """The reference's own C++ caller, snls::run_benchmark (harness.cpp:242-283), timing
    snls::shifted_nls_forward through the C++ drop-in (host/build/bench_gpu: libsnls_gpu.so
    over libsnls_cuda.so) on this workload's shape: fp64 host containers in and out, the
    conversions and copies inside the timed region (search only -- run_benchmark times the
    forward)."""
    exe = os.path.join(ROOT, "paper_2309_16849_b200", "host", "build", "bench_gpu")
    if not os.path.exists(exe):
        return {"unavailable": "host/build/bench_gpu not built (needs the reference headers)"}
    args = [str(x) for x in (wl["T"], wl["H"], wl["W"], wl["C"], wl["ws"], wl["wt"], wl["ps"],
                             wl["stride0"], wl["topl"], wl["metric"], 5)]
    try:
        p = subprocess.run([exe] + args, capture_output=True, text=True, timeout=600)
        r = json.loads(p.stdout.strip().splitlines()[-1])
    except Exception as e:  # reported, not fatal
        return {"unavailable": f"bench_gpu failed: {e}"}
    return {"value": r["queries_per_s"], "unit": UNIT, "ms_per_video": r["median_ms"],
            "api": "snls::shifted_nls_forward (reference C++ API; snls::run_benchmark, median of 5) "
                   "through libsnls_gpu.so -> libsnls_cuda.so, fp64 containers in/out",
            "ok": r["ok"]}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(wl, budget_s=20.0):
    crop = 96
    R, rows, run = reference_sample(wl, crop)
    t = run()  # warm-up + size probe
    times = []
    deadline = time.perf_counter() + budget_s
    while len(times) < 3 or (time.perf_counter() < deadline and len(times) < 40):
        times.append(run())
        if time.perf_counter() > deadline and len(times) >= 1:
            break
    med = statistics.median(times)
    return {"value": rows / med, "unit": UNIT, "cores": R.lib.ref_max_threads(),
            "kind": "reference", "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "sample": (f"reference snls::shifted_nls_forward + softmax_rows + wpsum"
                       f"{' + wpsum_backward + shifted_nls_backward' if wl.get('train') else ''} (oracle/_ref, "
                       f"fp64, OpenMP all host threads) on a {wl['T']}x{crop}x{crop}x{wl['C']} crop "
                       f"of the workload ({rows} queries, identical per-query work), median of "
                       f"{len(times)} runs after 1 warm-up ({t:.2f}s)")}


def run_reference(args, wl):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    crop = args.ref_crop
    R, rows, run = reference_sample(wl, crop)
    for _ in range(args.warmup):
        run()
    times = [run() for _ in range(args.steps)]
    tot = sum(times)
    value = rows * args.steps / tot
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference UniformStream video U[-1,1) (Q=K=V) and flows U[-2,2)",
        "config": {"workload": wl["name"], "sample": f"{wl['T']}x{crop}x{crop}x{wl['C']} crop",
                   "queries_per_step": rows},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": R.lib.ref_max_threads(),
                         "kind": "reference", "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                         "sample": f"{wl['T']}x{crop}x{crop}x{wl['C']} crop, {rows} queries/step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-crop", type=int, default=96)
    ap.add_argument("--pipe-chunk", type=int, default=int(os.environ.get("SNLS_PIPE_CHUNK", "0")),
                    help="query frames per chunk of the e2e host pipeline (0: 1)")
    ap.add_argument("--search-kernel", default=os.environ.get("SNLS_SEARCH_KERNEL", "auto"),
                    choices=["auto", "tiled", "stream"], help="stride1 == 1 register plan")
    ap.add_argument("--videos-per-gpu", type=int, default=1,
                    help="independent videos per rank and step (c4/c2; SURVEY 8e scaling ratio)")
    ap.add_argument("--deterministic", action="store_true",
                    help="c3: the backward in the reference's deterministic mode (int64 fixed point)")
    ap.add_argument("--mock-cpu", action="store_true",
                    help="plumbing check without a GPU: gloo ranks, a numpy stand-in step, same "
                         "launch / barrier / max-over-ranks / JSON path (tests/test_bench.py)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = WORKLOADS[args.workload]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus))
    _, world, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.mock_cpu:
        run_mock(args, wl)
    elif args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


def self_launch(n):
    """`--gpus N` outside torchrun: re-run this command as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1; rank 0's JSON line reaches our stdout."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_mock(args, wl):
    """The multi-rank harness without a GPU: gloo communicator, W warm-up and K timed steps of
    a fixed numpy stand-in, barrier on both sides, max over ranks, one JSON line on rank 0.
    Not a measurement (no kernels run) -- it exercises the launch path the driver uses."""
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    comm = init_dist(world, local, "gloo")
    a = np.random.default_rng(rank).standard_normal((256, 256))

    def step():
        return float((a @ a).sum())

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    tot = (time.perf_counter() - t0) * 1e3
    if world > 1:
        dist.barrier()
        t = torch.tensor([tot], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t[0])
    rows = work_model(wl)["rows"] * max(1, args.videos_per_gpu)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": rows * world / (tot / args.steps / 1e3),
                          "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": tot / args.steps, "mock": True, "comm": comm,
                          "config": {"workload": wl["name"], "videos_per_gpu": args.videos_per_gpu}}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
