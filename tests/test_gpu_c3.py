"""GPU parity of the training step at the BASELINE c3 configuration's REAL shape -- ps 7,
ws 9, wt 2, F 64 (two 32-channel slices in the row-centric backward), stride0 4, L 10 --
for both metrics, on reduced frames (5 x 20 x 20) the oracle finishes in about a second.

Checked against the oracle (search.cpp:499-711, aggregate.cpp:351-460) at the north star's
1e-5 (gradcheck_util.hpp:19-21):
  * dQ, dK, dFflow, dBflow from the device tape (fp32 offsets + relative chains) against the
    oracle on the SAME fp32 tape;
  * the same four gradients from the reference's own fp64 tape (centres + absolute chains,
    search.hpp:89-110) against the oracle on that tape -- the flow gradients included, with
    no looser bound;
  * the device's fp64 tape (snls_search_tape64) equals the reference's tape;
  * dV, dW (wpsum_backward) on the device's own selection;
  * the deterministic mode (search.cpp:687-696): bitwise identical on repeated runs, and
    within 1e-5 of the oracle."""
import numpy as np
import pytest

from oracle.oracle import Cfg
from tests.gpu_util import compare_search, dev, host, oracle_ranked, rel_chains, scfg, snls_mod
from tests.helpers import REL_TOL, f32, flow, max_rel, video

pytestmark = pytest.mark.gpu

T, H, W, F = 5, 20, 20, 64
_cache = {}


def c3_case(port, metric):
    if metric not in _cache:
        cfg = Cfg(ws=9, wt=2, ps=7, stride0=4, topl=10, metric=metric, softmax_scale=1.0 / 3136)
        q, k = video(port, T, H, W, F, 11), video(port, T, H, W, F, 12)
        ff, bf = flow(port, T, H, W, 14, 2.0), flow(port, T, H, W, 15, 2.0)
        fw = port.search_fwd(q, k, ff, bf, cfg)
        g = f32(port.uniform(16, -1, 1, fw["sims"].size).reshape(fw["sims"].shape))
        _cache[metric] = (cfg, q, k, ff, bf, fw, g)
    return _cache[metric]


def device_tape_from(fw, cfg):
    """The oracle's selection as the device tape (fp32 offsets, relative fp32 chains)."""
    return fw["offsets"].astype(np.float32), rel_chains(fw["chains"], cfg, T, H, W, fw["offsets"]).astype(np.float32)


def same_fp32_tape(offs32, chains32, cfg):
    """The fp64 reference tape that the fp32 device tape encodes (centres = query + offset)."""
    rows = offs32.shape[0]
    nh, nw = (H - 1) // cfg.stride0 + 1, (W - 1) // cfg.stride0 + 1
    r = np.arange(rows)
    base = np.stack([r // (nh * nw), ((r // nw) % nh) * cfg.stride0, (r % nw) * cfg.stride0], -1)
    cen = base[:, None, :].astype(np.float64) + offs32.astype(np.float64)
    ch = chains32.astype(np.float64).copy()
    dt = np.abs(np.rint(offs32[..., 0])).astype(int)
    used = np.arange(ch.shape[2])[None, None, :] < (dt - 1)[..., None]
    ch[..., 0] += np.where(used, base[:, None, None, 1], 0)
    ch[..., 1] += np.where(used, base[:, None, None, 2], 0)
    return cen, ch


def run_bwd(S, cfg, q, k, g, offs=None, chains=None, tape64=None, deterministic=False):
    res = S.SearchResult(sims=dev(np.zeros(g.shape)), offsets=dev(offs) if offs is not None else None,
                         chains=dev(chains) if chains is not None else None, cfg=scfg(cfg))
    t64 = None
    if tape64 is not None:
        import torch

        t64 = tuple(torch.tensor(np.ascontiguousarray(x), device="cuda", dtype=torch.float64)
                    for x in tape64)
    out = S.shifted_nls_backward(dev(g), res, dev(q), dev(k), deterministic=deterministic, tape64=t64)
    return [host(x) for x in out]


KEYS = ("dq", "dk", "dfflow", "dbflow")


@pytest.mark.parametrize("metric", ["ip", "l2"])
def test_c3_backward_device_tape_vs_oracle(port, metric):
    S = snls_mod()
    cfg, q, k, ff, bf, fw, g = c3_case(port, metric)
    offs32, ch32 = device_tape_from(fw, cfg)
    got = run_bwd(S, cfg, q, k, g, offs32, ch32)
    cen, ch = same_fp32_tape(offs32, ch32, cfg)
    want = port.search_bwd(q, k, cfg, cen, ch, g)
    for a, key in zip(got, KEYS):
        err = max_rel(a, want[key])
        print(f"[c3 {metric}] device tape {key}: max rel {err:.2e}")
        assert err <= REL_TOL, (key, err)


@pytest.mark.parametrize("deterministic", [False, True])
@pytest.mark.parametrize("metric", ["ip", "l2"])
def test_c3_backward_reference_tape_vs_oracle(port, metric, deterministic):
    """The reference's own fp64 tape in, every gradient (flows included) within 1e-5."""
    S = snls_mod()
    cfg, q, k, ff, bf, fw, g = c3_case(port, metric)
    got = run_bwd(S, cfg, q, k, g, tape64=(fw["centers"], fw["chains"]), deterministic=deterministic)
    want = port.search_bwd(q, k, cfg, fw["centers"], fw["chains"], g)
    for a, key in zip(got, KEYS):
        err = max_rel(a, want[key])
        print(f"[c3 {metric} det={deterministic}] reference tape {key}: max rel {err:.2e}")
        assert err <= REL_TOL, (key, err)
    if deterministic:
        again = run_bwd(S, cfg, q, k, g, tape64=(fw["centers"], fw["chains"]), deterministic=True)
        for a, b, key in zip(got, again, KEYS):
            assert np.array_equal(a, b), f"deterministic {key} differs between runs"


@pytest.mark.parametrize("metric", ["ip", "l2"])
def test_c3_device_forward_tape64_is_the_reference_tape(port, metric):
    """GPU forward -> snls_search_tape64 reproduces the reference's centres and chains on the
    rows where the selection agrees (compare_search checks the rest), and the training step
    run entirely on the device (forward, tape64, backward) matches the oracle's gradients
    of the same selection."""
    import torch

    S = snls_mod()
    cfg, q, k, ff, bf, fw, g = c3_case(port, metric)
    dff, dbf = dev(ff), dev(bf)
    r = S.shifted_nls_forward(dev(q), dev(k), dff, dbf, scfg(cfg), want_weights=True)
    st = compare_search(r, oracle_ranked(port, q, k, ff, bf, cfg), cfg, q, k, label=f" c3 {metric}")
    cen, ch = S.search_tape64(r, dff, dbf)
    cen, ch = cen.cpu().numpy(), ch.cpu().numpy()
    same = np.all(np.abs(host(r.offsets) - fw["offsets"]) <= 1e-5, axis=(1, 2))
    assert same.mean() >= 0.99, st
    assert np.max(np.abs(cen[same] - fw["centers"][same])) <= 1e-9  # (shift on the 2^-32 grid)
    assert np.max(np.abs(ch[same] - fw["chains"][same])) <= 1e-9
    got = [host(x) for x in S.shifted_nls_backward(dev(g), r, dev(q), dev(k),
                                                   tape64=(torch.tensor(cen, device="cuda"),
                                                           torch.tensor(ch, device="cuda")))]
    want = port.search_bwd(q, k, cfg, cen, ch, g)
    for a, key in zip(got, KEYS):
        assert max_rel(a, want[key]) <= REL_TOL, (key, max_rel(a, want[key]))


@pytest.mark.parametrize("metric", ["ip", "l2"])
def test_c3_wpsum_backward_vs_oracle(port, metric):
    S = snls_mod()
    cfg, q, k, ff, bf, fw, g = c3_case(port, metric)
    v = video(port, T, H, W, F, 13)
    wts = port.softmax_rows(fw["sims"], cfg.softmax_scale)
    out, counts = S.wpsum(dev(v), dev(wts), dev(fw["offsets"]), scfg(cfg))
    want, wc = port.wpsum(v, wts, fw["offsets"], cfg)
    assert np.array_equal(host(counts), wc)
    assert max_rel(host(out), want) <= REL_TOL
    go = f32(port.uniform(17, -1, 1, v.size).reshape(v.shape))
    dv, dw = S.wpsum_backward(dev(go), counts, dev(v), dev(wts), dev(fw["offsets"]), scfg(cfg))
    wdv, wdw = port.wpsum_bwd(go, wc, v, wts, fw["offsets"], cfg)
    print(f"[c3 {metric}] dV {max_rel(host(dv), wdv):.2e} dW {max_rel(host(dw), wdw):.2e}")
    assert max_rel(host(dv), wdv) <= REL_TOL
    assert max_rel(host(dw), wdw) <= REL_TOL


def test_deterministic_backward_random_configs(port):
    """Every phase-1 kernel (row-centric ps <= 7 at F 1..64, entry-centric ps 9) and the chain
    route in the deterministic mode: bitwise reproducible and within 1e-5 of the oracle."""
    S = snls_mod()
    rng = np.random.default_rng(4242)
    done = 0
    for i in range(16):
        t = int(rng.integers(2, 5))
        h, w = int(rng.integers(6, 12)), int(rng.integers(6, 12))
        f = int(rng.choice([1, 3, 4, 32, 40, 64]))
        ps = int(rng.choice([1, 3, 5, 7, 9]))
        cfg = Cfg(ws=int(rng.choice([3, 5])), wt=int(rng.integers(0, 3)), ps=ps,
                  stride0=int(rng.integers(1, 3)), stride1=float(rng.choice([1.0, 0.5])),
                  topl=int(rng.integers(1, 5)), metric=str(rng.choice(["ip", "l2"])))
        q, k = video(port, t, h, w, f, 61000 + i), video(port, t, h, w, f, 62000 + i)
        ff, bf = flow(port, t, h, w, 63000 + i, 1.5), flow(port, t, h, w, 64000 + i, 1.5)
        try:
            fw = port.search_fwd(q, k, ff, bf, cfg)
        except Exception:
            continue
        g = f32(port.uniform(65000 + i, -1, 1, fw["sims"].size).reshape(fw["sims"].shape))
        want = port.search_bwd(q, k, cfg, fw["centers"], fw["chains"], g)
        a = run_bwd(S, cfg, q, k, g, tape64=(fw["centers"], fw["chains"]), deterministic=True)
        b = run_bwd(S, cfg, q, k, g, tape64=(fw["centers"], fw["chains"]), deterministic=True)
        for x, y, key in zip(a, b, KEYS):
            assert np.array_equal(x, y), (i, key)
            assert max_rel(x, want[key]) <= REL_TOL, (i, key, max_rel(x, want[key]))
        done += 1
    assert done >= 10


@pytest.mark.parametrize("metric", ["ip", "l2"])
def test_train_backward_self_similarity_vs_oracle(port, metric):
    """snls_train_bwd with Q = K = V aliased (run_benchmark's self-similarity use) at the c3
    shape, from the fp64 tape, against the oracle's two backward operators: dQ, dK, dV, dW,
    dFflow, dBflow.  (With Q = K the self-matches make the flow gradients large and
    cancelling: the fp32 device tape's rounded positions then cost up to ~2e-5 there, the
    fp64 tape keeps them at ~3e-6 -- the training path takes the fp64 tape.)"""
    tape = "fp64"
    import torch

    S = snls_mod()
    cfg, q, _, ff, bf, _, _ = c3_case(port, metric)
    k = v = q  # aliased
    fw = port.search_fwd(q, k, ff, bf, cfg)
    g = f32(port.uniform(16, -1, 1, fw["sims"].size).reshape(fw["sims"].shape))
    wts = port.softmax_rows(fw["sims"], cfg.softmax_scale)
    _, counts = port.wpsum(v, wts, fw["offsets"], cfg)
    go = f32(port.uniform(17, -1, 1, v.size).reshape(v.shape))
    offs32, ch32 = device_tape_from(fw, cfg)
    res = S.SearchResult(sims=dev(fw["sims"]), offsets=dev(offs32), chains=dev(ch32), weights=dev(wts),
                         cfg=scfg(cfg))
    t64 = None
    if tape == "fp64":
        cen, ch = fw["centers"], fw["chains"]
        t64 = (torch.tensor(cen, device="cuda"), torch.tensor(ch, device="cuda"))
    else:
        cen, ch = same_fp32_tape(offs32, ch32, cfg)
    dq_, dk_, dv_, dff_, dbf_, dw_ = [host(x) for x in S.train_backward(
        dev(g), dev(go), dev(counts), res, dev(q), dev(k), dev(v), tape64=t64)]
    sb = port.search_bwd(q, k, cfg, cen, ch, g)
    wdv, wdw = port.wpsum_bwd(go, counts, v, wts, fw["offsets"], cfg)
    for got, want, name in ((dq_, sb["dq"], "dq"), (dk_, sb["dk"], "dk"), (dff_, sb["dfflow"], "dfflow"),
                            (dbf_, sb["dbflow"], "dbflow"), (dv_, wdv, "dv"), (dw_, wdw, "dw")):
        err = max_rel(got, want)
        print(f"[c3 fused {metric} {tape}] {name}: max rel {err:.2e}")
        assert err <= REL_TOL, (name, err)
