"""CPU: pin the oracle.  The plain-C restatement (oracle/snls_oracle.c) must reproduce the
reference bit for bit -- against the committed golden fixtures (made by the reference
itself, tests/gen_golden.py) and, where oracle/_ref is built, against the reference live on
fresh random configs modelled on its own tests."""
import glob
import os

import numpy as np
import pytest

from oracle.oracle import Cfg, OracleError
from tests.helpers import draw_cfg, f32, flow, video

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cfg = Cfg(**eval(str(z["cfg"])))
    return z, cfg


def test_uniform_stream_matches_mt19937_64(port):
    # std::mt19937_64 with the default seed: the standard pins the 10000th output
    assert port.uniform_bits(5489, 9999) == 9981545732273789042
    v = port.uniform(7, 0.0, 1.0, 5)
    assert np.all((v >= 0) & (v < 1))


def test_reflect_and_bilinear_known_answers(port):
    # test_tensor.cpp:38-46
    assert port.reflect_index(-1, 8) == 1
    assert port.reflect_index(8, 8) == 6
    assert port.reflect_index(0, 8) == 0
    assert port.reflect_index(7, 8) == 7
    assert port.reflect_index(-3, 4) == 3
    assert port.reflect_index(9, 4) == 3
    assert port.reflect_index(5, 1) == 0
    z, _ = load("known_answers")
    for i, n, r in z["reflect"]:
        assert port.reflect_index(int(i), int(n)) == int(r)
    # test_tensor.cpp:64-71: 4x4 ramp 4y+x at (1.25, 2.5) -> 7.5
    idx, w = port.bilinear_taps(4, 4, 1.25, 2.5)
    ramp = z["ramp"][0, :, :, 0]
    val = (w[0] * ramp[idx[0], idx[2]] + w[1] * ramp[idx[0], idx[3]]
           + w[2] * ramp[idx[1], idx[2]] + w[3] * ramp[idx[1], idx[3]])
    assert abs(val - 7.5) < 1e-12


def test_softmax_known_answer(port):
    # test_aggregate.cpp:91-106
    z, _ = load("known_answers")
    w = port.softmax_rows(np.array([[2.0, 1.0, 0.0]]), 1.0)
    assert np.array_equal(w, z["softmax_210"])
    assert abs(w[0, 0] - 0.6652) < 1e-4 and abs(w[0, 1] - 0.2447) < 1e-4


@pytest.mark.parametrize("name", sorted(os.path.basename(p)[:-4]
                                        for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                                        if "known" not in p))
def test_port_reproduces_golden_bitwise(port, name):
    z, cfg = load(name)
    q, k = z["q"].astype(np.float64), z["k"].astype(np.float64)
    ff, bf = z["fflow"].astype(np.float64), z["bflow"].astype(np.float64)
    res = port.search_fwd(q, k, ff, bf, cfg)
    assert np.array_equal(res["sims"], z["sims"])
    assert np.array_equal(res["offsets"], z["offsets"])
    assert np.array_equal(res["chains"], z["chains"])
    if "wpsum" in z:
        v = z["v"].astype(np.float64)
        w = port.softmax_rows(res["sims"], cfg.softmax_scale)
        assert np.array_equal(w, z["weights"])
        out, counts = port.wpsum(v, w, res["offsets"], cfg)
        assert np.array_equal(out, z["wpsum"]) and np.array_equal(counts, z["counts"])
        assert np.array_equal(port.gather_stack(v, w, res["offsets"], cfg), z["stack"])
        if "dv" in z:
            dv, dw = port.wpsum_bwd(z["grad_out"].astype(np.float64), counts, v, w,
                                    res["offsets"], cfg)
            assert np.array_equal(dv, z["dv"]) and np.array_equal(dw, z["dweights"])
    if "dq" in z:
        g = port.search_bwd(q, k, cfg, res["centers"], res["chains"],
                            z["grad_sims"].astype(np.float64))
        for key in ("dq", "dk", "dfflow", "dbflow"):
            assert np.array_equal(g[key], z[key]), key


def test_port_matches_reference_on_random_configs(port, ref):
    rng = np.random.default_rng(2309)
    checked = 0
    for i in range(60):
        t = int(rng.integers(1, 4))
        h, w, f = int(rng.integers(4, 10)), int(rng.integers(4, 10)), int(rng.integers(1, 4))
        cfg = draw_cfg(rng, t, ws=(1, 3, 5), ps=(1, 3, 5), hole_free=True)
        q, k = video(port, t, h, w, f, 100 + i), video(port, t, h, w, f, 200 + i)
        ff, bf = flow(port, t, h, w, 300 + i, 1.5), flow(port, t, h, w, 400 + i, 1.5)
        try:
            a = ref.search_fwd(q, k, ff, bf, cfg)
        except OracleError as e:
            with pytest.raises(OracleError) as ei:
                port.search_fwd(q, k, ff, bf, cfg)
            assert str(ei.value) == str(e) and ei.value.code == e.code
            continue
        b = port.search_fwd(q, k, ff, bf, cfg)
        for key in a:
            assert np.array_equal(a[key], b[key]), (i, key)
        # the reference's own twins agree with its fused path (test_search.cpp:317-347)
        s = ref.serial_search_fwd(q, k, ff, bf, cfg)
        assert np.array_equal(s["sims"], a["sims"]) and np.array_equal(s["offsets"], a["offsets"])
        gs = f32(port.uniform(500 + i, -1, 1, a["sims"].size).reshape(a["sims"].shape))
        ga = ref.search_bwd(q, k, cfg, a["centers"], a["chains"], gs)
        gb = port.search_bwd(q, k, cfg, a["centers"], a["chains"], gs)
        for key in ga:
            assert np.array_equal(ga[key], gb[key]), (i, key)
        wts = port.softmax_rows(a["sims"], 1.0)
        oa, ca = ref.wpsum(k, wts, a["offsets"], cfg)
        ob, cb = port.wpsum(k, wts, a["offsets"], cfg)
        assert np.array_equal(oa, ob) and np.array_equal(ca, cb)
        assert np.array_equal(ref.gather_stack(k, wts, a["offsets"], cfg),
                              port.gather_stack(k, wts, a["offsets"], cfg))
        go = f32(port.uniform(600 + i, -1, 1, q.size).reshape(q.shape))
        for x, y in zip(ref.wpsum_bwd(go, ca, k, wts, a["offsets"], cfg),
                        port.wpsum_bwd(go, ca, k, wts, a["offsets"], cfg)):
            assert np.array_equal(x, y)
        checked += 1
    assert checked >= 30


def test_validation_messages_match_reference(port, ref):
    bad = [Cfg(ws=4), Cfg(ps=2), Cfg(wt=-1), Cfg(stride0=0), Cfg(stride1=0.0),
           Cfg(stride1=float("inf")), Cfg(topl=1000), Cfg(softmax_scale=float("nan"))]
    for c in bad:
        with pytest.raises(OracleError) as a:
            ref.validate(c)
        with pytest.raises(OracleError) as b:
            port.validate(c)
        assert str(a.value) == str(b.value) and a.value.code == b.value.code == 1


def test_underfull_and_hole_errors(port):
    # test_search.cpp:509-537 / test_aggregate.cpp:259-276
    q = video(port, 2, 6, 6, 1, 127)
    ff, bf = flow(port, 2, 6, 6, 129, 1.0), flow(port, 2, 6, 6, 130, 1.0)
    with pytest.raises(OracleError, match="topl exceeds"):
        port.search_fwd(q, q, ff, bf, Cfg(ws=3, wt=1, ps=1, topl=27))
    v = video(port, 1, 6, 6, 1, 71)
    with pytest.raises(OracleError, match="hole-free"):
        port.wpsum(v, np.ones((36, 1)), np.zeros((36, 1, 3)), Cfg(ws=3, ps=3, stride0=1, topl=1))


# ---- frame-alignment pieces: the restatement vs the reference -----
def _ref():
    from oracle.oracle import Checker, have_reference

    if not have_reference():
        pytest.skip("oracle/_ref not built")
    return Checker("reference")


def test_block_match_port_equals_reference():
    from oracle.oracle import Checker

    P, R = Checker("port"), _ref()
    rng = np.random.default_rng(5)
    for i in range(6):
        h, w, f = int(rng.integers(5, 23)), int(rng.integers(5, 23)), int(rng.choice([1, 3]))
        block, radius = int(rng.choice([1, 3, 5, 9])), int(rng.integers(0, 5))
        a = np.floor(P.uniform(700 + i, 0, 256, h * w * f)).reshape(h, w, f)
        b = np.roll(a, (1, -2), axis=(0, 1)) if i % 2 else np.floor(P.uniform(800 + i, 0, 256, h * w * f)).reshape(h, w, f)
        assert np.array_equal(P.block_match(a, b, block, radius), R.block_match(a, b, block, radius))
    with pytest.raises(Exception, match="block must be odd"):
        P.block_match(np.zeros((4, 4, 1)), np.zeros((4, 4, 1)), 2, 1)


def test_psnr_and_gaussian_noise_port_equal_reference():
    from oracle.oracle import Checker

    P, R = Checker("port"), _ref()
    v = P.uniform(31, 0, 255, 2 * 5 * 7 * 3).reshape(2, 5, 7, 3)
    for sigma, seed in ((0.0, 1), (10.0, 7), (25.0, 123)):
        assert np.array_equal(P.add_gaussian_noise(v, sigma, seed), R.add_gaussian_noise(v, sigma, seed))
    n = R.add_gaussian_noise(v, 15.0, 3)
    assert P.psnr(n, v) == R.psnr(n, v)
    assert P.psnr(v, v) == np.inf


@pytest.mark.parametrize("source", [0, 2])
def test_align_frames_composition_equals_reference(source):
    """The oracle's composition of the restated pieces reproduces snls::align_frames."""
    from oracle.oracle import Cfg, Checker

    P, R = Checker("port"), _ref()
    t, h, w, f = 3, 14, 12, 3
    clean = np.floor(P.uniform(41, 0, 256, t * h * w * f)).reshape(t, h, w, f)
    cfg = Cfg(ws=5, wt=0, ps=3, stride0=2, stride1=1.0, topl=1, metric="l2", softmax_scale=1.0)
    a = P.align_frames(clean, cfg, source=source, sigma=8.0, seed=9, bm_block=5, bm_radius=2)
    b = R.align_frames(clean, cfg, source=source, sigma=8.0, seed=9, bm_block=5, bm_radius=2)
    for k in ("aligned", "offsets", "used_flow", "psnr"):
        assert np.array_equal(a[k], b[k]), k
