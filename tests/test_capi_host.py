"""CPU: the C-ABI library loads, exports every entry point include/snls_cuda.h declares,
and its host-side logic (validation messages, query grid, synthetic-input RNG, error codes)
matches the reference -- no device needed."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle.oracle import Cfg, OracleError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "snls_cuda.h")


@pytest.fixture(scope="module")
def S():
    from paper_2309_16849_b200 import build, snls

    build.build()
    return snls


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(snls_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("snls_search_fwd", "snls_topl", "snls_replay", "snls_search_bwd",
                 "snls_softmax_rows", "snls_wpsum_fwd", "snls_gather_stack", "snls_wpsum_bwd",
                 "snls_ctx_create", "snls_ctx_sync_check", "snls_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol(S):
    lib = C.CDLL(S.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.snls_abi_version() == 1


def test_validation_messages_equal_the_reference(S, port):
    bad = [Cfg(ws=4), Cfg(ps=2), Cfg(wt=-1), Cfg(stride0=0), Cfg(stride1=0.0),
           Cfg(stride1=float("inf")), Cfg(topl=1000), Cfg(softmax_scale=float("nan"))]
    for c in bad:
        with pytest.raises(OracleError) as want:
            port.validate(c)
        with pytest.raises(S.ConfigError) as got:
            S.validate(S.SearchConfig(**c.__dict__))
        assert str(got.value) == str(want.value)
    S.validate(S.SearchConfig(ws=3, topl=9))


def test_query_grid(S, port):
    for (t, h, w, s) in ((3, 64, 64, 1), (5, 128, 128, 4), (10, 256, 256, 2), (2, 7, 9, 3)):
        rows, nh, nw = S.query_grid(t, h, w, s)
        assert (nh, nw) == ((h - 1) // s + 1, (w - 1) // s + 1)
        from oracle.oracle import query_grid

        assert rows == query_grid(t, h, w, s)[0]


def test_uniform_fill_is_the_reference_stream(S, port):
    for seed, lo, hi in ((1, 0.0, 255.0), (100, -1.0, 1.0), (501, -2.0, 2.0)):
        got = S.uniform_fill(seed, lo, hi, 4096)
        want = port.uniform(seed, lo, hi, 4096).astype(np.float32)
        assert np.array_equal(got, want)


def test_no_device_is_a_loud_error(S):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    lib = C.CDLL(S.LIB_PATH)
    h = C.c_void_p()
    rc = lib.snls_ctx_create(0, None, C.byref(h))
    assert rc == 3  # SNLS_ECUDA, never a CPU fallback
    lib.snls_last_error.restype = C.c_char_p
    assert b"device" in lib.snls_last_error()


def test_null_arguments_rejected_before_any_device_work(S):
    lib = C.CDLL(S.LIB_PATH)
    lib.snls_last_error.restype = C.c_char_p
    assert lib.snls_search_fwd(None, None, S._Dims(1, 1, 1, 1), None, None, None, None, 0,
                               None, None, None, None) == 4
    # the backward entry points (null context first), including the round-2 additions
    d = S._Dims(1, 1, 1, 1)
    assert lib.snls_wpsum_bwd_ex(None, None, d, 0, 1, *([None] * 7), 1) == 4
    assert lib.snls_search_bwd_ex(None, None, d, 0, 1, *([None] * 11), 1) == 4
    assert lib.snls_train_bwd(None, None, d, *([None] * 17), 1) == 4
    assert b"context" in lib.snls_last_error()


def test_host_gaussian_noise_matches_reference_stream():
    """snls_gaussian_noise_f32 (host side of align_frames) == add_gaussian_noise with the
    reference's GaussianStream (rng.hpp:30-53), rounded to fp32 -- no device needed."""
    import numpy as np

    from oracle.oracle import Checker
    from paper_2309_16849_b200 import snls as S

    P = Checker("port")
    v = np.floor(P.uniform(3, 0, 256, 2 * 6 * 5 * 3)).reshape(2, 6, 5, 3).astype(np.float32)
    for sigma, seed in ((0.0, 1), (4.0, 2), (30.0, 99)):
        want = P.add_gaussian_noise(v.astype(np.float64), sigma, seed).astype(np.float32)
        assert np.array_equal(S.add_gaussian_noise(v, sigma, seed), want)
    with pytest.raises(S.ConfigError, match="sigma must be non-negative"):
        S.add_gaussian_noise(v, -1.0, 0)
