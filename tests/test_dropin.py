"""The C++ drop-in adapter: libsnls_gpu.so defines the reference's search.hpp/aggregate.hpp
surface (CPU check of the exported symbols) and passes the in-process comparison against the
reference compiled as namespace snls_ref (GPU test running host/build/test_dropin)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "paper_2309_16849_b200", "host", "build")
LIB = os.path.join(HOST, "libsnls_gpu.so")
BIN = os.path.join(HOST, "test_dropin")

# every function search.cpp / aggregate.cpp define (search.hpp:27-175, aggregate.hpp:22-85)
API = ["snls::SearchConfig::validate() const", "snls::ExecPolicy::resolved_threads() const",
       "snls::QueryGrid::over(int, int, int, int)", "snls::temporal_scan_order(int)",
       "snls::shifted_nls_forward(", "snls::nls_forward(", "snls::top_l(",
       "snls::shifted_nls_backward(", "snls::replay_similarities(",
       "snls::detail::accumulate_shift(", "snls::detail::patch_similarity(",
       "snls::softmax_rows(", "snls::wpsum(", "snls::gather_stack(", "snls::wpsum_backward("]


def _exports():
    out = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True).stdout
    return out


@pytest.mark.skipif(not os.path.exists(LIB), reason="adapter not built (needs /root/reference headers)")
def test_adapter_exports_the_reference_api():
    text = _exports()
    missing = [a for a in API if a not in text]
    assert not missing, missing


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in test binary not built")
def test_dropin_against_reference_in_process():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
