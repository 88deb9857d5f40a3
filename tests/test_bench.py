"""bench.py on CPU: the work model reproduces SURVEY 8d's algorithmic-work table, and the
reference arm (`--impl reference`, the reference compiled from its sources in oracle/_ref)
prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.parametrize("name,extra,search,wpsum", [
    ("c4", {}, 8.68e10, 3.78e9),
    ("c2", {}, 6.06e9, 7.87e8),
    ("c5", {}, 2.56e12, 1.22e11),
    ("c2", {"stride0": 1}, 9.70e10, None),
])
def test_work_model_matches_survey(name, extra, search, wpsum):
    import bench

    m = bench.work_model(dict(bench.WORKLOADS[name], **extra))
    assert abs(m["search_instr"] / search - 1) < 0.01, m["search_instr"]
    if wpsum is not None:
        assert abs(m["wpsum_instr"] / wpsum - 1) < 0.01, m["wpsum_instr"]


def test_reference_arm_json_line():
    from oracle.oracle import have_reference

    if not have_reference():
        pytest.skip("oracle/_ref not built")
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--ref-crop", "16"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
