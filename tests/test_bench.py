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


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_flag_self_launches_n_ranks(n):
    """`python bench.py --gpus N` (no torchrun environment) re-launches itself as N ranks and
    rank 0 reports n_gpus == N with an N-rank communicator (gloo stand-in step on CPU)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--mock-cpu", "--steps", "3",
                        "--warmup", "3", "--videos-per-gpu", "2"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == n and line["comm"]["nranks"] == n
    assert line["config"]["videos_per_gpu"] == 2
    assert p.stderr.count("communicator nranks=") == n


def test_world_size_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--mock-cpu"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode != 0 and "WORLD_SIZE" in (p.stderr + p.stdout)
