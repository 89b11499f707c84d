"""CPU: bench.py's reference arm prints one JSON line with the contract keys
(the B200 arm needs a GPU and is exercised by the driver on the box)."""

import json
import os
import subprocess
import sys

from conftest import REPO


def test_reference_arm_json_line():
    env = dict(os.environ)
    out = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
         "--workload", "c1"],
        capture_output=True, text=True, timeout=600, env=env, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_is_silent_on_nonzero_ranks():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0"],
        capture_output=True, text=True, timeout=300, env=env, cwd=REPO)
    assert out.returncode == 0
    assert out.stdout.strip() == ""


def test_gpus_n_launches_n_ranks_with_the_c5_strong_record():
    """`bench.py --gpus 2` outside torchrun re-launches itself with one rank
    per GPU (torch.distributed.run, rendezvous on 127.0.0.1); the CPU plumbing
    mode runs the rank split of the C5 window and the per-step all-reduce over
    gloo and prints n_gpus == 2 with a c5_strong record whose parts tile the
    window."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--selftest-cpu", "--gpus", "2", "--c5-steps", "2"],
        capture_output=True, text=True, timeout=600, env=env, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    c5 = d["c5_strong"]
    assert c5["n_ranks"] == 2 and c5["covers_window"] and len(c5["parts"]) == 2


def test_both_arms_print_the_same_config():
    """The reference arm's config dict equals the one the B200 arm prints
    (bench.workload_config); run-specific details live under other keys."""
    sys.path.insert(0, REPO)
    import bench

    env = dict(os.environ, TRITPERM_BENCH_NUMBA="0")
    out = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
         "--workload", "c2"],
        capture_output=True, text=True, timeout=600, env=env, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")][0])
    assert d["config"] == bench.workload_config("c2")
    assert d["sample_per_step"]["terms"] > 0 and d["ms_per_step"] < 60_000
