"""The bench.py JSON-line contract the driver parses (both arms)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"]


def _line(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_reference_arm_contract():
    from oracle.oracle import Oracle
    if not (Oracle.available("ref") or Oracle.available("orc")):
        pytest.skip("oracle not built")
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "0"], 600)
    for k in KEYS:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_self_launch_two_ranks():
    """--gpus 2 outside torchrun re-launches under torch.distributed.run: two
    ranks, the strong-scaling frame split and the max over ranks (gloo)."""
    d = _line(["--dry-run", "--gpus", "2", "--workload", "c5"], 300)
    assert d["dry_run"] and d["n_gpus"] == 2 and d["gpus_flag"] == 2
    assert d["frames_rank0"] == 512 and d["max_over_ranks"] == 2.0


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", "--gpus", "4"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr


@pytest.mark.gpu
def test_device_arm_contract():
    d = _line(["--frames", "32", "--batch", "16", "--steps", "1", "--warmup", "1",
               "--e2e-steps", "1", "--no-cpu-baseline", "--no-extensions", "--streams", "2"], 900)
    for k in KEYS + ["roofline", "gpu_launches", "clocks"]:
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] < 1
    assert d["parity"]["ok"] and d["parity"]["device_frames_checked"] == 4


@pytest.mark.gpu
@pytest.mark.parametrize("wl", ["c3", "c5"])
def test_device_arm_fhd_workloads(wl):
    d = _line(["--workload", wl, "--frames", "16", "--steps", "1", "--warmup", "1",
               "--e2e-steps", "1", "--no-cpu-baseline", "--no-extensions"], 1200)
    assert d["workload"] == wl and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["parity"]["ok"] and d["parity"]["device_frames_checked"] == 2
