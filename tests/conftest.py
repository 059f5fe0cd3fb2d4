import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

PARAM_KEYS = ["window", "d_min", "d_max", "neighbor_jump_threshold", "outlier_radius_start",
              "outlier_radius_step", "cleanup_iterations", "fill_radius_radial",
              "fill_radius_disc", "smoothing_radius", "alpha", "eta_smooth",
              "refine_iterations", "min_zncc"]
INT_KEYS = {"window", "d_min", "d_max", "outlier_radius_start", "outlier_radius_step",
            "cleanup_iterations", "fill_radius_radial", "fill_radius_disc", "smoothing_radius",
            "refine_iterations"}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    out = {k: z[k] for k in z.files}
    if "params" in out:
        out["params"] = {k: (int(v) if k in INT_KEYS else float(v))
                         for k, v in zip(PARAM_KEYS, out["params"])}
    return out


GOLDEN_CHAINS = ["tex_d16", "low_d16", "tex_trace", "tex_default", "win7", "win13"]


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    if not Oracle.available("orc"):
        import subprocess
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True,
                       capture_output=True)
    return Oracle("orc")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle
    if not Oracle.available("ref"):
        pytest.skip("reference library oracle/_ref not built (needs /root/reference)")
    return Oracle("ref")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
