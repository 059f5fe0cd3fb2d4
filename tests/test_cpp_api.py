"""Runs the C++ drop-in test (tests/cpp/test_api.cpp) against the GPU library."""
import os
import subprocess

import pytest

from conftest import ROOT

EXE = os.path.join(ROOT, "tests", "cpp", "build", "test_api")


def test_cpp_test_builds():
    from paper_2007_12623_b200.build import build
    build(verbose=False)
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_cpp_api_on_gpu():
    from paper_2007_12623_b200.build import build
    build(verbose=False)
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "test_api OK" in r.stdout
