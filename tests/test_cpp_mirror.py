"""Runs the C++ mirror tests (tests/cpp/test_mirror.cpp): the reference's own
test cases written against include/cluspath/*.hpp over the C-ABI."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


def build():
    subprocess.run(["make", "-s", "-C", CPP], check=True)
    return os.path.join(CPP, "_build", "test_mirror")


def test_cpp_mirror_compiles():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_cpp_mirror_parity():
    exe = build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, cwd=CPP)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed; " in r.stdout
