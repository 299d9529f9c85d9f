"""The C++ reference-shaped adapter (include/warmgp_b200.hpp) compiles against
the C-ABI and, on a B200, runs the three solvers and the outer loop."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2405_18328_b200")
OUT = os.path.join(PKG, "_build", "adapter_test")


def build():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "adapter_test.cpp"), "-L", PKG, "-lwarmgp_b200",
           f"-Wl,-rpath,{PKG}", "-o", OUT]
    subprocess.run(cmd, check=True)
    return OUT


def test_adapter_compiles_and_links():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_adapter_runs_on_device():
    exe = build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "adapter ok" in r.stdout
