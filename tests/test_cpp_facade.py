"""The C++ drop-in facade (include/sliceeig/*.hpp): compiles and links here (CPU), runs on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_acceptance.cpp")
PKG = os.path.join(ROOT, "paper_1802_05215_b200")
BIN = os.path.join(PKG, "_build", "dropin_acceptance")


def build_dropin():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", f"-I{os.path.join(ROOT, 'include')}", SRC, "-o", BIN,
           f"-L{PKG}", "-lsliceeig_cuda", f"-Wl,-rpath,{PKG}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return BIN


def test_facade_compiles_and_links():
    assert os.path.exists(build_dropin())


@pytest.mark.gpu
def test_facade_runs_reference_style_code_on_gpu():
    b = build_dropin()
    r = subprocess.run([b], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASSED" in r.stdout
