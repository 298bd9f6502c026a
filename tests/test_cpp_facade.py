"""The C++ façade (include/flexcomm_b200/flexcomm.hpp) builds on CPU and its
reference-style tests (tests/cpp/test_facade.cpp) pass on a B200."""
from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2312_02493_b200"
SRC = ROOT / "tests" / "cpp" / "test_facade.cpp"
BIN = ROOT / "tests" / "cpp" / "test_facade"


def build() -> Path:
    cxx = shutil.which("g++") or "g++"
    cmd = [cxx, "-std=c++20", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}",
           f"-I{ROOT / 'tests' / 'cpp'}", str(SRC), f"-L{LIBDIR}", "-l:libfc_b200.so",
           f"-Wl,-rpath,{LIBDIR}", "-o", str(BIN)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return BIN


def test_facade_compiles():
    assert build().exists()


@pytest.mark.gpu
def test_facade_reference_tests_on_gpu():
    exe = build()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "[FAIL]" not in r.stdout
