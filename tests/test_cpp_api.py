"""The header-only C++ drop-in API (include/fht_b200/fht.hpp, as_fht.hpp):
compiles here (CPU) and, on a GPU box, runs reference-style code bit-exactly
against the oracle."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "test_api.cpp"
BIN = ROOT / "build" / "test_cpp_api"


def _build():
    BIN.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", f"-I{ROOT / 'include'}", str(SRC), "-o", str(BIN),
           f"-L{ROOT / 'paper_2411_07351_b200'}", "-lfht_b200", f"-Wl,-rpath,{ROOT / 'paper_2411_07351_b200'}",
           str(ROOT / "oracle" / "liboracle.so"), f"-Wl,-rpath,{ROOT / 'oracle'}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_api_compiles():
    _build()
    assert BIN.exists()


@pytest.mark.gpu
def test_cpp_api_runs_bit_exact():
    _build()
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
