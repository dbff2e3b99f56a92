"""The C++ mirror of the reference API (include/csf/b200.hpp) runs the
reference's own TSDF/ICP test cases on the device (tests/cpp/api_parity.cpp,
oracle as checker).  Compiling it needs no GPU; running it does."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "api_parity.cpp"
BIN = ROOT / "tests" / "cpp" / "_build" / "api_parity"
LIBDIR = ROOT / "paper_2405_02187_b200" / "_build"


def build():
    if not (LIBDIR / "libcsf_b200.so").exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "paper_2405_02187_b200")], check=True)
    BIN.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-fopenmp", f"-I{ROOT / 'include'}",
           f"-I{ROOT / 'oracle'}", str(SRC), f"-L{LIBDIR}", "-lcsf_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(BIN)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_cpp_api_compiles():
    build()
    assert BIN.exists()


@pytest.mark.gpu
def test_cpp_api_reference_cases_on_device():
    if not BIN.exists() or BIN.stat().st_mtime < max(SRC.stat().st_mtime, (ROOT / "include" / "csf" / "b200.hpp").stat().st_mtime,
                                                     (ROOT / "include" / "csf" / "csf.hpp").stat().st_mtime):
        build()
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "failures=0" in r.stdout
