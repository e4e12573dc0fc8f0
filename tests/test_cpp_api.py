"""The C++ host API (include/gcpb.hpp) compiles against the C-ABI and links
libgcpb.so (CPU); the demo runs on a GPU (gpu marker)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "cpp" / "host_api_demo.cpp"
LIBDIR = ROOT / "paper_1906_01687_b200"
EXE = ROOT / "tests" / "cpp" / "host_api_demo"


def _build():
    cmd = ["g++", "-std=c++17", "-O2", "-I", str(ROOT / "include"), str(SRC), "-o", str(EXE),
           f"-L{LIBDIR}", "-lgcpb", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_host_api_builds():
    _build()
    assert EXE.exists()


@pytest.mark.gpu
def test_cpp_host_api_runs():
    _build()
    out = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == "ok"
