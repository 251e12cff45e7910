"""The C++ drop-in (include/sparsink_b200.hpp -> libsparsink_b200.so): the
reference's unit-test scenarios restated in C++ (tests/cpp/test_dropin.cpp),
built here with g++ and run on the GPU."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2306_06581_b200"


def _build(tmp_path: Path) -> Path:
    exe = tmp_path / "test_dropin"
    res = subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", str(ROOT / "include"),
                          str(ROOT / "tests" / "cpp" / "test_dropin.cpp"), "-o", str(exe), f"-L{PKG}",
                          "-lsparsink_b200", "-lspk_b200", f"-Wl,-rpath,{PKG}"], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return exe


def test_dropin_compiles_and_links(tmp_path):
    """CPU: the C++ API header compiles and links against the shim."""
    _build(tmp_path)


@pytest.mark.gpu
def test_dropin_reference_scenarios(tmp_path):
    exe = _build(tmp_path)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failed" in res.stdout
