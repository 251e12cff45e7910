"""Compile the reference's own unit tests UNMODIFIED against the B200 C++
drop-in (test infrastructure, run by __graft_entry__.build()).

  /root/reference/proj/tests/{test_solvers,test_sparsify,test_geometry}.cpp
  + tests/cpp/shim/doctest.h          (own minimal doctest-compatible runner)
  + tests/cpp/shim/sparsink/*.hpp     (reference header names -> include/sparsink_b200.hpp)
  -> tests/cpp/_ref_tests/<name>      (git-ignored; travels to the GPU box)

The sources are read where they lie (never copied). tests/test_cpp_dropin.py
runs the binaries on the GPU."""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
REF_TESTS = Path("/root/reference/proj/tests")
NAMES = ["test_solvers", "test_sparsify", "test_geometry"]
OUT = ROOT / "tests" / "cpp" / "_ref_tests"


def build(quiet: bool = True) -> list[Path]:
    if not REF_TESTS.exists():
        if not quiet:
            print("reference tests not present; keeping prebuilt binaries (if any)")
        return sorted(OUT.glob("test_*"))
    OUT.mkdir(parents=True, exist_ok=True)
    pkg = ROOT / "paper_2306_06581_b200"
    out = []
    for name in NAMES:
        exe = OUT / name
        cmd = ["g++", "-std=c++20", "-O2", "-I", str(ROOT / "tests" / "cpp" / "shim"), "-I", str(ROOT / "include"),
               str(REF_TESTS / f"{name}.cpp"), "-o", str(exe), f"-L{pkg}", "-lsparsink_b200", "-lspk_b200",
               "-Wl,-rpath,$ORIGIN/../../../paper_2306_06581_b200", f"-Wl,-rpath,{pkg}"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stderr)
            raise RuntimeError(f"reference test {name} does not compile against the drop-in")
        out.append(exe)
    return out


if __name__ == "__main__":
    print(build(quiet=False))
