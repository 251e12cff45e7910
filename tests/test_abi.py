"""The drop-in boundary on CPU: the C-ABI library loads, exports exactly what
include/spk.h declares, and the ctypes stub binds every entry point.
No compute calls (no GPU here)."""
import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "spk.h"


def declared_functions(header: Path) -> set[str]:
    text = re.sub(r"/\*.*?\*/", "", header.read_text(), flags=re.S)
    return set(re.findall(r"\b(spk_[a-z_0-9]+)\s*\(", text))


def exported_symbols(lib: Path) -> set[str]:
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_library_built_and_loads():
    from paper_2306_06581_b200 import _lib

    lib = _lib.load()
    assert isinstance(lib, ctypes.CDLL)


def test_every_declared_symbol_is_exported():
    from paper_2306_06581_b200 import _lib

    decl = declared_functions(HEADER)
    assert len(decl) >= 20
    missing = decl - exported_symbols(_lib.LIB_PATH)
    assert not missing, f"declared in spk.h but not exported: {sorted(missing)}"


def test_ctypes_stub_covers_header():
    from paper_2306_06581_b200 import _lib

    assert declared_functions(HEADER) == set(_lib.SIGNATURES)


def test_struct_layouts_match_header():
    """ctypes structs must match the C layout (sizes computed by the C compiler)."""
    from paper_2306_06581_b200 import _lib as L

    src = r"""
    #include <stdio.h>
    #include "spk.h"
    int main(void){printf("%zu %zu %zu %zu\n", sizeof(spk_kernel_desc), sizeof(spk_solver_cfg),
                          sizeof(spk_sketch_opts), sizeof(spk_report)); return 0;}
    """
    exe = Path("/tmp/spk_sizes")
    res = subprocess.run(["gcc", "-x", "c", "-", "-I", str(ROOT / "include"), "-o", str(exe)], input=src,
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    sizes = [int(s) for s in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert sizes == [ctypes.sizeof(L.KernelDesc), ctypes.sizeof(L.SolverCfg), ctypes.sizeof(L.SketchOpts),
                     ctypes.sizeof(L.Report)]


def test_header_compiles_as_c_and_cpp():
    for lang, comp in (("c", "gcc"), ("c++", "g++")):
        res = subprocess.run([comp, "-x", lang, "-fsyntax-only", "-Wall", "-Wextra", "-I", str(ROOT / "include"), "-"],
                             input='#include "spk.h"\nint main(void){return SPK_ABI_VERSION - 1;}\n',
                             capture_output=True, text=True)
        assert res.returncode == 0, res.stderr


def test_no_device_fails_loudly():
    """Without a GPU the product refuses to run (no CPU fallback)."""
    import paper_2306_06581_b200 as spk

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(spk.SparsinkError):
        spk.Context(0)


def test_error_classes_mirror_reference():
    """Exception classes and categories of errors.hpp:30-47."""
    import paper_2306_06581_b200 as spk

    names = {"NegativeWeight", "LengthMismatch", "NotNormalized", "AllBlack", "EmptyOutput", "DimensionMismatch",
             "NonPositiveEta", "NonPositiveEpsilon", "DegenerateSupport", "AllZeroKernel", "ThetaOutOfRange",
             "BudgetTooLarge", "EmptyWindow", "InfiniteCostOnSupport", "IoError", "ZeroDenominator",
             "BaselineFailed", "DegenerateSketchError"}
    assert names <= set(spk.ERRORS)
    for n in names:
        assert issubclass(spk.ERRORS[n], spk.SparsinkError)
