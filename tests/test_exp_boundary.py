"""The K != 0 boundary of kernel_from_cost (geometry.cpp:95): the reference's
glibc exp is correctly rounded in the subnormal range, so exp(x) != 0 exactly
for x >= the double just above -1075 ln 2. The device's exp_ref
(csrc/common.cuh) hard-codes that boundary; here it is re-derived from the
host libm, and on the GPU the device K of costs straddling it is compared
with glibc's: support bit-exact (it fixes the sketch's draw counters),
subnormal values within a few quanta."""
import ctypes
import ctypes.util
import math
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
libm = ctypes.CDLL(ctypes.util.find_library("m"))
libm.exp.restype = ctypes.c_double
libm.exp.argtypes = [ctypes.c_double]


def _bits(x: float) -> int:
    return int(np.float64(x).view(np.int64))


def _from_bits(b: int) -> float:
    return float(np.int64(b).view(np.float64))


def test_boundary_constant_is_glibc():
    lo, hi = _bits(-745.0), _bits(-746.0)  # negative doubles: larger pattern = more negative
    assert libm.exp(_from_bits(lo)) != 0.0 and libm.exp(_from_bits(hi)) == 0.0
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if libm.exp(_from_bits(mid)) != 0.0:
            lo = mid
        else:
            hi = mid
    src = (ROOT / "paper_2306_06581_b200" / "csrc" / "common.cuh").read_text()
    const = float.fromhex(re.search(r"kExpLastNonzero = (-0x[0-9a-fp+.]+);", src).group(1))
    assert _from_bits(lo) == const
    assert libm.exp(const) == 5e-324 and libm.exp(math.nextafter(const, -math.inf)) == 0.0


@pytest.mark.gpu
def test_device_kernel_from_cost_matches_glibc_at_underflow(ctx):
    import ctypes as C

    from paper_2306_06581_b200 import _lib as L

    base = 745.13321910194110842
    cs = [math.nextafter(base, math.inf), base, math.nextafter(base, -math.inf)]
    rng = np.random.default_rng(3)
    cs += list(708.0 + 37.2 * rng.random(20000))  # the whole subnormal range
    cs += list(base + np.linspace(-1e-9, 1e-9, 2001))
    Cm = np.ascontiguousarray(cs, dtype=np.float64)
    K = np.empty_like(Cm)
    nnz = C.c_int64()
    rc = ctx.lib.spk_kernel_from_cost(ctx.ptr, L.dptr(Cm), len(Cm), 1.0, L.dptr(K), C.byref(nnz))
    assert rc == 0
    ref = np.array([libm.exp(-c) for c in Cm])
    assert np.array_equal(K != 0.0, ref != 0.0), "support differs from glibc"
    assert nnz.value == int(np.count_nonzero(ref))
    quanta = np.abs(K.view(np.int64) - ref.view(np.int64))
    assert quanta.max() <= 64, quanta.max()  # subnormal values: a few 2^-1074 quanta (relative ~1e-14 at the top)


def test_sequential_sum_emulation(tmp_path):
    """csrc/seqsum.h: the reference's sequential sum of N equal grid terms,
    emulated in O(binades): equal to the plain loop on random cases and to
    the committed 10^12-term config-4 normaliser (17 CPU-minutes to sum)."""
    import json
    import subprocess

    exe = tmp_path / "seqsum"
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-I",
                    str(ROOT / "paper_2306_06581_b200" / "csrc"), str(ROOT / "tests" / "cpp" / "test_seqsum.cpp"),
                    "-o", str(exe)], check=True)
    fx = json.loads((ROOT / "tests" / "golden" / "c4_normaliser.json").read_text())
    ra = math.sqrt(1.0 / 1_000_000) / float.fromhex(fx["sa"])
    res = subprocess.run([str(exe), (ra * ra).hex(), str(fx["kernel_nnz"])], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout
    assert float.fromhex(res.stdout.split()[-1]) == float.fromhex(fx["total"])
