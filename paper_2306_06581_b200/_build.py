"""In-tree build of the native libraries (no JIT cache, so the .so files travel
with the repo snapshot to the GPU box).

  libspk_b200.so       CUDA kernels + the C ABI (include/spk.h), sm_100a
  libsparsink_b200.so  C++ drop-in shim (namespace sparsink, include/sparsink_b200.hpp)
                       over the C ABI
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CUDA_SOURCES = ["spk_api.cu", "sampler.cu", "loop.cu", "blocked.cu", "dense.cu", "readout.cu", "shard.cu", "ibp.cu", "batch.cu", "small.cu", "comm.cu", "sharded.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
              "-Xptxas", "-v", "-I", str(ROOT / "include")]

LIB = PKG / "libspk_b200.so"
SHIM = PKG / "libsparsink_b200.so"


def _run(cmd: list[str], log: Path | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    deps = [CSRC / s for s in CUDA_SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [
        ROOT / "include" / "spk.h"]
    build_dir = PKG / "_obj"
    build_dir.mkdir(exist_ok=True)
    if force or _stale(LIB, deps):
        from concurrent.futures import ThreadPoolExecutor

        objs, todo = [], []
        for src in CUDA_SOURCES:
            obj = build_dir / (Path(src).stem + ".o")
            if force or _stale(obj, deps):
                todo.append((src, obj))
            objs.append(str(obj))

        def compile_one(item):
            src, obj = item
            _run([NVCC, *ARCH, *NVCC_FLAGS, "-c", str(CSRC / src), "-o", str(obj)],
                 log=build_dir / (Path(src).stem + ".ptxas.txt"))
            if verbose:
                print("compiled", src)

        with ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4) or 1) as ex:
            list(ex.map(compile_one, todo))
        # no link-time NCCL: comm.cu dlopens libnccl.so.2 when a communicator is made
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    shim_src = CSRC / "host" / "sparsink_b200.cpp"
    if shim_src.exists():
        shim_deps = [shim_src, ROOT / "include" / "sparsink_b200.hpp", ROOT / "include" / "spk.h"]
        if force or _stale(SHIM, shim_deps) or _stale(SHIM, [LIB]):
            _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", "-I", str(ROOT / "include"),
                  "-o", str(SHIM), str(shim_src), f"-L{PKG}", "-lspk_b200", f"-Wl,-rpath,{PKG}",
                  "-Wl,-rpath,$ORIGIN"])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
