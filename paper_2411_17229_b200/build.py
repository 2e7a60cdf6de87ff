"""Build recipe for the native pieces (nvcc -> sm_100a, in-tree).

``build_native()`` compiles paper_2411_17229_b200/csrc/*.cu into
``paper_2411_17229_b200/libdade_gpu.so`` (the product: kernels + C ABI) and
``tests/cpp/host_api_test`` (the C++ mirror of the reference API exercised
by the GPU tests). Nothing here touches the oracle; __graft_entry__.build()
builds that separately as test infrastructure.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libdade_gpu.so"
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "-Xptxas", "-v", "--expt-relaxed-constexpr", "-cudart", "static",
]
SOURCES = ["scan.cu", "filter.cu", "umma.cu", "coarse.cu", "prep.cu", "seed.cu", "build.cu", "capi.cu", "comm.cu"]


def _run(cmd, log=None):
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(map(str, cmd))}\n{res.stdout}\n{res.stderr}")
    return res


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> Path:
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + \
        [ROOT / "include" / "dade_gpu.h", Path(__file__)]
    objdir = ROOT / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    if force or _stale(LIB, deps):
        objs = []
        headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "dade_gpu.h"]
        for s in SOURCES:
            o = objdir / (s + ".o")
            if force or _stale(o, [CSRC / s, *headers, Path(__file__)]):
                _run([NVCC, *NVCC_FLAGS, "-I", str(ROOT / "include"), "-c", str(CSRC / s), "-o", str(o)],
                     log=objdir / (s + ".log"))
            objs.append(str(o))
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *objs, "-ldl"])
    cpp_test = ROOT / "tests" / "cpp" / "host_api_test.cpp"
    if cpp_test.exists():
        exe = ROOT / "build" / "host_api_test"
        if force or _stale(exe, [cpp_test, ROOT / "include" / "dade_gpu.hpp", LIB]):
            _run(["g++", "-O2", "-std=c++20", "-I", str(ROOT / "include"), str(cpp_test), "-o", str(exe),
                  f"-L{PKG}", "-ldade_gpu", f"-Wl,-rpath,{PKG}"])
    return LIB


if __name__ == "__main__":
    print(build_native(force=True))
