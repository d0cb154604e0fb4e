"""In-tree build of libdpb200.so (sm_100a CUDA kernels + C++ host + C-ABI).

Kernels: nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3.
Host C++: g++ -O2 -ffp-contract=off (bit-identical fixture generators, see host_gen.cpp).
The library is written to paper_2201_01446_b200/lib/ so it travels with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "lib" / "libdpb200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ... ({r.returncode})")


def _deps() -> float:
    newest = 0.0
    for p in list(CSRC.glob("*")) + [ROOT / "include" / "dp_b200.h", Path(__file__)]:
        newest = max(newest, p.stat().st_mtime)
    return newest


def build(verbose: bool = False, force: bool = False) -> Path:
    """Compile every source; relink when anything changed. Returns the library path."""
    nvcc = _nvcc()
    OBJ.mkdir(parents=True, exist_ok=True)
    LIB.parent.mkdir(parents=True, exist_ok=True)
    newest = _deps()
    if LIB.exists() and not force and LIB.stat().st_mtime >= newest:
        return LIB
    inc = ["-I", str(ROOT / "include"), "-I", str(CSRC)]
    objs = []
    jobs = []
    for src in sorted(CSRC.glob("*.cu")):
        o = OBJ / (src.stem + ".cu.o")
        objs.append(o)
        jobs.append([nvcc, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                     "--expt-relaxed-constexpr", *inc, "-c", str(src), "-o", str(o)])
    for src in sorted(CSRC.glob("*.cpp")):
        o = OBJ / (src.stem + ".cpp.o")
        objs.append(o)
        jobs.append(["/usr/bin/g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-fopenmp",
                     "-Wall", "-Wno-unused-function", *inc, "-I", "/usr/local/cuda/include",
                     "-c", str(src), "-o", str(o)])
    procs = []
    for cmd in jobs:
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                            text=True)))
    failed = False
    for cmd, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"FAILED: {' '.join(cmd)}\n{out}{err}\n")
        elif verbose and (out or err):
            sys.stderr.write(out + err)
    if failed:
        raise RuntimeError("libdpb200 build failed")
    tmp = LIB.with_suffix(".so.tmp")
    _run([nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lgomp", "-lnccl"], verbose)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
