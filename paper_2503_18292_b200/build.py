"""Build libjenga_b200.so in-tree: the host C++ runtime (g++ -std=c++20) and
the sm_100a kernels (nvcc -gencode arch=compute_100a,code=sm_100a), linked
into one shared library exporting only the C ABI of include/jenga_gpu.h.

No GPU is needed: nvcc cross-compiles.  Object files go to build/ (ignored);
the .so lands next to this file so it travels with the repository snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "jenga_b200"
LIB = PKG / "libjenga_b200.so"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--use_fast_math",
    "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v",
    "-I", str(ROOT / "include"),
]
CXX_FLAGS = ["-std=c++20", "-O2", "-g", "-fPIC", "-fvisibility=hidden", "-Wall", "-Wextra",
             "-I", str(ROOT / "include")]


def _sources():
    host = sorted((CSRC / "host").glob("*.cpp"))
    dev = sorted((CSRC / "kernels").glob("*.cu"))
    headers = list((CSRC).rglob("*.hpp")) + list(CSRC.rglob("*.cuh")) + [ROOT / "include" / "jenga_gpu.h"]
    return host, dev, headers


def _stale(obj: Path, src: Path, headers) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(h.stat().st_mtime > t for h in headers)


def _compile(cmd, log):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if log is not None:
        log.write(r.stderr)


def build(verbose: bool = False, force: bool = False) -> Path:
    host, dev, headers = _sources()
    BUILD.mkdir(parents=True, exist_ok=True)
    jobs = []
    objs = []
    for src in host:
        obj = BUILD / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, src, headers):
            jobs.append([CXX, *CXX_FLAGS, "-c", str(src), "-o", str(obj)])
    for src in dev:
        obj = BUILD / (src.stem + ".cu.o")
        objs.append(obj)
        if force or _stale(obj, src, headers):
            jobs.append([NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)])
    log_path = BUILD / "ptxas.log"
    with open(log_path, "a") as log:
        with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
            list(ex.map(lambda c: _compile(c, log), jobs))
    if jobs or force or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs),
                "-Xlinker", "--exclude-libs,ALL"]
        _compile(link, None)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_variant(name: str, defines) -> Path:
    """A profiling-only copy of the library with compile-time defines (e.g. a
    decode split policy), at paper_2503_18292_b200/variants/libjenga_b200_<name>.so;
    load it with JENGA_B200_LIB=<path>.  The product build is untouched."""
    build()
    host, dev, headers = _sources()
    vdir = ROOT / "build" / "variants" / name
    vdir.mkdir(parents=True, exist_ok=True)
    flags = [f"-D{d}" for d in defines]
    objs = []
    for src in dev:
        obj = vdir / (src.stem + ".cu.o")
        _compile([NVCC, *NVCC_FLAGS, *flags, "-c", str(src), "-o", str(obj)], None)
        objs.append(obj)
    objs += [BUILD / (src.stem + ".o") for src in host]
    out = PKG / "variants" / f"libjenga_b200_{name}.so"
    out.parent.mkdir(exist_ok=True)
    _compile([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(out), *map(str, objs),
              "-Xlinker", "--exclude-libs,ALL"], None)
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":  # --variant NAME DEFINE...
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        build(verbose=True, force="--force" in sys.argv)
