"""Build the test oracles (TEST INFRASTRUCTURE ONLY — never imported by the
product package):

  oracle/_ref/liboracle.so    the plain-C restatement (jenga_oracle.c)
  oracle/_ref/libjenga_bridge_test.so  the reference-side bridge
                              (integration/jenga_gpu_bridge.hpp) compiled
                              against the reference headers, with the
                              reference objects and tests/bridge/
                              bridge_harness.cpp, linked to the product
                              library (tests/test_gpu_bridge.py);
  oracle/_ref/libjenga_ref.so the UNMODIFIED reference library compiled from
                              its own sources under /root/reference/proj/src
                              plus our extern "C" shim (ref_shim.cpp), when
                              /root/reference is present.  The reference needs
                              nlohmann/json (git-ignored vendor/ in the
                              reference, proj/.gitignore:2); we point at the
                              copy shipped with cudnn_frontend (3.11.3).

Outputs go only to oracle/_ref/ (git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "_ref"
REF = Path(os.environ.get("JENGA_REFERENCE", "/root/reference"))
REF_SRC = REF / "proj" / "src"
REF_INC = REF / "proj" / "include"


def _json_dir():
    cands = glob.glob(str(Path(sys.prefix) / "lib" / "python3*" / "site-packages" / "include" / "cudnn_frontend" /
                          "thirdparty" / "nlohmann"))
    cands += glob.glob("/opt/prime-rl/.venv/lib/python3*/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
    for c in cands:
        if Path(c, "json.hpp").exists():
            return c
    return None


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def _stale(out: Path, srcs) -> bool:
    return not out.exists() or any(Path(s).stat().st_mtime > out.stat().st_mtime for s in srcs)


def build_c_oracle() -> Path:
    OUT.mkdir(exist_ok=True)
    out = OUT / "liboracle.so"
    src = HERE / "jenga_oracle.c"
    if _stale(out, [src]):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-Wall", str(src), "-o", str(out), "-lm"])
    return out


def build_reference() -> Path | None:
    """Compile the reference jenga_core sources + shim; None when unavailable."""
    if not REF_SRC.exists():
        return None
    jd = _json_dir()
    if jd is None:
        return None
    OUT.mkdir(exist_ok=True)
    out = OUT / "libjenga_ref.so"
    srcs = sorted(str(p) for p in REF_SRC.glob("*.cpp")) + [str(HERE / "ref_shim.cpp")]
    if _stale(out, srcs):
        objdir = OUT / "obj"
        objdir.mkdir(exist_ok=True)
        objs = []
        procs = []
        for s in srcs:
            o = objdir / (Path(s).stem + ".o")
            objs.append(str(o))
            if _stale(o, [s]):
                procs.append(subprocess.Popen(
                    ["g++", "-std=c++20", "-O2", "-fPIC", "-fvisibility=hidden", "-w", "-I", str(REF_INC), "-I", jd,
                     "-c", s, "-o", str(o)], stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
        for p in procs:
            so, se = p.communicate()
            if p.returncode != 0:
                raise RuntimeError(f"reference build failed: {p.args}\n{so}\n{se}")
        _run(["g++", "-shared", "-o", str(out), *objs])
    return out


def build_bridge() -> Path | None:
    """The INTEGRATION.md §1 bridge, compiled as a reference maintainer would:
    against the reference headers, the reference objects (minus our shim) and
    libjenga_b200.so (+ the CUDA runtime for its device buffers)."""
    if build_reference() is None:
        return None
    root = HERE.parent
    lib = root / "paper_2503_18292_b200" / "libjenga_b200.so"
    cuda = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
    if not lib.exists() or not (cuda / "include" / "cuda_runtime_api.h").exists():
        return None
    out = OUT / "libjenga_bridge_test.so"
    src = root / "tests" / "bridge" / "bridge_harness.cpp"
    hdr = root / "integration" / "jenga_gpu_bridge.hpp"
    objs = sorted(str(o) for o in (OUT / "obj").glob("*.o") if o.stem != "ref_shim")
    if _stale(out, [src, hdr, root / "include" / "jenga_gpu.h", lib, *objs]):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-w", "-I", str(REF_INC), "-I", _json_dir(),
              "-I", str(root / "integration"), "-I", str(root / "include"), "-I", str(cuda / "include"), str(src),
              *objs, "-o", str(out), "-L", str(lib.parent), "-l:libjenga_b200.so", "-L", str(cuda / "lib64"),
              "-lcudart", "-Wl,-rpath,$ORIGIN/../../paper_2503_18292_b200", f"-Wl,-rpath,{cuda / 'lib64'}"])
    return out


def build() -> None:
    build_c_oracle()
    build_reference()
    build_bridge()


if __name__ == "__main__":
    build()
    print("oracle built:", sorted(p.name for p in OUT.glob("*.so")))
