"""In-tree build of the native libraries.

* ``paper_2011_01805_b200/_lib/libtiletensor_b200.so`` -- the product: C-ABI +
  sm_100a kernels (nvcc, ``-gencode arch=compute_100a,code=sm_100a``).
* ``paper_2011_01805_b200/_lib/tt_host_tests`` -- C++ tests of the host mirror
  headers (run by ``tests/test_cpp_host.py`` on a GPU).
* ``oracle/_build/libttoracle.so`` -- the CPU restatement (test checker only).
* ``oracle/_ref/libttref.so`` -- the reference itself, compiled from its headers
  where they lie (``/root/reference`` in this container) or from the git-ignored
  copy ``baseline/_ref/include`` that travels to the GPU box.

Sources are compiled only when newer than their outputs.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
OBJ_DIR = LIB_DIR / "obj"
LIB = LIB_DIR / "libtiletensor_b200.so"
HOST_TESTS = LIB_DIR / "tt_host_tests"
CPP_BENCH = LIB_DIR / "tt_bench_cpp"
PYFAST = PKG / ("_ttfast" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "_build" / "libttoracle.so"
REF_LIB = ORACLE_DIR / "_ref" / "libttref.so"
REF_SRC = Path("/root/reference/proj/include")
# the reference headers travel to the GPU box as a git-ignored copy,
# so `make ref` also works where /root/reference does not exist
REF_COPY = ROOT / "baseline" / "_ref" / "include"
REF_INC = Path(os.environ.get("TT_REFERENCE_INCLUDE",
                              str(REF_SRC if (REF_SRC / "tiletensor").is_dir() else REF_COPY)))

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler",
           "-ffp-contract=off", "--fmad=false", "-I", str(ROOT / "include"), "-I", str(CSRC)]
SOURCES = ["tt_shape.cpp", "tt_schedule.cpp", "tt_capi.cpp", "tt_kernels.cu", "tt_tma_pack.cu"]
HEADERS = [CSRC / "tt_internal.hpp", CSRC / "tt_launch.hpp", CSRC / "tt_pdl.cuh", ROOT / "include" / "tiletensor_b200.h",
           *sorted((CSRC / "kernels").glob("*.cuh"))]


def _run(cmd: list[str], cwd: Path | None = None) -> None:
    proc = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd)}")


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.exists() and d.stat().st_mtime > t for d in deps)


def build_product(verbose: bool = False) -> Path:
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = OBJ_DIR / (src + ".o")
        objs.append(o)
        if _stale(o, [s, *HEADERS]):
            if verbose:
                print(f"[build] nvcc {src}")
            _run([NVCC, *ARCH, *NVFLAGS, "-Xptxas", "-v" if verbose else "-O3", "-c", str(s),
                  "-o", str(o)])
    if _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"])
    build_pyfast(verbose)
    return LIB


def build_pyfast(verbose: bool = False) -> Path:
    """The CPython fast-call module over the C-ABI (csrc/tt_pyfast.c)."""
    src = CSRC / "tt_pyfast.c"
    if _stale(PYFAST, [src, LIB, ROOT / "include" / "tiletensor_b200.h"]):
        if verbose:
            print("[build] gcc tt_pyfast.c")
        _run(["gcc", "-O2", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"], "-I",
              str(ROOT / "include"), str(src), "-o", str(PYFAST), "-L", str(LIB_DIR),
              "-ltiletensor_b200", "-Wl,-rpath,$ORIGIN/_lib"])
    return PYFAST


def build_host_tests(verbose: bool = False) -> Path:
    src = PKG / "tests_cpp" / "host_tests.cpp"
    hdrs = sorted((PKG / "include" / "tiletensor_b200").glob("*.hpp"))
    if src.exists() and _stale(HOST_TESTS, [src, LIB, *hdrs]):
        if verbose:
            print("[build] g++ host_tests.cpp")
        _run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", str(ROOT / "include"),
              "-I", str(PKG / "include"), str(src), "-o", str(HOST_TESTS), "-L", str(LIB_DIR),
              "-ltiletensor_b200", "-Wl,-rpath,$ORIGIN", "-pthread"])
    return HOST_TESTS


def _copy_reference_headers() -> None:
    """Mirror the reference's headers into baseline/_ref/include (git-ignored,
    shipped with the gpurun snapshot); never written back to the reference."""
    import shutil
    src = REF_SRC / "tiletensor"
    if not src.is_dir():
        return
    dst = REF_COPY / "tiletensor"
    dst.mkdir(parents=True, exist_ok=True)
    for f in src.glob("*.hpp"):
        out = dst / f.name
        if not out.exists() or out.read_bytes() != f.read_bytes():
            shutil.copyfile(f, out)


def build_cpp_bench(verbose: bool = False) -> Path:
    """The C++ performance leg (tests_cpp/bench_cpp.cpp) over the drop-in headers."""
    src = PKG / "tests_cpp" / "bench_cpp.cpp"
    hdrs = sorted((PKG / "include" / "tiletensor_b200").glob("*.hpp"))
    if src.exists() and _stale(CPP_BENCH, [src, LIB, *hdrs]):
        if verbose:
            print("[build] g++ bench_cpp.cpp")
        _run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", str(ROOT / "include"),
              "-I", str(PKG / "include"), "-I", "/usr/local/cuda/include", str(src), "-o",
              str(CPP_BENCH), "-L", str(LIB_DIR), "-ltiletensor_b200", "-L", "/usr/local/cuda/lib64",
              "-lcudart", "-Wl,-rpath,$ORIGIN", "-Wl,-rpath,/usr/local/cuda/lib64", "-pthread"])
    return CPP_BENCH


def build_oracle(verbose: bool = False) -> None:
    _copy_reference_headers()
    targets = ["oracle"]
    if (REF_INC / "tiletensor").is_dir():
        targets.append("ref")
    _run(["make", "-s", "-C", str(ORACLE_DIR), *targets, f"REF_INC={REF_INC}"])


def build_all(verbose: bool = False) -> None:
    build_product(verbose)
    build_oracle(verbose)
    build_host_tests(verbose)
    build_cpp_bench(verbose)


if __name__ == "__main__":
    build_all(verbose="-v" in sys.argv)
    print(f"built {LIB}")
