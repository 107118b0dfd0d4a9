"""Builds libterralio_gpu.so (sm_100a) in-tree, and the CPU oracle.

Usage: python -m paper_2509_26222_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libterralio_gpu.so"
OBJ_DIR = ROOT / "build" / "obj"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", *ARCH,
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
    "--expt-relaxed-constexpr",
    "-I", str(ROOT / "include"),
]

SOURCES = ["model.cu", "grid.cu", "eval.cu", "select.cu", "dense.cu", "update.cu", "assemble.cu", "prof.cu",
           "scan.cu", "consumers.cu", "match.cu", "abi.cu"]
DIAG_LIB = LIB_DIR / "libterralio_diag.so"
# match.cu restates the matcher's scalar geometry (centroids, scatter, 3x3
# eigen sweeps, residuals) with the reference's unfused rounding
EXTRA_FLAGS = {"match.cu": ["-fmad=false"]}


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("command failed: " + " ".join(cmd))
    if r.stderr.strip():
        sys.stderr.write(r.stderr)


def build_gpu(force: bool = False, verbose: bool = False) -> Path:
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "terralio_gpu.h"]
    jobs = []
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = OBJ_DIR / (src + ".o")
        objs.append(o)
        if force or _stale(o, [s, *headers]):
            cmd = [NVCC, *NVCC_FLAGS, *EXTRA_FLAGS.get(src, []), "-c", str(s), "-o", str(o)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)
    if jobs:
        with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            list(ex.map(_run, jobs))
    if force or jobs or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart_static",
              "-lrt", "-lpthread", "-ldl"])
    # diagnostics (not the product ABI): its own library on top of the product
    dsrc = CSRC / "diag" / "diag.cu"
    dobj = OBJ_DIR / "diag.cu.o"
    if force or _stale(dobj, [dsrc, *headers, ROOT / "include" / "terralio_diag.h"]):
        _run([NVCC, *NVCC_FLAGS, "-c", str(dsrc), "-o", str(dobj)])
    if force or _stale(DIAG_LIB, [dobj, LIB]):
        _run([NVCC, *ARCH, "-shared", "-o", str(DIAG_LIB), str(dobj), "-L", str(LIB_DIR),
              "-lterralio_gpu", "-Xlinker", f"-rpath,{LIB_DIR}", "-lcudart_static", "-lrt",
              "-lpthread", "-ldl"])
    return LIB


REFERENCE = Path("/root/reference/proj")


def build_oracle(force: bool = False) -> Path:
    """The CPU checkers (test infrastructure): the plain-C++ restatement, and,
    where /root/reference exists (the build container; the GPU box only gets
    the prebuilt files), the reference itself compiled into oracle/_ref."""
    odir = ROOT / "oracle"
    if force:
        _run(["make", "-C", str(odir), "clean", "clean-ref"])
    _run(["make", "-C", str(odir)])
    if REFERENCE.exists():
        _run(["make", "-C", str(odir), f"-j{os.cpu_count() or 4}", "ref"])
    return odir / "_build" / "liboracle.so"


DROPIN_TESTS = ["test_kernel", "test_center_select", "test_terrain_model", "test_kinematics",
                "test_matcher"]
DROPIN_OUT = ROOT / "tests" / "cpp" / "_build"


def build_dropin_tests(force: bool = False) -> Path | None:
    """The reference's own unit-test files, compiled in place from
    /root/reference against include/terralio_dropin (the Eigen-typed drop-in
    on the C-ABI; Eigen and doctest from oracle/'s minimal stand-ins) and
    linked with libterralio_gpu.so: tests/cpp/_build/ref_tests_dropin. Only
    where /root/reference exists; the binary travels to the GPU box."""
    if not REFERENCE.exists():
        return None
    DROPIN_OUT.mkdir(parents=True, exist_ok=True)
    exe = DROPIN_OUT / "ref_tests_dropin"
    srcs = [REFERENCE / "tests" / "unit" / f"{t}.cpp" for t in DROPIN_TESTS]
    support = ROOT / "tests" / "cpp" / "dropin" / "support.cpp"
    hdrs = list((ROOT / "include" / "terralio_dropin").rglob("*.hpp")) + [
        ROOT / "include" / "terralio_gpu.h"]
    if not force and not _stale(exe, [*srcs, support, *hdrs, LIB]):
        return exe
    cxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else "g++"
    inc = ["-I", str(ROOT / "include" / "terralio_dropin"), "-I", str(ROOT / "oracle" / "eigen_subset"),
           "-I", str(ROOT / "oracle" / "shims"), "-I", str(ROOT / "include"),
           "-I", str(REFERENCE / "core" / "include")]
    objs = []
    jobs = []
    for src in [*srcs, support]:
        obj = DROPIN_OUT / (src.stem + ".o")
        objs.append(obj)
        jobs.append([cxx, "-std=c++20", "-O2", "-w", *inc, "-c", str(src), "-o", str(obj)])
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        list(ex.map(_run, jobs))
    cuda = Path("/usr/local/cuda")
    _run([cxx, *map(str, objs), "-L", str(LIB_DIR), "-lterralio_gpu", f"-Wl,-rpath,{LIB_DIR}",
          "-L", str(cuda / "lib64"), "-lcudart", f"-Wl,-rpath,{cuda / 'lib64'}", "-lpthread",
          "-o", str(exe)])
    return exe


def main() -> None:
    force = "--force" in sys.argv
    print(build_oracle(force))
    print(build_gpu(force, verbose="-v" in sys.argv))
    print(build_dropin_tests(force))


if __name__ == "__main__":
    main()
