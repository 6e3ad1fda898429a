"""In-tree build of the sm_100a backend (libreseq_cuda.so) and of the test oracle.

`nvcc` cross-compiles without a GPU, so this runs on the CPU build box; the resulting
shared objects are git-ignored but travel to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOST = PKG / "host"
LIB = PKG / "libreseq_cuda.so"
OBJ = PKG / "build"

CUDA_SOURCES = ["capi.cu", "radix.cu", "scan.cu", "sa.cu", "index.cu"]
HOST_SOURCES = ["greedy.cpp", "synth.cpp"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-Wall",
    "--expt-relaxed-constexpr",
    "-diag-suppress", "177",
]


def _nvcc() -> str:
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        raise RuntimeError("nvcc not found: cannot build the sm_100a backend")
    return nvcc


def _stamp(paths) -> str:
    h = hashlib.sha256()
    for p in sorted(paths):
        h.update(str(p).encode())
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build_library(force: bool = False, verbose: bool = False) -> Path:
    srcs = [CSRC / s for s in CUDA_SOURCES] + [HOST / s for s in HOST_SOURCES]
    deps = srcs + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "reseq_cuda.h"]
    stamp_file = OBJ / "stamp"
    stamp = _stamp(deps)
    if not force and LIB.exists() and stamp_file.exists() and stamp_file.read_text() == stamp:
        return LIB
    OBJ.mkdir(exist_ok=True)
    nvcc = _nvcc()
    inc = ["-I", str(ROOT / "include"), "-I", str(CSRC)]
    objs = []
    procs = []
    for s in srcs:
        o = OBJ / (s.stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *inc, "-c", str(s), "-o", str(o)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(o)
    for s, p in procs:
        out, _ = p.communicate()
        if verbose and out:
            print(out)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s.name}:\n{out}")
    link = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(LIB),
            *map(str, objs)]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}")
    stamp_file.write_text(stamp)
    return LIB


TOOL = PKG / "reseq_b200"


def build_tools() -> Path:
    """tools/reseq_b200.cpp -> paper_1404_3456_b200/reseq_b200 (build-sa / bench with the reference's
    file formats), linked against the in-tree library."""
    src = ROOT / "tools" / "reseq_b200.cpp"
    deps = [src, ROOT / "include" / "reseq_cuda.h", ROOT / "include" / "reseq_b200" / "reseq_cuda.hpp"]
    if TOOL.exists() and all(TOOL.stat().st_mtime >= d.stat().st_mtime for d in deps + [LIB]):
        return TOOL
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", str(ROOT / "include"), str(src), str(LIB),
           "-Wl,-rpath,$ORIGIN", "-o", str(TOOL)]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"tool build failed:\n{r.stdout}")
    return TOOL


def build_oracle() -> None:
    """Compiles oracle/liboracle.so and, when /root/reference is present, oracle/_ref."""
    r = subprocess.run(["make", "-C", str(ROOT / "oracle"), "all"], stdout=subprocess.PIPE,
                       stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}")
    # the reference's own classes over libreseq_cuda.so (oracle/_ref/dropin_test; needs /root/reference)
    r = subprocess.run([sys.executable, str(ROOT / "oracle" / "make_dropin.py")], stdout=subprocess.PIPE,
                       stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"drop-in test build failed:\n{r.stdout}")


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose="-v" in sys.argv)
    build_tools()
    build_oracle()
    print(LIB)
