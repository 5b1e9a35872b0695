"""Compile the CUDA engine (csrc/*.cu) into an in-tree shared library.

    python -m paper_2101_09441_b200.build        # or __graft_entry__.build()

Output: paper_2101_09441_b200/_lib/libdbl_b200.so, built for sm_100a only
(`-gencode arch=compute_100a,code=sm_100a`).  nvcc cross-compiles without a
GPU, so this runs in the authoring container; the .so travels to the GPU
box with the repository snapshot.
"""
from __future__ import annotations

import concurrent.futures
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUTDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUTDIR, "libdbl_b200.so")
SOURCES = ["graph.cu", "select.cu", "fixpoint.cu", "query.cu", "verify.cu", "insert_one.cu", "abi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-I" + os.path.join(ROOT, "include")]
# query.cu tail-launches the BFS hard path from the device (CUDA dynamic
# parallelism): relocatable device code, device-linked against cudadevrt.
RDC = {"query.cu"}
LINK = ["-rdc=true", "-lcudadevrt", "-lcudart"]


def _flags(src: str) -> list:
    return FLAGS + (["-rdc=true"] if src in RDC else [])


def _inputs():
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "dbl_b200.h"))
    return deps


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _inputs())


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(OUTDIR, os.path.basename(src).replace(".cu", ".o"))
    cmd = [NVCC, *ARCH, *_flags(src), "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build_variant(name: str, defines: list[str]) -> str:
    """Experimental build with extra -D flags into _lib/variant_<name>.so."""
    os.makedirs(OUTDIR, exist_ok=True)
    out = os.path.join(OUTDIR, f"variant_{name}.so")
    objs = []
    for src in SOURCES:
        obj = os.path.join(OUTDIR, f"{name}_{src.replace('.cu', '.o')}")
        subprocess.check_call([NVCC, *ARCH, *_flags(src), *[f"-D{d}" for d in defines], "-c",
                               os.path.join(CSRC, src), "-o", obj], stderr=subprocess.DEVNULL)
        objs.append(obj)
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", out, *objs, *LINK])
    for o in objs:
        os.remove(o)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OUTDIR, exist_ok=True)
    with concurrent.futures.ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(_compile, SOURCES))
    objs = [o for o, _ in results]
    with open(os.path.join(OUTDIR, "ptxas.log"), "w") as f:
        for (_, log), src in zip(results, SOURCES):
            f.write(f"=== {src}\n{log}\n")
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, *LINK]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
