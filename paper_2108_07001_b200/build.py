"""Build libkkb200.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2108_07001_b200.build [--force]

The shared library lands at paper_2108_07001_b200/_lib/libkkb200.so (git
ignored, but shipped to the GPU box with the repo snapshot).  nvcc
cross-compiles here without a GPU.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libkkb200.so")
SOURCES = ["kk_capi.cu", "kk_kk.cu", "kk_static.cu", "kk_ddlms.cu", "kk_metrics.cu", "kk_fft.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def _digest() -> str:
    h = hashlib.sha256()
    # every file under csrc/ (sources and all headers they may include)
    for f in sorted(os.listdir(CSRC)):
        if not f.endswith((".cu", ".cuh", ".h", ".hpp")):
            continue
        h.update(f.encode())
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(fh.read())
    with open(os.path.join(REPO, "include", "kkb200.h"), "rb") as fh:
        h.update(fh.read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, defines=(), name: str = "") -> str:
    """Build the library; `defines`/`name` make a tuning variant at
    _lib/variants/libkkb200_<name>.so (load it with KKB200_LIB=...)."""
    out_dir = os.path.join(OUT_DIR, "variants", name) if name else OUT_DIR
    lib_path = os.path.join(out_dir, f"libkkb200_{name}.so") if name else LIB
    os.makedirs(out_dir, exist_ok=True)
    stamp = os.path.join(out_dir, "build.sha256")
    flags = NVCC_FLAGS + [f"-D{d}" for d in defines]
    dig = _digest() + " ".join(flags)
    if not force and os.path.exists(lib_path) and os.path.exists(stamp):
        with open(stamp) as f:
            if f.read().strip() == dig:
                return lib_path
    nvcc = _nvcc()
    objs = []
    logs = []
    for src in SOURCES:
        obj = os.path.join(out_dir, src.replace(".cu", ".o"))
        cmd = [nvcc, *flags, "-I", os.path.join(REPO, "include"), "-dc" if False else "-c",
               os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}")
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        objs.append(obj)
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", lib_path]
    r = subprocess.run(cmd, capture_output=True, text=True)
    logs.append(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}")
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    with open(os.path.join(out_dir, "build.log"), "w") as f:
        f.write("\n".join(logs))
    with open(stamp, "w") as f:
        f.write(dig)
    if verbose:
        print("\n".join(logs))
    return lib_path


if __name__ == "__main__":
    # python -m paper_2108_07001_b200.build [--force] [-v] [--variant NAME -DX=1 ...]
    av = sys.argv[1:]
    nm = av[av.index("--variant") + 1] if "--variant" in av else ""
    print(build(force="--force" in av, verbose="-v" in av, name=nm,
                defines=[a[2:] for a in av if a.startswith("-D")]))
