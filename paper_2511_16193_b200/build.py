"""Build the in-tree CUDA extension ``libspecrollout_b200.so`` for sm_100a.

``python -m paper_2511_16193_b200.build`` compiles every ``csrc/*.cu`` with
nvcc (``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3``) in parallel
and links one shared library next to this file, so it travels to the GPU box
with the repo snapshot.  Objects are cached under ``build/`` by source hash.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libspecrollout_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v,-warn-spills"]
# measurement builds only (e.g. -DSR_ATTN_PROBE=1, attention.cu)
FLAGS += os.environ.get("SR_EXTRA_NVCC_FLAGS", "").split()


def _digest(src: Path) -> str:
    h = hashlib.sha1()
    h.update(" ".join(ARCH + FLAGS).encode())
    for f in sorted(CSRC.glob("*.cuh")) + [src] + sorted(INCLUDE.glob("*.h")):
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


def _compile(src: Path) -> Path:
    obj = OBJ / f"{src.stem}-{_digest(src)}.o"
    if obj.exists():
        return obj
    log = OBJ / f"{src.stem}.ptxas.log"
    cmd = [NVCC, *ARCH, *FLAGS, "-I", str(INCLUDE), "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr[-6000:]}")
    return obj


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        objs = list(pool.map(_compile, sources))
    stamp = hashlib.sha1("".join(o.name for o in objs).encode()).hexdigest()[:16]
    marker = OBJ / "link.stamp"
    if LIB.exists() and marker.exists() and marker.read_text() == stamp:
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    os.replace(tmp, LIB)
    marker.write_text(stamp)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
