"""Build libisvd.so (sm_100a) in-tree with nvcc.

``python -m paper_2605_24514_b200.build`` or ``__graft_entry__.build()``.
The shared library lands next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "isvd"
LIB = PKG / "libisvd.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         f"-I{ROOT / 'include'}", f"-I{CSRC}"] + os.environ.get("ISVD_NVCC_FLAGS", "").split()
# the core kernels tail-launch their fallback kernels from the device (CUDA
# dynamic parallelism): relocatable device code for those files only (it
# costs registers elsewhere, e.g. 40 -> 86 in the projection kernel) and a
# device link against cudadevrt
RDC = {"core_svd.cu", "arrow_svd.cu"}


def _sources():
    return sorted(CSRC.glob("*.cu"))


STAMP = PKG / "libisvd.so.sha256"


def _source_hash() -> str:
    """Digest of every input of the library (sources, header, flags, nvcc
    version): the library is rebuilt whenever it differs from the digest
    recorded next to it by the last build, whatever the file times say."""
    import hashlib

    h = hashlib.sha256()
    deps = sorted(CSRC.glob("*")) + [ROOT / "include" / "isvd.h", Path(__file__)]
    for p in deps:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(ARCH + FLAGS + sorted(RDC)).encode())
    try:
        h.update(subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout.encode())
    except OSError:
        pass
    return h.hexdigest()


def _needs_build() -> bool:
    if not LIB.exists() or not STAMP.exists():
        return True
    return STAMP.read_text().strip() != _source_hash()


def _compile(src: Path, verbose: bool) -> Path:
    obj = BUILD / (src.stem + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, *(["-rdc=true"] if src.name in RDC else []), "-c", str(src), "-o",
           str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    return obj


def build_lib(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _needs_build():
        return LIB
    BUILD.mkdir(parents=True, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), _sources()))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-rdc=true", "-shared", "-o", str(tmp), *map(str, objs), "-lcudadevrt",
           "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    STAMP.write_text(_source_hash() + "\n")
    return LIB


if __name__ == "__main__":
    build_lib(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
