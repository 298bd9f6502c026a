"""Build the in-tree CUDA library ``libfc_b200.so`` for sm_100a.

The library is the product: hand-written sm_100a kernels plus the C-ABI
(include/flexcomm_b200.h).  It is built in-tree so that the ``.so`` travels
with the repo snapshot to the GPU box.  NCCL comes from the torch-bundled
``nvidia-nccl`` wheel (2.28.9) so that a process that also imports torch
loads exactly one NCCL.
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
LIB = PKG / "libfc_b200.so"
SOURCES = [CSRC / "fc_kernels.cu", CSRC / "fc_ctx.cu", CSRC / "fc_costmodel.cpp", CSRC / "fc_moo.cpp"]
HEADERS = [CSRC / "fc_device.cuh", ROOT / "include" / "flexcomm_b200.h", ROOT / "include" / "fc_synth.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_root() -> Path:
    """Directory holding include/nccl.h and lib/libnccl.so.2 (torch's NCCL)."""
    env = os.environ.get("FC_NCCL_ROOT")
    if env:
        return Path(env)
    for p in sys.path:
        cand = Path(p) / "nvidia" / "nccl"
        if (cand / "include" / "nccl.h").exists():
            return cand
    return Path("/usr")


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return exe


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(s.stat().st_mtime > t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, out: Path | None = None,
          defines: tuple[str, ...] = ()) -> Path:
    if out is None and not force and not needs_build():
        return LIB
    out = out or LIB
    tmp = out.with_name(out.name + ".tmp")  # built aside, then renamed: readers never see a partial file
    nr = nccl_root()
    libdir = nr / "lib"
    cmd = [
        nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared",
        "-Xptxas", "-v" if verbose else "-O3",
        *[f"-D{d}" for d in defines],
        f"-I{ROOT / 'include'}", f"-I{nr / 'include'}",
        *[str(s) for s in SOURCES],
        f"-L{libdir}", "-l:libnccl.so.2", f"-Xlinker", f"-rpath={libdir}",
        "-o", str(tmp),
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    if verbose:
        sys.stderr.write(res.stdout + res.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
