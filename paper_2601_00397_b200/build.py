"""Builds libtwb200.so in-tree with nvcc for sm_100a (no torch JIT cache involved)."""

from __future__ import annotations

import glob
import hashlib
import json
import os
import shutil
import subprocess
import time

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib", "libtwb200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",  # exact fp64: no FMA contraction anywhere
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(HERE, "..", "include", "twb200.h")
    ]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_native(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    tmp = OUT + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, "-o", tmp, *sources()]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    if verbose:
        print(proc.stderr)
    os.replace(tmp, OUT)
    with open(os.path.join(HERE, "lib", "ptxas.log"), "w") as fh:
        fh.write(proc.stderr)
    with open(OUT, "rb") as fh:
        digest = hashlib.sha256(fh.read()).hexdigest()
    info = {"library": os.path.relpath(OUT, os.path.dirname(HERE)), "sha256": digest,
            "built_at_unix": int(time.time()), "nvcc": [os.path.basename(cmd[0]), *NVCC_FLAGS],
            "sources": [os.path.relpath(x, os.path.dirname(HERE)) for x in sources()]}
    with open(os.path.join(HERE, "lib", "build_info.json"), "w") as fh:
        json.dump(info, fh, indent=1)
    return OUT


def build_oracle() -> str:
    """The CPU checker (oracle/), test infrastructure only."""
    root = os.path.dirname(HERE)
    proc = subprocess.run(["make", "-C", os.path.join(root, "oracle")], capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{proc.stdout}\n{proc.stderr}")
    return os.path.join(root, "oracle", "build", "libtwb_oracle.so")


if __name__ == "__main__":
    print(build_native(force=True, verbose=True))
