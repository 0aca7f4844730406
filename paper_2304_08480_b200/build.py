"""In-tree build of the sm_100a extension: ``python -m paper_2304_08480_b200.build``.

Plain nvcc (no torch.utils.cpp_extension: the library has a pure C ABI and
links no torch or NCCL symbols).  Output: paper_2304_08480_b200/_disco_b200.so.
"""

import os
import shutil
import subprocess
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
SOURCES = [os.path.join(_HERE, "csrc", "disco_b200.cu")]
DEPS = SOURCES + [os.path.join(_HERE, "csrc", f) for f in
                  ("ptx.cuh", "common.cuh", "logits.cuh", "gemm.cuh", "tails.cuh", "host.cuh")] + \
    [os.path.join(ROOT, "include", "disco_b200.h")]
OUT = os.path.join(_HERE, "_disco_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """Build the library (``defines``: extra -D switches for kernel-variant builds that
    tools/ab_kernels.py --so-b compares against the default build)."""
    if out == OUT and not defines and not force and up_to_date():
        return OUT
    cmd = [nvcc_path(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
           "-o", out + ".tmp", *SOURCES]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--out", default=OUT)
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=True, out=a.out, defines=a.defines))
