"""Build libhwb200.so in-tree for sm_100a (no JIT cache: the .so travels with
the repo snapshot to the GPU box), plus libhwb200_margin.so: the same sources
with -DHWB_FFT_MARGIN=1, whose FFT ladders record the largest rounding residual
|y - rint(y)| (test instrumentation only; never loaded by the product path)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libhwb200.so")
LIB_MARGIN = os.path.join(HERE, "libhwb200_margin.so")
SOURCES = [os.path.join(HERE, "csrc", "hwb_kernels.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", "hwb_device.cuh"), os.path.join(HERE, "csrc", "hwb_tc.cuh"),
                  os.path.join(HERE, "csrc", "hwb_fft.cuh"), os.path.join(REPO, "include", "hwb.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    # (not -split-compile: measured to cost registers / add stack frames in the ladder
    # kernels -- blind_rotate_fft_tm_kernel 234 -> 255 registers + 160 B stack)
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in DEPS)


def _cmd(out: str, extra=(), verbose=False):
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", out + ".tmp", *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    return cmd


def build(force: bool = False, verbose: bool = False, margin: bool = True) -> str:
    jobs = []
    if force or stale(LIB):
        jobs.append((LIB, subprocess.Popen(_cmd(LIB, (), verbose))))
    if margin and (force or stale(LIB_MARGIN)):
        jobs.append((LIB_MARGIN, subprocess.Popen(_cmd(LIB_MARGIN, ("-DHWB_FFT_MARGIN=1",), verbose))))
    for out, proc in jobs:
        if proc.wait() != 0:
            raise subprocess.CalledProcessError(proc.returncode, f"nvcc -> {out}")
        os.replace(out + ".tmp", out)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, margin="--no-margin" not in sys.argv))
