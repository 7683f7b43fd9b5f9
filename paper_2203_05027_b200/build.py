"""Build libcfb200.so in-tree with nvcc for sm_100a (no JIT cache, travels with gpurun)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libcfb200.so")
SOURCES = ["cf_kernels.cu", "cf_setup.cu", "cf_api.cu", "cf_batch.cu", "cf_h2d.cu", "cf_gen.cu", "cf_nvls.cu", "cf_io.cpp"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",            # every fp64 op rounds like its numpy counterpart (parity)
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "cfb200.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """defines/out: experiment variants (e.g. CF_GATHER_WARPS=12) built beside the product library."""
    target = os.path.abspath(out) if out else OUT
    if not force and out is None and not defines and not needs_build():
        return OUT
    tmp = target + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(tmp, target)
    return target


# Compile-time variants tested beside the product library: the checked build (device
# bounds asserts + buffer guard canaries) that stands in for compute-sanitizer.
VARIANTS = {"checked": ["CF_CHECKED=1"]}
# experiments (python -m paper_2203_05027_b200.build --exp NAME=DEFINE,...): built on demand only


def variant_path(name: str) -> str:
    return os.path.join(HERE, f"libcfb200_{name}.so")


def build_variants(verbose: bool = False) -> list:
    return [build(force=True, verbose=verbose, out=variant_path(k), defines=v) for k, v in VARIANTS.items()]


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    if "--all" in sys.argv:
        print(build_variants(verbose=True))
