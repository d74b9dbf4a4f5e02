"""Build libfllf.so in-tree with nvcc for sm_100a (no GPU needed to build).

    python -m paper_2206_04681_b200.build

The library is written to paper_2206_04681_b200/lib/libfllf.so (git-ignored,
but it travels to the GPU box with the repository snapshot).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libfllf.so")
SOURCES = ["fllf_host.cpp", "fllf_kernels.cu", "fllf_fused.cu", "fllf_color.cu", "fllf_naive.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def build(verbose: bool = False, extra: list[str] | None = None, out: str | None = None) -> str:
    """Compile every source to an object (in parallel), then link the shared
    library; static cudart, exported symbols = the C ABI only."""
    from concurrent.futures import ThreadPoolExecutor
    import tempfile
    os.makedirs(LIBDIR, exist_ok=True)
    lib = out or LIB
    common = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", "-I", INCLUDE, "-I", CSRC, "-DFLLF_BUILD", *(extra or [])]
    with tempfile.TemporaryDirectory(prefix="fllf_build_") as tmp:
        def compile_one(src: str) -> tuple[str, subprocess.CompletedProcess]:
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            cmd = [nvcc(), *common, "-Xptxas", "-v" if verbose else "-O3", "-c", os.path.join(CSRC, src), "-o", obj]
            return obj, subprocess.run(cmd, capture_output=True, text=True)
        with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
            results = list(ex.map(compile_one, SOURCES))
        for (obj, r), src in zip(results, SOURCES):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed compiling {src}")
            if verbose:
                sys.stderr.write(r.stderr)
        cmd = [nvcc(), *ARCH, "-shared", "-o", lib, *[o for o, _ in results]]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed linking libfllf.so")
    return lib


if __name__ == "__main__":
    # python -m paper_2206_04681_b200.build [-v] [--variant NAME -DMACRO=V ...]: variants go to
    # lib/variants/libfllf_NAME.so (select with FLLF_LIB=...) for compile-time A/B runs
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], [a for a in sys.argv[i + 2:] if a.startswith("-D")]
        os.makedirs(os.path.join(LIBDIR, "variants"), exist_ok=True)
        print(build(extra=defs, out=os.path.join(LIBDIR, "variants", f"libfllf_{name}.so")))
    else:
        print(build(verbose="-v" in sys.argv))
