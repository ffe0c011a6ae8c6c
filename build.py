"""Build the sm_100a decision-plane library in-tree.

    python build.py            # -> paper_2512_00719_b200/_lib/libdecplane_b200.so

nvcc cross-compiles here (no GPU needed); the .so travels to the GPU box with
the repo snapshot.  Also builds the oracle's nothing (pure numpy) — kept as a
single entry point for __graft_entry__.build().
"""

from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_2512_00719_b200")
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libdecplane_b200.so")
SOURCES = ["capi.cu", "sample_topk.cu", "sample_warp.cu", "sample_general.cu", "summary.cu", "aux_kernels.cu", "collective.cu", "sample_persist.cu", "sample_hot.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "decplane_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile + link the library.  `defines` / `out` build an A-B variant
    (e.g. defines=["DP_MW_BLOCKS=6"], out=".../_lib/variants/x.so")."""
    lib = out or LIB
    if not force and not defines and out is None and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(ROOT, "build", "obj" if not defines else "obj_" + "_".join(defines).replace("=", ""))
    os.makedirs(objdir, exist_ok=True)
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
    if verbose:
        common += ["-Xptxas", "-v"]
    common += ["-D" + d for d in defines]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        r = subprocess.run(common + ["-c", os.path.join(CSRC, src), "-o", obj], capture_output=True, text=True)
        return src, obj, r

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for src, _, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed compiling {src}")
        if verbose:
            sys.stderr.write(r.stderr)
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    link = [NVCC, *ARCH, "--shared", "-o", lib + ".tmp"] + [obj for _, obj, _ in results] + ["-ldl"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libdecplane_b200.so")
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, out=outs[0] if outs else None))
