"""Build libdnls.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = [os.path.join(HERE, "csrc", "dnls.cu"), os.path.join(HERE, "csrc", "dnls_cluster.cu"),
       os.path.join(HERE, "csrc", "symbolic.cpp")]
DEPS = SRC + [os.path.join(HERE, "csrc", f) for f in ("phases.cuh", "bl.cuh", "lie.cuh", "symbolic.h")] + [
    os.path.join(os.path.dirname(HERE), "include", "dnls.h")]
OUT = os.path.join(HERE, "lib", "libdnls.so")
OUT_TRACE = os.path.join(HERE, "lib", "libdnls_trace.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC,-fvisibility=hidden,-O2", "-shared", "-cudart", "static"]


def up_to_date(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def build(force: bool = False, verbose: bool = False, trace: bool = False, variant: str = "",
          defines=()) -> str:
    """Compile libdnls.so (or, trace=True, the -DDNLS_TRACE debug variant libdnls_trace.so; or a
    development variant lib/libdnls_<variant>.so with extra -D defines, loaded with DNLS_LIB)."""
    out = OUT_TRACE if trace else OUT
    if variant:
        out = os.path.join(os.path.dirname(OUT), f"libdnls_{variant}.so")
    if not force and up_to_date(out):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    tmp = out + ".tmp"
    extra = (["-DDNLS_TRACE"] if trace else []) + [f"-D{d}" for d in defines] + (["-Xptxas", "-v"] if verbose else [])
    # the translation units compile in parallel (-c), then one nvcc link step
    tag = os.path.basename(out).replace(".so", "")
    objs = [os.path.join(os.path.dirname(out), f".{tag}.{os.path.basename(src)}.o") for src in SRC]
    cflags = [f for f in FLAGS if f not in ("-shared",)]
    procs = [subprocess.Popen([NVCC] + cflags + extra + ["-c", "-o", o, src], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for src, o in zip(SRC, objs)]
    errs = []
    for pr in procs:
        so, se = pr.communicate()
        if pr.returncode != 0:
            errs.append(so + se)
        elif verbose:
            sys.stderr.write(se)
    if errs:
        sys.stderr.write("".join(errs))
        raise RuntimeError("nvcc failed building libdnls.so")
    r = subprocess.run([NVCC] + FLAGS + ["-o", tmp] + objs, capture_output=True, text=True)
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libdnls.so")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
