"""Build libbubblespec.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbubblespec.so")
SOURCES = ["api.cu", "verify.cu", "index.cu", "state.cu", "synth.cu", "exchange.cu", "ngram.cu", "bubble.cu", "attn.cu", "lmhead.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2,-Wall", "-Xptxas", "-v",
]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "bubblespec.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Compile libbubblespec.so (or libbubblespec_<variant>.so with extra -D defines)."""
    lib = LIB if not variant else os.path.join(HERE, f"libbubblespec_{variant}.so")
    if not force and not _stale(lib):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-shared", "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES], "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    if "--trace" in sys.argv:
        print(build(force=True, variant="trace", defines=["BS_TRACE"]))
    elif "--timing" in sys.argv:
        print(build(force=True, variant="timing", defines=["BS_PHASE_TIMING"]))
    elif "--variant" in sys.argv:  # --variant NAME DEF [DEF ...]: experiment builds
        i = sys.argv.index("--variant")
        print(build(force=True, verbose="-v" in sys.argv, variant=sys.argv[i + 1],
                    defines=[d for d in sys.argv[i + 2:] if d != "-v"]))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
