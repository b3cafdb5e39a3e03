"""Build libchess_b200.so (sm_100a) in-tree with nvcc.

The shared library is the drop-in C-ABI (include/chess_b200.h).  It is built
in-tree so it travels to the GPU box with the repo snapshot; `*.so` is
git-ignored.  Object files are rebuilt only when a source or header changed.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
BUILD = PKG_DIR / "_build"
LIB = PKG_DIR / "libchess_b200.so"
TRACE_LIB = PKG_DIR / "libchess_b200_trace.so"
SOURCES = ["capi.cu", "k_index.cu", "k_select.cu", "k_attn.cu", "k_entropy.cu"]
HEADERS = [CSRC / "common.cuh", CSRC / "tc.cuh", CSRC / "k_select_tc.cuh", CSRC / "k_attn_tc.cuh", REPO / "include" / "chess_b200.h"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler",
    "-fPIC",
    "-Xptxas",
    "-v",
    f"-I{REPO / 'include'}",
]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, trace: bool = False, variant: str = "",
          defines=()) -> Path:
    """Product library; trace=True builds the debug-timeline variant
    (-DCHESS_TRACE=1) as libchess_b200_trace.so for the micro-benchmarks
    (select it with CHESS_B200_LIB).  variant/defines build an experiment
    library libchess_b200_<variant>.so with extra -D flags."""
    bdir = BUILD / "trace" if trace else BUILD
    lib = TRACE_LIB if trace else LIB
    extra = ["-DCHESS_TRACE=1"] if trace else []
    if variant:
        bdir = BUILD / variant
        lib = PKG_DIR / f"libchess_b200_{variant}.so"
        extra += [f"-D{x}" for x in defines]
    bdir.mkdir(parents=True, exist_ok=True)
    objs, todo = [], []
    for src in SOURCES:
        s = CSRC / src
        o = bdir / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s, *HEADERS]):
            todo.append((src, s, o))

    def compile_one(job):
        src, s, o = job
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", str(s), "-o", str(o)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        (bdir / (s.stem + ".ptxas.log")).write_text(res.stdout + res.stderr)
        return src, res

    # the translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        for src, res in ex.map(compile_one, todo):
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                print(f"compiled {src}")
    if force or _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc link failed")
        if verbose:
            print(f"linked {lib}")
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    defs = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--define=")]
    build(verbose=True, force="--force" in sys.argv, trace="--trace" in sys.argv, variant=var, defines=defs)
