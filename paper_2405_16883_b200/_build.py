"""Build recipe for ``libstc.so`` (the CUDA kernels + C ABI, sm_100a only).

Compiled in-tree with plain ``nvcc`` so the shared object travels with the
repository snapshot to the GPU box; no JIT cache is involved.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libstc.so"
# checked build: device-side bounds / protocol checks (STC_CHECK) compiled in; for test runs
# only (tools/run_checked.sh loads it through STC_LIBRARY)
LIB_CHECKED = PKG / "libstc_checked.so"
SOURCES = ["abi_common.cu", "spmm.cu", "spmm_wide.cu", "mttkrp_prepared.cu", "attention.cu", "spgemm.cu",
           "construct.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    mtime = lib.stat().st_mtime
    deps = list(CSRC.glob("*")) + [PKG.parent / "include" / "stc.h"]
    return any(p.stat().st_mtime > mtime for p in deps)


def build(verbose: bool = False, force: bool = False, checked: bool = False) -> Path:
    """Compile every .cu to an object, link ``libstc.so`` (``libstc_checked.so`` with
    ``checked``: STC_CHECKED defined); returns its path."""
    lib = LIB_CHECKED if checked else LIB
    if not force and not needs_build(lib):
        return lib
    nvcc = _nvcc()
    build_dir = PKG / ("build_checked" if checked else "build")
    build_dir.mkdir(exist_ok=True)
    objs = [str(build_dir / (Path(src).stem + ".o")) for src in SOURCES]
    defs = ["-DSTC_CHECKED"] if checked else []
    cmds = [[nvcc, *ARCH, *FLAGS, *defs, "-I", str(PKG.parent / "include"), "-c", str(CSRC / src), "-o", obj]
            for src, obj in zip(SOURCES, objs)]
    # the translation units are independent: compile them concurrently
    procs = [subprocess.Popen(c, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for c in cmds]
    failed = None
    for src, p in zip(SOURCES, procs):
        out, err = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out + err)
            failed = failed or src
        elif verbose:
            sys.stderr.write(err)
    if failed:
        raise RuntimeError(f"nvcc failed on {failed}")
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True, checked="--checked" in sys.argv))
