"""Build the in-tree C-ABI shared library ``libtneat.so`` for sm_100a.

Every ``csrc/*.cu`` is compiled by nvcc for ``-gencode
arch=compute_100a,code=sm_100a`` (B200 only -- no other architecture, no PTX
fallback) with ``-lineinfo`` so ncu's source page maps to the code, then linked
into one shared library next to this file.  No torch headers are involved: the
library exports plain ``extern "C"`` functions (include/tneat.h) and the host
package calls them through ctypes with device pointers and a CUDA stream.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libtneat.so")
BUILD = os.path.join(os.path.dirname(HERE), "build", "tneat")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# evolve.cu reproduces numpy's float64 rounding: no FMA contraction there
PER_FILE = {"evolve.cu": ["-fmad=false"]}
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libtneat.so")


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def _flags_changed(extra: list[str]) -> bool:
    """The objects record the flags they were built with (a stamp file): a
    build with different TNEAT_NVCC_EXTRA knobs (diagnostic -D switches compute
    wrong outputs by design) never leaves its objects behind for a plain build."""
    stamp = os.path.join(BUILD, "flags.stamp")
    key = " ".join(ARCH + FLAGS + extra + [f"{k}:{' '.join(v)}" for k, v in sorted(PER_FILE.items())])
    old = open(stamp).read() if os.path.exists(stamp) else None
    if old != key:
        with open(stamp, "w") as f:
            f.write(key)
        return old is not None or any(f.endswith(".o") for f in os.listdir(BUILD))
    return False


def build(verbose: bool = False, force: bool = False) -> str:
    nvcc = _nvcc()
    os.makedirs(BUILD, exist_ok=True)
    extra = os.environ.get("TNEAT_NVCC_EXTRA", "").split()  # tuning experiments (-D knobs) only
    force = _flags_changed(extra) or force
    srcs = sources()
    objs = [os.path.join(BUILD, os.path.basename(s)[:-3] + ".o") for s in srcs]

    def compile_one(pair):
        src, obj = pair
        if not force and not _stale(obj, src):
            return obj, ""
        cmd = [nvcc, *ARCH, *FLAGS, *PER_FILE.get(os.path.basename(src), []), *extra, "-I", CSRC, "-c", src,
               "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{res.stdout}\n{res.stderr}")
        return obj, res.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        logs = list(ex.map(compile_one, zip(srcs, objs)))
    if verbose:
        for obj, log in logs:
            if log:
                print(f"== {os.path.basename(obj)}\n{log}", file=sys.stderr)
    relink = force or not os.path.exists(OUT) or any(
        os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs)
    if relink:
        cmd = [nvcc, *ARCH, "-shared", "-o", OUT, *objs]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
