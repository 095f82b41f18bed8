"""Build libpilotann.so in-tree with nvcc for sm_100a only (no JIT, no torch
extension machinery): every .cu/.cpp under csrc/ is compiled in parallel with
`-gencode arch=compute_100a,code=sm_100a -lineinfo` and linked into one shared
library next to this file."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import shlex
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libpilotann.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3,-mavx2,-mfma,-pthread",
          f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps_mtime():
    files = _sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "pilotann.h"), __file__]
    return max(os.path.getmtime(f) for f in files)


def _include_closure(path, seen=None):
    """Local headers `path` includes, recursively (#include "x" resolved in csrc/
    and include/)."""
    import re
    seen = set() if seen is None else seen
    try:
        text = open(path).read()
    except OSError:
        return seen
    for name in re.findall(r'^\s*#\s*include\s+"([^"]+)"', text, re.M):
        for d in (CSRC, os.path.join(ROOT, "include")):
            h = os.path.join(d, name)
            if os.path.exists(h) and h not in seen:
                seen.add(h)
                _include_closure(h, seen)
                break
    return seen


def _deps_mtime_of(src):
    return max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in _include_closure(src)])


def _compile(src, extra, force=False):
    """Compile one source unless its object is newer than it and every local
    header it includes, and was built with the same extra flags (incremental
    rebuilds; `--force` after changing COMMON)."""
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    stamp = obj + ".flags"
    flags = " ".join(extra)
    if not force and os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == flags \
            and os.path.getmtime(obj) >= _deps_mtime_of(src):
        return obj, ""
    cmd = [NVCC] + GENCODE + COMMON + extra + ["-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if os.environ.get("PA_PTXAS_V") else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(stamp, "w") as f:
        f.write(flags)
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    # the kernels' tuning constants are fixed in the sources; PA_NVCC_EXTRA
    # (-D overrides of those constants) exists for A/B builds in a scratch copy only
    # (scripts/ab_variant.sh), never for the shipped library
    extra = shlex.split(os.environ.get("PA_NVCC_EXTRA", ""))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        outs = list(ex.map(lambda s: _compile(s, extra, force), _sources()))
    objs = [o for o, _ in outs]
    if verbose:
        for _, err in outs:
            if err.strip():
                print(err, file=sys.stderr)
    tmp = LIB + ".tmp"
    cmd = [NVCC] + GENCODE + ["-shared", "-o", tmp] + objs + ["-lpthread"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
