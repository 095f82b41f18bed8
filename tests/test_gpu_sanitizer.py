"""compute-sanitizer over every kernel path (scripts/sanitize_run.py: tcgen05
projection + FES, pipelined traversal with bloom / exact / forced-spill visited
sets, binary16 rows, v1 traversal, SIMT fallbacks, stages 2-3 on the GPU) on C0:
no memory errors and no shared-memory hazards (racecheck found the missing
__syncwarp before the merge-first reordering was fixed).

The GPU pool this repo is tested on has closed compute-sanitizer (runs under it
left GPUs needing a reset), so these tests run only with PA_RUN_SANITIZER=1 on a
box that allows it; profiles/sanitizer/ keeps the round-1 logs (0 errors, 0
hazards).  On this pool the element-by-element parity tests against the oracle
over every kernel path are the check that remains."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if os.environ.get("PA_RUN_SANITIZER") != "1":
        pytest.skip("compute-sanitizer runs only with PA_RUN_SANITIZER=1 (closed on this GPU pool)")
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    import __graft_entry__ as g
    g.build_library()
    r = subprocess.run([cs, "--tool", tool, "--print-limit", "10", sys.executable,
                        os.path.join(ROOT, "scripts", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        pytest.skip(out.strip()[:200])
    assert "sanitize run done" in out, out[-3000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out, out[-3000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
