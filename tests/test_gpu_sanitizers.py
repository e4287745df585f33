"""compute-sanitizer over every kernel family (tools/sanitize_probe.py: the
streaming kernels in every mode, the finalize and decide, the AdamW and
reduce-scatter fusions, in-process peer ranks, the direct-mapped, tiered and
global caches): memcheck, racecheck and synccheck must report 0 errors.

Some GPU pools close compute-sanitizer (the binary on PATH is a wrapper that
refuses to run and says so); there the test is skipped -- the committed logs
under profiles/sanitizers/ are the last clean runs, and the parity suites'
bounds checks cover the kernels."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.fail("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    r = subprocess.run([_sanitizer(), "--tool", tool, "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_probe.py")], cwd=ROOT, capture_output=True, text=True,
                       timeout=900, env=dict(os.environ, AF_SANITIZE_TOOL=tool))
    out = r.stdout + r.stderr
    if r.returncode != 0 and "compute-sanitizer is closed" in out:
        pytest.skip("compute-sanitizer is closed on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert r.returncode == 0, out[-3000:]
    assert "sanitize probe done" in out
    assert "0 errors" in out, out[-3000:]
