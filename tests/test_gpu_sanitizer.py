"""GPU: compute-sanitizer over every device path (tests/tools/sanitize_driver.py):
memcheck (out-of-bounds / misaligned accesses), racecheck (shared-memory
hazards, e.g. in k_tail's block-resident lists), synccheck (barrier misuse:
k_tail's grid barrier sits between block barriers) -- zero errors each.
racecheck and synccheck run the same kernels as plain launches
(--host-loop-only): under racecheck the whole-solve CUDA graph (conditional
WHILE node + cooperative k_tail node) crashed the tool's host side
intermittently while every kernel of it passed as a plain launch."""
import os
import shutil
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "7", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tests", "tools", "sanitize_driver.py")]
    if tool != "memcheck":
        cmd.append("--host-loop-only")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    if "sanitizer is closed" in out or "sanitizer is disabled" in out:
        # the GPU pool's own wrapper refuses the tool (it exits before running
        # anything); the last clean run is kept in profiles/r02/sanitizer.txt
        pytest.skip("compute-sanitizer refused by this GPU pool: " + out.strip()[:200])
    assert r.returncode == 0, out[-4000:]
    assert "sanitize driver ok" in out, out[-4000:]
    # memcheck / synccheck: "ERROR SUMMARY: 0 errors"; racecheck: "... (0 errors, 0 warnings)"
    assert "ERROR SUMMARY: 0 errors" in out or "hazards displayed (0 errors" in out, out[-4000:]
    print(out[-600:])
