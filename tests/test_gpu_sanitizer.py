"""compute-sanitizer over small driver runs (the lock-free split-record
pool — volatile ready flags plus fences — and the shared-memory split stacks and
tallies were never checked). memcheck (out-of-bounds / misaligned device
accesses), racecheck (shared-memory hazards), synccheck (illegal barrier and
warp-synchronous use) must each report zero errors on the throughput engine
(cold start + a steady step, fixed-point and fp64 tally layouts) and memcheck
on the exact engine."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


def _run(tool, args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    p = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        os.path.join(ROOT, "scripts", "sanitize_case.py")] + args,
                       cwd=ROOT, capture_output=True, text=True, timeout=1800, env=e)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
    assert "ok" in p.stdout


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_philox_engine_clean(tool):
    _run(tool, ["philox", "2", "4000", "2"])


def test_philox_fp64_tallies_memcheck():
    _run("memcheck", ["philox", "2", "4000", "2"], env={"HWWG_FAST_FIX": "0"})


def test_philox_config3_memcheck():
    _run("memcheck", ["philox", "3", "4000", "3"])


def test_exact_engine_memcheck():
    _run("memcheck", ["exact", "2", "2000", "2"])
