"""Bounds-checked builds in place of compute-sanitizer (which is not available on
the GPU pool): paper_2512_19925_b200/_build_checked/libhwwg.so is the same
engine compiled with -DHWWG_CHECKS, whose device code checks the indices that
could go wrong — split-stack depth, pool tickets, source claims, tally slots
and keys, window-centre cells, edges, comb teeth and their source particles,
the multi-rank permutation — and traps on a violation (a failed launch, a
nonzero exit). Small runs of every engine path must finish clean and give the
same bookkeeping as the production build."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2512_19925_b200", "_build_checked", "libhwwg.so")


def _run(args, extra_env=None):
    if not os.path.exists(CHECKED):
        pytest.fail("checked build missing: run __graft_entry__.build()")
    env = dict(os.environ, HWWG_LIB=CHECKED, **(extra_env or {}))
    p = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py")] + args,
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    out = p.stdout + p.stderr
    assert p.returncode == 0 and "HWWG_CHECK failed" not in out, out[-3000:]
    return out


@pytest.mark.parametrize("which,H,steps", [(2, 20000, 3), (3, 20000, 3), (4, 20000, 2),
                                           (1, 20000, 4)])
def test_philox_paths_checked(which, H, steps):
    _run(["philox", str(which), str(H), str(steps)])


def test_philox_fp64_and_aggregated_tallies_checked():
    _run(["philox", "2", "20000", "3"], {"HWWG_FAST_FIX": "0"})
    _run(["philox", "2", "20000", "3"], {"HWWG_FAST_AGG": "1"})


def test_exact_path_checked():
    _run(["exact", "2", "5000", "2"])


def test_multirank_checked():
    code = ("import sys; sys.path.insert(0, '.'); from tests.test_gpu_multirank import run_world, c2;"
            "r = run_world(c2(20000, 3, 5), 3, 3, with_bank=True); print('ok', r[0][-1][0].segments)")
    env = dict(os.environ, HWWG_LIB=CHECKED)
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=900, env=env)
    assert p.returncode == 0 and "HWWG_CHECK failed" not in p.stdout + p.stderr, \
        (p.stdout + p.stderr)[-3000:]
