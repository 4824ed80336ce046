"""K1's non-default completion modes (SPECDEC_K1_SPLIT, read once per process) against the
oracle: the verify tests (planted, natural ties / NaN / +-0, EOS / budget / inactive rows,
brute force, fuzz), the round brute force and the pool epochs, each mode in its own
process.  Modes: 0 grid-wide last-CTA arrival; 2 per-row arrival (+ the plan arrival for
specdec_verify).  The default (1 for specdec_verify, 2 for specdec_pool_verify) runs in
every other test."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["0,0", "2,2"])
def test_k1_completion_mode_matches_oracle(mode):
    env = dict(os.environ, SPECDEC_K1_SPLIT=mode)
    sel = ["tests/test_gpu_verify.py", "tests/test_gpu_brute.py::test_round_brute_force",
           "tests/test_gpu_pool.py::test_pool_epochs_match_oracle",
           "tests/test_gpu_pool.py::test_native_epoch_executor_matches_python_driver",
           "tests/test_host_drivers.py::test_kernels_per_round"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *sel],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
