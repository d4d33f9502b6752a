"""Every fix-up / partition mode of the whole-SM stream kernel, bit-exact on the GPU.

The library picks, per launch: the CTA-level fix-up for
whole-SM Stream-K launches, slice-aligned CTA ranges for single-item launches
at batch >= 2, the warp-level protocol for pipelined launches.  The default
selection is what every other GPU test exercises; the alternatives stay
selectable (GQSA_CTA_FIX, GQSA_CTA_SLICEK, read once per process), so each is
run here in a fresh process over tests/sanitize_small.py: every kernel family
in exact-integer mode against the fp64 oracle (PAPER.md:64-69 [Eq. 3],
95-101 [§3.2]), including whole-GPU launches whose slices cross CTA
boundaries, tiny layers with idle warps, and long-slice layers whose
slice-aligned CTA ranges are empty.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [
    {"GQSA_CTA_FIX": "0"},       # warp-level protocol in whole-SM launches
    {"GQSA_CTA_SLICEK": "1"},    # slice-aligned CTA ranges at every batch (also B = 1)
    {"GQSA_CTA_SLICEK": "0"},    # Stream-K + CTA-level fix-up at every batch
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_mode_bit_exact(env):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_small.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "sanitize_small: ok" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])
