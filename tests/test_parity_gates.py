"""The parity gates themselves (tests/parity.py) on CPU: G2 must accept the
kernel-class rounding it is sized for and reject most single dropped groups
(a group's signed contribution can cancel to ~0, so no tolerance gate sees
all of them; the exact-integer GPU tests, bit-exact, are the strict check)."""
import numpy as np
import pytest

from oracle import gqsa_oracle as O
from paper_2412_17560_b200 import synth
from tests.parity import abs_bound, check_gates


@pytest.mark.parametrize("bits,rows,cols", [(4, 64, 4096), (2, 64, 14336), (8, 64, 4096), (4, 32, 28672)])
def test_g2_rejects_one_dropped_group(bits, rows, cols):
    bsr = synth.make_layer(synth.seed_for(f"gates/{bits}/{rows}/{cols}"), rows, cols, bits=bits, sparsity=0.5)
    x = synth.make_x(synth.seed_for(f"gates-x/{bits}/{cols}"), 1, cols)
    y = O.gemv(bsr, x)
    A = abs_bound(bsr, x)
    # fp32-class perturbation (well inside the gate) passes
    rng = np.random.default_rng(0)
    check_gates(y * (1 + 2.0 ** -22 * rng.uniform(-1, 1, A.shape)) + 1e-7 * A * rng.uniform(-1, 1, A.shape),
                y, A, "perturbed")
    # dropping one group (its exact contribution removed): G2 must see most
    ri = bsr["row_index"]
    ratios = []
    for r in range(0, rows, 5):
        for g in range(int(ri[r]), int(ri[r + 1]), 13):
            one = dict(bsr)
            keep_s = np.zeros_like(bsr["scales_f16"])
            keep_s[g] = bsr["scales_f16"][g]
            one["scales_f16"] = keep_s  # only group g contributes (other s = 0)
            c = O.gemv_rows(one, x, np.array([r]))[0, 0]
            ratios.append(abs(c) / (1e-5 * A[0, r]))
            if abs(c) > 1e-5 * A[0, r]:
                yd = y.copy()
                yd[0, r] -= c
                with pytest.raises(AssertionError):
                    check_gates(yd, y, A, "dropped")
    ratios = np.array(ratios)
    assert np.median(ratios) > 2.0 and np.mean(ratios > 1.0) > 0.6, (np.median(ratios), np.mean(ratios > 1))
