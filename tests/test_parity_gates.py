"""The parity gates themselves (tests/parity.py) on CPU: G2 must accept the
kernel-class rounding it is sized for and reject most single dropped groups
(a group's signed contribution can cancel to ~0, so no tolerance gate sees
all of them; the exact-integer GPU tests, bit-exact, are the strict check)."""
import numpy as np
import pytest

from oracle import gqsa_oracle as O
from paper_2412_17560_b200 import synth
from tests.parity import FOLD_REL_WORST, abs_bound, check_gates


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


def _emulate_w4_kernel_fp32(bsr, x_bits):
    """The kernel's W4 folded arithmetic emulated in numpy float32 (test-only):
    per group two FHFMA chains start at -P - zQ and 0 and add the exact
    products (1024 + q_t) x_t (t even) / (1024 + 16 q_t) x_t (t odd) in t
    order, t = fma(dd, 1/16, de), the row adds s * t (fp32) group by group."""
    f32 = np.float32
    G = 16
    X = np.asarray(x_bits).view(np.float16).astype(np.float64)[0]
    ri = bsr["row_index"]
    q_all = O.unpack_codes(bsr["codes"], int(bsr["nnzg"]) * G, 4).reshape(-1, G)
    s_all = O.f16_bits_to_f64(bsr["scales_f16"])
    z_all = O.f16_bits_to_f64(bsr["zeros_f16"])
    y = np.zeros(int(bsr["rows"]))
    for r in range(int(bsr["rows"])):
        acc = f32(0)
        for g in range(int(ri[r]), int(ri[r + 1])):
            xs = X[int(bsr["group_cols"][g]) * G:(int(bsr["group_cols"][g]) + 1) * G]
            xe, xo = f32(0), f32(0)
            for t in range(0, G, 2):  # column sums in t order (fp32, exact products)
                xe = f32(xe + f32(xs[t]))
                xo = f32(xo + f32(xs[t + 1]))
            P = f32(f32(1024.0 * float(xe)) + f32(64.0 * float(xo)))
            Q = f32(xe + xo)
            de = f32(-float(P) - float(z_all[g]) * float(Q))  # the chain starts at fma(z, -Q, -P)
            dd = f32(0)
            for t in range(G):
                prod = f32((1024.0 + (q_all[g, t] if t % 2 == 0 else 16 * q_all[g, t])) * xs[t])
                if t % 2 == 0:
                    de = f32(de + prod)
                else:
                    dd = f32(dd + prod)
            tt = f32(float(dd) * 0.0625 + float(de))
            acc = f32(float(s_all[g]) * float(tt) + float(acc))
        y[r] = float(acc)
    return y


def test_g2x_bounds_emulated_kernel_on_extreme_inputs():
    """G2x (the worst-case fold bound used for fp16-extreme activations) is a
    valid bound for the kernel's folded fp32 arithmetic, emulated step by step
    on extreme z / s / x."""
    bsr = synth.make_layer(synth.seed_for("g2x/extreme"), 48, 1024, bits=4, sparsity=0.5, mode="extreme")
    x = synth.make_x(synth.seed_for("g2x/extreme-x"), 1, 1024, mode="extreme")
    ref = O.gemv(bsr, x)[0]
    emu = _emulate_w4_kernel_fp32(bsr, x)
    A_worst = abs_bound(bsr, x, fold_rel=FOLD_REL_WORST)[0]
    assert np.all(np.abs(emu - ref) <= 1e-5 * A_worst + 1e-30)
