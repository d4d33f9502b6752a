"""Pins for the compression front-end oracle (oracle/gqsa_frontend.py), CPU
only.  Each expected value is fixed by something other than the oracle's own
code: a SPEC worked example, the paper's listing, an exhaustive brute force,
a closed form (diagonal H), or a property that must hold for any correct
implementation (exact pruned count, nestedness, homogeneity)."""
import itertools
import math

import numpy as np
import pytest

from oracle import gqsa_frontend as F
from oracle import gqsa_oracle as O


# ---------------------------------------------------------------- Hessian
def test_hessian_spec_example_unit_sample():
    # single sample x = e_1, d = 2 -> pre-damping H = [[2,0],[0,0]]
    H0 = F.estimate_hessian(np.array([[1.0, 0.0]]), damping=0.0)
    assert np.array_equal(H0, np.array([[2.0, 0.0], [0.0, 0.0]]))
    H = F.estimate_hessian(np.array([[1.0, 0.0]]))  # damped: 0.01 * mean(diag) = 0.01
    assert np.array_equal(H, np.array([[2.01, 0.0], [0.0, 0.01]]))
    assert np.all(np.diag(H) > 0)


def test_hessian_isotropic_and_symmetric():
    # orthonormal inputs covering all axes -> H proportional to I
    H = F.estimate_hessian(np.eye(4) * 3.0, damping=0.0)
    assert np.allclose(H, (2.0 / 4) * 9.0 * np.eye(4), rtol=0, atol=0)
    rng = np.random.default_rng(1)
    X = rng.standard_normal((17, 9))
    H = F.estimate_hessian(X)
    assert np.array_equal(H, H.T)
    # against the closed form 2/N X^T X (a different summation: BLAS matmul)
    assert np.allclose(H - np.diag(np.diag(H)), (2.0 / 17) * (X.T @ X) - np.diag(np.diag((2.0 / 17) * (X.T @ X))),
                       rtol=1e-12, atol=1e-12)


def test_hessian_needs_samples():
    with pytest.raises(ValueError):
        F.estimate_hessian(np.zeros((0, 3)))


def test_inverse_diagonal_closed_form():
    # diagonal H: [H^-1]_cc = 1 / H_cc exactly representable cases
    d = F.hessian_inv_diag(np.diag([2.0, 4.0, 0.5]))
    assert np.array_equal(d, np.array([0.5, 0.25, 2.0]))


# ---------------------------------------------------------------- Eq. 4
def test_weight_saliency_diagonal_hessian():
    # H = diag(a, b) -> s_{r,0} = W[r,0]^2 a^2
    a, b = 2.0, 4.0
    W = np.array([[3.0, -1.0], [0.5, 2.0]])
    s = F.weight_saliency(W, F.hessian_inv_diag(np.diag([a, b])))
    assert np.array_equal(s, np.array([[9.0 * a * a, 1.0 * b * b], [0.25 * a * a, 4.0 * b * b]]))


def test_weight_saliency_zero_row_and_homogeneity():
    rng = np.random.default_rng(2)
    W = rng.standard_normal((3, 8))
    W[1] = 0.0
    d = rng.uniform(0.5, 2.0, 8)
    s = F.weight_saliency(W, d)
    assert np.all(s >= 0) and np.all(s[1] == 0)
    s4 = F.weight_saliency(4.0 * W, d)                    # SPEC.md:208 (t = 4: exact powers of two)
    assert np.array_equal(s4, 16.0 * s)


# ---------------------------------------------------------------- groups
def test_group_saliency_spec_examples():
    assert np.array_equal(F.group_saliency(np.array([[1.0, 1.0, 3.0, 3.0]]), 2), np.array([[1.0, 3.0]]))
    assert np.array_equal(F.group_saliency(np.full((2, 6), 5.0), 3), np.full((2, 2), 5.0))
    row = np.array([[1.0, 2.0, 3.0, 6.0]])
    assert np.array_equal(F.group_saliency(row, 4), np.array([[3.0]]))
    with pytest.raises(ValueError):
        F.group_saliency(np.zeros((1, 5)), 2)


def test_select_spec_example_and_ties():
    # scores [[1,2],[3,4]], S = 0.5 -> prune (0,0), (0,1)
    keep = F.select_groups(np.array([[1.0, 2.0], [3.0, 4.0]]), 0.5)
    assert keep.tolist() == [[False, False], [True, True]]
    assert F.select_groups(np.array([[1.0, 2.0], [3.0, 4.0]]), 0.0).all()
    keep = F.select_groups(np.ones((2, 3)), 0.5)                               # SPEC.md:341 tie rule
    assert keep.tolist() == [[False, False, False], [True, True, True]]


@pytest.mark.parametrize("shape", [(2, 3), (3, 2), (1, 7)])
def test_select_bruteforce(shape):
    """Exhaustive check: the pruned set is the one minimising the total score
    among all sets of that size, ties broken by the lexicographically smallest
    index set (scores drawn from a small alphabet to force ties)."""
    rng = np.random.default_rng(sum(shape))
    n = shape[0] * shape[1]
    for trial in range(20):
        sc = rng.integers(0, 4, size=shape).astype(np.float64)
        for sp in (0.0, 0.25, 0.34, 0.5, 0.75, 0.99):
            k = int(math.floor(sp * n))
            flat = sc.reshape(-1)
            # brute force: minimal total score, then the lexicographically
            # smallest index tuple (any min-sum set holds the k smallest values)
            best = min(itertools.combinations(range(n), k), key=lambda idx: (sum(flat[list(idx)]), idx))
            keep = F.select_groups(sc, sp).reshape(-1)
            pruned = tuple(i for i in range(n) if not keep[i])
            assert pruned == best, (sc.tolist(), sp)


def test_select_nested_and_exact_count():
    rng = np.random.default_rng(5)
    sc = rng.standard_normal((16, 32))
    prev = np.ones_like(sc, dtype=bool)
    for sp in (0.0, 0.2, 0.3, 0.4, 0.5, 0.8):
        keep = F.select_groups(sc, sp)
        assert (~keep).sum() == math.floor(sp * sc.size)   # SPEC.md:366 exact count
        assert np.all(keep <= prev)                         # SPEC.md:367 nested keep-sets
        prev = keep
    # homogeneity: scaling W by t scales saliency by t^2 -> same ranking
    W = rng.standard_normal((8, 64))
    d = rng.uniform(0.1, 1.0, 64)
    k1 = F.select_groups(F.group_saliency(F.weight_saliency(W, d), 16), 0.5)
    k2 = F.select_groups(F.group_saliency(F.weight_saliency(3.0 * W, d), 16), 0.5)
    assert np.array_equal(k1, k2)


def test_dominant_row_survives():
    # a row 100x larger keeps all its groups at 50% sparsity
    rng = np.random.default_rng(7)
    W = rng.standard_normal((8, 64))
    W[3] *= 100.0
    _, keep, _ = F.compress_layer(W, np.ones(64), 0.5, 4)
    assert keep[3].all()


# ---------------------------------------------------------------- build_gqs
def test_paper_listing_topology():
    # rows own groups {1}, {0, 1}, {}, {1}
    keep = np.array([[False, True], [True, True], [False, False], [False, True]])
    W = np.arange(32, dtype=np.float32).reshape(4, 8) - 10.0
    bsr = F.build_gqs(W, keep, 4, 4)
    assert bsr["row_index"].tolist() == [0, 1, 3, 3, 4]
    assert bsr["group_cols"].tolist() == [1, 0, 1, 1]


def test_all_kept_roundtrip_within_half_step():
    # SPEC.md:265 / 385: all kept -> |W_hat - W| <= s/2 per element (s after fp16 rounding: + slack)
    rng = np.random.default_rng(9)
    W = (rng.standard_normal((6, 64)) * 0.02).astype(np.float32)
    bsr = F.build_gqs(W, np.ones((6, 4), bool), 16, 4)
    What = O.decompress(bsr)
    s = O.f16_bits_to_f64(bsr["scales_f16"])
    for g in range(bsr["nnzg"]):
        r, c = divmod(g, 4)
        err = np.abs(What[r, c * 16:(c + 1) * 16] - W[r, c * 16:(c + 1) * 16])
        assert np.all(err <= s[g] / 2 + 16 * s[g] * 2.0 ** -11 + 1e-12)


def test_all_pruned_and_codes_match_quantizer():
    W = np.linspace(-1, 1, 2 * 32, dtype=np.float32).reshape(2, 32)
    bsr = F.build_gqs(W, np.zeros((2, 2), bool), 16, 4)
    assert bsr["nnzg"] == 0 and bsr["row_index"].tolist() == [0, 0, 0]
    assert not O.decompress(bsr).any()
    # one kept group: codes are the SPEC quantizer's, packed low bits first
    keep = np.array([[True, False], [False, False]])
    bsr = F.build_gqs(W, keep, 16, 4)
    s, z = O.compute_qparams(W[0, :16].astype(np.float64), 4)
    q = O.quantize_group(W[0, :16].astype(np.float64), s, z, 4)
    assert list(O.unpack_codes(bsr["codes"], 16, 4)) == q
