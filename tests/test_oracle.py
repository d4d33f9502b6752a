"""Pins for the fp64 oracle (CPU only).  Each test names what fixes the
expected value independently of the oracle's own code: the paper's worked
example, SPEC worked examples, exact rational brute force, or a library
routine (numpy matmul) on data built without the oracle."""
import json
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import gqsa_oracle as O
from paper_2412_17560_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _pack_codes_int(codes, bits):
    """Independent n-bit little-endian packer (Python big-int) for the tests."""
    acc = 0
    for e, c in enumerate(codes):
        acc |= int(c) << (e * bits)
    nbytes = (len(codes) * bits + 7) // 8
    return np.frombuffer(acc.to_bytes(max(nbytes, 1), "little"), dtype=np.uint8)[:nbytes].copy()


def _f16(v):
    return np.asarray(v, dtype=np.float64).astype(np.float16).view(np.uint16)


# ---------------------------------------------------------------- unpack
def test_unpack_spec_examples():
    # SPEC.md:149 "codes [5, 1] -> byte 0x15"; "[15] -> 0x0F".
    assert list(O.unpack_codes(np.array([0x15], np.uint8), 2, 4)) == [5, 1]
    assert list(O.unpack_codes(np.array([0x0F], np.uint8), 1, 4)) == [15]


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_unpack_matches_bitwise_definition(bits):
    rng = random.Random(bits)
    n = 257
    codes = [rng.randrange(1 << bits) for _ in range(n)]
    packed = _pack_codes_int(codes, bits)
    assert list(O.unpack_codes(packed, n, bits)) == codes
    # and the generator's packer writes the same stream
    assert np.array_equal(synth.pack_bits(np.array(codes), bits), packed)


# ---------------------------------------------------------------- paper fixture
def _fixture():
    with open(os.path.join(GOLDEN, "paper_fig3.json")) as f:
        fx = json.load(f)
    bsr = {
        "rows": fx["rows"], "cols": fx["cols"], "group_size": fx["group_size"], "bits": fx["bits"],
        "nnzg": len(fx["group_cols"]),
        "row_index": np.array(fx["row_index"], np.int32),
        "group_cols": np.array(fx["group_cols"], np.uint16),
        "codes": _pack_codes_int(fx["codes"], fx["bits"]),
        "scales_f16": _f16(fx["scales"]), "zeros_f16": _f16(fx["zeros"]),
    }
    return fx, bsr


def test_paper_fixture_decompress():
    fx, bsr = _fixture()
    W = O.decompress(bsr)
    G = fx["group_size"]
    expect = np.zeros((fx["rows"], fx["cols"]))
    vals = np.array(fx["values"], float).reshape(-1, G)
    for r in range(fx["rows"]):
        for g in range(fx["row_index"][r], fx["row_index"][r + 1]):
            c = fx["group_cols"][g]
            expect[r, c * G:(c + 1) * G] = vals[g]
    assert np.array_equal(W, expect)
    assert np.all(W[2] == 0.0)  # the empty row (rowIndex[2] == rowIndex[3])


def test_paper_fixture_gemv_exact():
    fx, bsr = _fixture()
    for case in fx["cases"]:
        x = _f16(case["x"])
        y = O.gemv(bsr, x)[0]
        assert list(y) == [float(v) for v in case["y"]]
    # empty row yields exactly the bias
    bias = np.array([0.5, -1.0, 3.25, 0.0], np.float32)
    y = O.gemv(bsr, _f16(fx["cases"][0]["x"]), bias=bias)[0]
    assert y[2] == 3.25 and y[0] == 22.5


# ---------------------------------------------------------------- brute force
def _exact_y(keep, Q, s, z, x, G):
    """Exact rational y from the definition, independent of the oracle."""
    rows, gpr = keep.shape
    y = []
    gi = 0
    for r in range(rows):
        acc = Fraction(0)
        for c in range(gpr):
            if keep[r, c]:
                for t in range(G):
                    acc += (Fraction(int(Q[gi][t])) - Fraction(float(z[gi]))) * Fraction(float(s[gi])) \
                        * Fraction(float(x[c * G + t]))
                gi += 1
        y.append(acc)
    return y


@pytest.mark.parametrize("grid", [(2, 3), (3, 2)])
def test_bruteforce_every_mask(grid):
    rows, gpr = grid
    G, bits = 4, 4
    rng = np.random.default_rng(1234 + rows)
    for m in range(1 << (rows * gpr)):
        keep = np.array([(m >> i) & 1 for i in range(rows * gpr)], bool).reshape(rows, gpr)
        nnzg = int(keep.sum())
        Q = rng.integers(0, 16, size=(nnzg, G))
        s = rng.uniform(0.01, 2.0, nnzg).astype(np.float16).astype(np.float64)
        z = rng.uniform(-2.0, 17.0, nnzg).astype(np.float16).astype(np.float64)
        x = rng.normal(0, 3, gpr * G).astype(np.float16)
        bsr = synth.bsr_from_parts(rows, gpr * G, G, bits, keep, Q, s, z)
        y = O.gemv(bsr, x.view(np.uint16))[0]
        ex = _exact_y(keep, Q, s, z, x.astype(np.float64), G)
        for r in range(rows):
            # only additions round in fp64 (products exact): |err| <= n*u*sum|terms|
            bound = 0.0
            assert abs(Fraction(y[r]) - ex[r]) <= Fraction(64 * 2.0 ** -53) * (abs(ex[r]) + 1000)
        # dyadic integer inputs: the result is exact
        xi = rng.integers(-4, 5, gpr * G).astype(np.float16)
        si = rng.choice([0.5, 1.0, 2.0], nnzg)
        zi = rng.integers(0, 16, nnzg).astype(float)
        bsr = synth.bsr_from_parts(rows, gpr * G, G, bits, keep, Q, si, zi)
        y = O.gemv(bsr, xi.view(np.uint16))[0]
        ex = _exact_y(keep, Q, si, zi, xi.astype(np.float64), G)
        assert [Fraction(v) for v in y] == ex


# ---------------------------------------------------------------- library routine
@pytest.mark.parametrize("sparsity,mask", [(0.0, "uniform"), (0.5, "uniform"), (0.5, "skewed"),
                                           (0.3, "row_balanced")])
def test_dense_matmul_equivalence(sparsity, mask):
    """S=0 (and any mask): y equals numpy's dense matmul of a matrix the test
    builds itself from a dense code matrix -- exactly, in exact-integer mode."""
    rows, K, G, bits = 24, 96, 16, 4
    rng = np.random.default_rng(7)
    gpr = K // G
    keep = rng.random((rows, gpr)) >= sparsity if mask == "uniform" else None
    if mask == "skewed":
        keep = np.zeros((rows, gpr), bool)
        keep[rng.choice(rows, rows // 2, replace=False)] = True
    if mask == "row_balanced":
        keep = np.ones((rows, gpr), bool)
        for r in range(rows):
            keep[r, rng.choice(gpr, int(sparsity * gpr), replace=False)] = False
    Qd = rng.integers(0, 16, size=(rows, K))                # dense codes
    Sd = rng.choice([0.5, 1.0, 2.0], size=(rows, gpr))      # dense per-group s
    Zd = rng.integers(0, 16, size=(rows, gpr)).astype(float)
    x = rng.integers(-4, 5, size=K).astype(np.float16)
    # dense reference: pruned groups are zero
    Wd = (Qd - np.repeat(Zd, G, 1)) * np.repeat(Sd, G, 1) * np.repeat(keep, G, 1)
    ref = Wd @ x.astype(np.float64)
    # BSR of the kept groups, CSR order
    Qg = Qd.reshape(rows, gpr, G)[keep]
    bsr = synth.bsr_from_parts(rows, K, G, bits, keep, Qg, Sd[keep], Zd[keep])
    y = O.gemv(bsr, x.view(np.uint16))[0]
    assert np.array_equal(y, ref)
    # decompress places zeros at pruned positions and reproduces Wd
    assert np.array_equal(O.decompress(bsr), Wd)


def test_realistic_vs_blas_and_ascending_loop():
    bsr = synth.make_layer(11, 64, 256, sparsity=0.5)
    x = synth.make_x(12, 1, 256)
    y = O.gemv(bsr, x)[0]
    W = O.decompress(bsr)
    xf = x.view(np.float16).astype(np.float64)[0]
    # BLAS reorders the sum: agreement to 1e-12 relative of the absolute sum
    absum = np.abs(W) @ np.abs(xf)
    assert np.all(np.abs(W @ xf - y) <= 1e-12 * absum + 1e-300)
    # explicit ascending-column loop over the dense matrix: bit-exact (pruned
    # positions add +0.0)
    for r in range(0, 64, 7):
        acc = 0.0
        for j in range(256):
            acc += W[r, j] * xf[j]
        assert acc == y[r]


# ---------------------------------------------------------------- invariants
def test_linearity_and_batch():
    bsr = synth.make_layer(3, 32, 128, sparsity=0.5)
    x1 = synth.make_x(4, 1, 128)[0].view(np.float16).astype(np.float64)
    x2 = synth.make_x(5, 1, 128)[0].view(np.float16).astype(np.float64)
    a = 0.75
    y1, y2 = O.gemv(bsr, x1)[0], O.gemv(bsr, x2)[0]
    y12 = O.gemv(bsr, a * x1 + x2)[0]
    W = O.decompress(bsr)
    absum = np.abs(W) @ (np.abs(a * x1) + np.abs(x2))
    assert np.all(np.abs(y12 - (a * y1 + y2)) <= 1e-13 * absum)
    Y = O.gemv(bsr, np.stack([x1, x2]))
    assert np.array_equal(Y[0], y1) and np.array_equal(Y[1], y2)


def test_empty_layer():
    bsr = synth.make_layer(1, 8, 64, sparsity=1.0)
    assert bsr["nnzg"] == 0
    y = O.gemv(bsr, synth.make_x(2, 1, 64))
    assert np.array_equal(y, np.zeros((1, 8)))
    bias = np.arange(8, dtype=np.float32)
    assert np.array_equal(O.gemv(bsr, synth.make_x(2, 1, 64), bias=bias)[0], bias.astype(np.float64))


def test_validate_rejects_malformed():
    bsr = synth.make_layer(1, 8, 64, sparsity=0.5)
    O.validate_bsr(bsr)
    bad = dict(bsr, row_index=bsr["row_index"].copy())
    bad["row_index"][3], bad["row_index"][4] = bad["row_index"][4] + 1, bad["row_index"][3]
    with pytest.raises(ValueError):
        O.validate_bsr(bad)
    bad = dict(bsr, group_cols=bsr["group_cols"].copy())
    r0 = int(np.argmax(np.diff(bsr["row_index"]) >= 2))
    g = int(bsr["row_index"][r0])
    bad["group_cols"][g + 1] = bad["group_cols"][g]  # duplicate column in a row
    with pytest.raises(ValueError):
        O.validate_bsr(bad)


# ---------------------------------------------------------------- quantizer
def test_quantizer_spec_examples():
    # SPEC.md:122 / 124: [0, 1.5, 3] -> s=0.2, z=0 ; [-1, 2] -> s=0.2, z=5
    s, z = O.compute_qparams([0.0, 1.5, 3.0], 4)
    assert math.isclose(s, 0.2) and z == 0
    s2, z2 = O.compute_qparams([-1.0, 2.0], 4)
    assert math.isclose(s2, 0.2) and z2 == 5
    # codes [0, 8, 15] (7.5 rounds away from zero)
    assert O.quantize_group([0.0, 1.5, 3.0], s, z, 4) == [0, 8, 15]
    # out-of-range clamps
    assert O.quantize_group([10.0], 0.2, 0.0, 4) == [15]
    # dequantized [0, 1.6, 3.0]
    deq = O.dequantize_group([0, 8, 15], s, z)
    assert np.allclose(deq, [0.0, 1.6, 3.0])
    # reading R7: with fp16 storage of s, 8 * fp16(0.2) = 1.599609375
    assert 8 * float(np.float16(0.2)) == 1.599609375


def test_quantizer_roundtrip_property():
    rng = np.random.default_rng(0)
    for _ in range(2000):
        w = rng.normal(0, 1, 16)
        s, z = O.compute_qparams(w, 4)
        q = O.quantize_group(w, s, z, 4)
        assert min(q) >= 0 and max(q) <= 15
        deq = O.dequantize_group(q, s, z)
        assert np.max(np.abs(np.array(deq) - w)) <= s / 2 + 1e-6
    # degenerate group (reading R9): exact reconstruction
    for c in (0.0, 3.5, -0.125):
        s, z = O.compute_qparams([c] * 16, 4)
        q = O.quantize_group([c] * 16, s, z, 4)
        assert O.dequantize_group(q, s, z) == [c] * 16


# ---------------------------------------------------------------- partition / footprint
def test_partition_stream_k_spec_examples():
    sizes = [hi - lo for lo, hi in O.partition_stream_k(10, 3)]
    assert sizes == [4, 3, 3]
    parts = O.partition_stream_k(4, 8)
    assert sum(1 for lo, hi in parts if hi - lo == 1) == 4 and sum(1 for lo, hi in parts if hi == lo) == 4
    for total in range(0, 60):
        for p in range(1, 13):
            pr = O.partition_stream_k(total, p)
            sz = [hi - lo for lo, hi in pr]
            assert sum(sz) == total and max(sz) - min(sz) <= 1
            assert all(pr[i][1] == pr[i + 1][0] for i in range(p - 1))


def test_footprint_spec_example():
    # 4096x4096, G=16, n=4, 50% kept
    fp = O.footprint_bytes(4096, 4096, 524288, 16, 4)
    assert fp["codes"] * 8 == 33554432
    assert fp["scales"] * 8 == fp["zeros"] * 8 == fp["group_cols"] * 8 == 8388608
    assert fp["row_index"] * 8 == 131104
    bpw = fp["payload_file_bytes"] * 8 / (4096 * 4096)
    assert abs(bpw - 3.51) < 0.01
    assert 4.0 <= fp["ratio_vs_fp16"] <= 5.0  # brackets PAPER.md:399 "4.3x"
    # SURVEY Appendix B counted bytes
    assert fp["total"] == 7380996
    assert O.footprint_bytes(14336, 4096, 1835008, 16, 4)["total"] == 25812996
    assert O.footprint_bytes(4096, 14336, 1835008, 16, 4)["total"] == 25751556
