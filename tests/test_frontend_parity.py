"""The product front-end (C ABI gqsa_compress + torch Hessian) against the
compression oracle (oracle/gqsa_frontend.py), CPU only.  Both sides evaluate
in fp64 in the paper's order, so given the same diag(H^-1) the keep mask,
codes and fp16 s/z bit patterns must be identical (bit-exact); the Hessian
inverse diagonal (two different factorisations) agrees to 1e-9 relative."""
import numpy as np
import pytest

from oracle import gqsa_frontend as F
from paper_2412_17560_b200 import frontend, gqsa, synth


def _same_bsr(a, b):
    for k in ("rows", "cols", "group_size", "bits", "nnzg"):
        assert int(a[k]) == int(b[k]), k
    for k in ("row_index", "group_cols", "codes", "scales_f16", "zeros_f16"):
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


CASES = [
    # rows, cols, G, bits, sparsity
    (64, 256, 16, 4, 0.5),
    (33, 128, 16, 2, 0.3),
    (16, 512, 16, 8, 0.8),
    (7, 96, 16, 4, 0.0),
    (40, 64, 8, 4, 0.45),
    (5, 48, 4, 2, 0.99),
]


@pytest.mark.parametrize("rows,cols,G,bits,sp", CASES)
def test_compress_bit_exact_vs_oracle(rows, cols, G, bits, sp):
    seed = synth.seed_for(f"frontend/{rows}/{cols}/{G}/{bits}/{sp}")
    W = synth.make_dense(seed, rows, cols)
    W[0, :G] = 0.0                    # a zero group (R9: s = 1, z = 0)
    W[1 % rows, G:2 * G] = -0.37      # a constant negative group
    W[2 % rows, :] = W[3 % rows, :]   # identical rows: tied scores
    X = synth.make_calib(seed + 1, 64, cols)
    d = F.hessian_inv_diag(F.estimate_hessian(X))
    ref, keep, per_group = F.compress_layer(W, d, sp, bits, G)
    got, sal = frontend.compress(W, d, sp, bits, G, return_saliency=True)
    assert np.array_equal(sal, per_group)
    _same_bsr(got, ref)


def test_compress_wide_dynamic_range_fp16_rounding():
    """Groups whose s, z span subnormal to large fp16 values: the C++ RNE
    conversion must match numpy's float64 -> float16."""
    rng = np.random.default_rng(3)
    rows, cols = 32, 256
    mag = 10.0 ** rng.uniform(-6, 2, size=(rows, cols // 16))
    W = (rng.standard_normal((rows, cols // 16, 16)) * mag[..., None]).reshape(rows, cols).astype(np.float32)
    W[5, 16:32] = 1.0 + 0.5 * rng.random(16)   # same-sign group: z = -30-ish
    d = np.ones(cols)
    ref, _, _ = F.compress_layer(W, d, 0.25, 4)
    _same_bsr(frontend.compress(W, d, 0.25, 4), ref)
    # a narrow same-sign group: z overflows fp16 -> both sides reject (reading R8)
    W[5, 16:32] = 100.0 + 1e-3 * rng.random(16)
    with pytest.raises(ValueError):
        F.compress_layer(W, d, 0.0, 4)
    with pytest.raises(gqsa.GQSAError) as e:
        frontend.compress(W, d, 0.0, 4)
    assert e.value.status == -2


def test_hessian_inverse_diag_vs_oracle():
    X = synth.make_calib(11, 256, 128)
    a = frontend.hessian_inv_diag(X)
    b = F.hessian_inv_diag(F.estimate_hessian(X))
    assert np.allclose(a, b, rtol=1e-9, atol=0)


def test_compress_feeds_pack_and_roundtrips():
    W = synth.make_dense(21, 128, 512)
    d = frontend.hessian_inv_diag(synth.make_calib(22, 128, 512))
    bsr = frontend.compress(W, d, 0.5, 4)
    assert bsr["nnzg"] == 128 * 32 - 128 * 16
    blob, desc = gqsa.pack(bsr)
    back = gqsa.unpack(blob)
    _same_bsr(back, bsr)


def test_compress_errors():
    W = np.zeros((4, 32), np.float32)
    d = np.ones(32)
    with pytest.raises(gqsa.GQSAError) as e:
        frontend.compress(W, d, 1.0, 4)
    assert e.value.status == -1
    with pytest.raises(gqsa.GQSAError) as e:
        frontend.compress(W, d, 0.5, 3)
    assert e.value.status == -3
    bad = d.copy()
    bad[3] = 0.0
    with pytest.raises(gqsa.GQSAError) as e:
        frontend.compress(W, bad, 0.5, 4)
    assert e.value.status == -2
    Wn = W.copy()
    Wn[1, 1] = np.nan
    with pytest.raises(gqsa.GQSAError) as e:
        frontend.compress(Wn, d, 0.5, 4)
    assert e.value.status == -2
    with pytest.raises(gqsa.GQSAError) as e:
        frontend.compress(np.zeros((4, 30), np.float32), np.ones(30), 0.5, 4)
    assert e.value.status == -1


def test_compress_other_group_sizes():
    """The front-end handles any G dividing K (plain BSR, checked against the
    oracle); the packer takes G = 8 / 32 at W4 (round trip) and rejects them
    at other widths (GQSA_ERR_UNSUPPORTED)."""
    W = synth.make_dense(31, 16, 128)
    d = np.ones(128)
    for G in (8, 32):
        ref, _, _ = F.compress_layer(W, d, 0.5, 4, G)
        got = frontend.compress(W, d, 0.5, 4, G)
        _same_bsr(got, ref)
        blob, desc = gqsa.pack(got)
        assert desc.group_size == G
        _same_bsr(gqsa.unpack(blob), got)
    got2 = frontend.compress(W, d, 0.5, 2, 8)
    _same_bsr(got2, F.compress_layer(W, d, 0.5, 2, 8)[0])
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.pack(got2)
    assert e.value.status == -3


def test_concat_rows_merges_layers_exactly():
    """frontend.concat_rows (merged q/k/v, gate/up): the merged BSR's rows are
    the inputs' rows in order, bit for bit, and its oracle GEMV is the
    concatenation of the inputs' GEMVs."""
    from oracle import gqsa_oracle as O
    parts = [synth.make_layer(60 + i, r, 512, bits=b, sparsity=0.5) for i, (r, b) in
             enumerate(((64, 4), (16, 4), (16, 4)))]
    merged = frontend.concat_rows(parts)
    assert merged["rows"] == 96 and merged["nnzg"] == sum(p["nnzg"] for p in parts)
    lo = 0
    for p in parts:
        sl = synth.slice_rows(merged, lo, lo + p["rows"])
        _same_bsr(sl, p)
        lo += p["rows"]
    x = synth.make_x(5, 2, 512)
    assert np.array_equal(O.gemv(merged, x), np.concatenate([O.gemv(p, x) for p in parts], axis=1))
    blob, desc = gqsa.pack(merged)
    _same_bsr(gqsa.unpack(blob), merged)
    with pytest.raises(ValueError):
        frontend.concat_rows([parts[0], synth.make_layer(1, 8, 256)])
