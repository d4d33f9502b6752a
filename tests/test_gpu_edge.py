"""GPU parity at the edges of the value ranges (reading R6: z is
any finite fp16 after E2E-OQP, not an integer in [0, 2^n-1]) and of the inputs:

* z over the fp16 range -- large |z| (up to ~1e3), negative z, integer z
  outside [0, 2^n-1], fp16-subnormal z -- with fp16-subnormal scales, and x
  with fp16 extremes (|x| up to 65504, subnormals, exact zeros), for W2 / W4 /
  W8, batch 1 and 2, Stream-K and Slice-K, against the fp64 oracle under the
  gates G1, G3 and G2x (G2 with the worst-case summation bound of the folded
  chains, tests/parity.py / DESIGN.md §7: with |x| up to 65504 the fold
  offsets 1024 |x| dominate), at a full LLaMA shape (sampled rows) too;
* an infinite activation: rows whose kept groups do not touch it stay finite
  and exact (padding slots read the zero block, never x), rows that touch it
  are non-finite like the oracle's.
"""
import numpy as np
import pytest

from oracle import gqsa_oracle as O
from paper_2412_17560_b200 import gqsa, synth
from tests.parity import FOLD_REL_WORST, abs_bound, check_gates

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.init()


def _run(L, x, part):
    X = torch.from_numpy(np.ascontiguousarray(x)).view(torch.float16).cuda()
    y = L.gemm(X, partition=part)
    torch.cuda.synchronize()
    assert int(L.ws.count_nonzero()) == 0
    return y.cpu().numpy()


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("B", [1, 2])
def test_extreme_z_s_x_gates(bits, B):
    seed = synth.seed_for(f"edge/extreme/{bits}/{B}")
    bsr = synth.make_layer(seed, 2048, 4096, bits=bits, sparsity=0.5, mode="extreme")
    x = synth.make_x(seed + 1, B, 4096, mode="extreme")
    z = O.f16_bits_to_f64(bsr["zeros_f16"])
    qmax = (1 << bits) - 1
    assert (z < 0).any() and (z > qmax).any() and np.abs(z).max() > 500  # the range R6 allows
    assert ((np.abs(z) < 2.0 ** -14) & (z != 0)).any()  # fp16-subnormal zeros
    assert (O.f16_bits_to_f64(bsr["scales_f16"]) < 2.0 ** -14).any()  # fp16-subnormal scales
    ref = O.gemv(bsr, x)
    A = abs_bound(bsr, x, fold_rel=FOLD_REL_WORST)
    L = gqsa.Layer(bsr)
    for part in (gqsa.PARTITION_STREAM_K, gqsa.PARTITION_SLICE_K):
        check_gates(_run(L, x, part), ref, A, f"extreme W{bits} B{B} part{part}")


@pytest.mark.parametrize("part", [gqsa.PARTITION_STREAM_K, gqsa.PARTITION_SLICE_K])
def test_extreme_values_full_llama_down_proj_sampled(part):
    """4096 x 14336 (LLaMA-3-8B down_proj) W4S50 with extreme z / s / x, in the
    bench's launch configuration: 256 sampled rows against the oracle."""
    seed = synth.seed_for("edge/extreme/down")
    bsr = synth.make_layer(seed, 4096, 14336, bits=4, sparsity=0.5, mode="extreme")
    x = synth.make_x(seed + 1, 1, 14336, mode="extreme")
    rows = np.sort(np.random.default_rng(0).choice(4096, size=256, replace=False))
    y = _run(gqsa.Layer(bsr), x, part)[:, rows]
    check_gates(y, O.gemv_rows(bsr, x, rows), abs_bound(bsr, x, rows, fold_rel=FOLD_REL_WORST),
                f"extreme down_proj part{part}")


@pytest.mark.parametrize("bits", [4, 2])
def test_infinite_activation_stays_in_its_rows(bits):
    """x[j] = +inf: the rows that keep the group of column j are non-finite
    (as in the oracle); every other row -- including rows whose lanes hold
    padding slots -- is finite and bit-exact (exact-integer mode)."""
    seed = synth.seed_for(f"edge/inf/{bits}")
    bsr = synth.make_layer(seed, 777, 1024, bits=bits, sparsity=0.7, mask="uniform", mode="exact_int")
    x = synth.make_x(seed + 1, 1, 1024, mode="exact_int")
    j = 37
    x = x.copy()
    x[0, j] = np.float16(np.inf).view(np.uint16)
    ref = O.gemv(bsr, x)[0]
    ri, gc = bsr["row_index"], bsr["group_cols"]
    touch = np.array([np.any(gc[ri[r]:ri[r + 1]] == j // 16) for r in range(777)])
    assert touch.any() and (~touch).any()
    L = gqsa.Layer(bsr)
    for part in (gqsa.PARTITION_STREAM_K, gqsa.PARTITION_SLICE_K):
        y = _run(L, x, part)[0].astype(np.float64)
        assert np.array_equal(y[~touch], ref[~touch]), part
        assert not np.isfinite(y[touch]).any() and not np.isfinite(ref[touch]).any(), part
