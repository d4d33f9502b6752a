"""Full-size parity at BASELINE.json's configurations, in the launch
configuration bench.py times (same Layer / gqsa_gemv path, same grid):
sampled output rows are compared with the oracle evaluated row by row
(oracle.gemv_rows), under the same gates; exact-integer mode is compared on
every row."""
import numpy as np
import pytest

from oracle import gqsa_oracle as O
from paper_2412_17560_b200 import gqsa, synth
from tests.parity import abs_bound, check_gates

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SHAPES_8B = [(4096, 4096), (14336, 4096), (4096, 14336)]


def _sample_rows(n, k, seed):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([[0, n - 1], rng.choice(n, size=min(n, k), replace=False)]))


@pytest.mark.parametrize("rows,cols", SHAPES_8B)
@pytest.mark.parametrize("bits,sp", [(4, 0.5), (4, 0.3), (2, 0.5), (8, 0.5)])
def test_llama3_8b_shapes_sampled(rows, cols, bits, sp):
    name = f"llama3-8b/{rows}x{cols}/{bits}/{sp}/16/uniform"
    seed = synth.seed_for(name)
    bsr = synth.make_layer(seed, rows, cols, bits=bits, sparsity=sp)
    L = gqsa.Layer(bsr)
    for B in (1, 3, 8):  # 4096x14336 at B = 8: two launches of 4
        x = synth.make_x(seed + 1, B, cols)
        X = torch.from_numpy(x).view(torch.float16).cuda()
        y = (L.gemv(X[0])[None] if B == 1 else L.gemm(X)).cpu().numpy()
        rs = _sample_rows(rows, 192, seed + B)
        ref = O.gemv_rows(bsr, x, rs)
        check_gates(y[:, rs], ref, abs_bound(bsr, x, rs), name + f" B{B}")


@pytest.mark.parametrize("rows,cols", [(28672, 8192), (8192, 28672)])
def test_llama31_70b_shapes_sampled(rows, cols):
    name = f"llama3.1-70b/{rows}x{cols}/4/0.5/16/uniform"
    seed = synth.seed_for(name)
    bsr = synth.make_layer(seed, rows, cols, bits=4, sparsity=0.5)
    L = gqsa.Layer(bsr)
    x = synth.make_x(seed + 1, 1, cols)
    y = L.gemv(torch.from_numpy(x).view(torch.float16).cuda()[0]).cpu().numpy()[None]
    rs = _sample_rows(rows, 128, seed)
    check_gates(y[:, rs], O.gemv_rows(bsr, x, rs), abs_bound(bsr, x, rs), name)


def test_full_shape_exact_every_row():
    bsr = synth.make_layer(81, 14336, 4096, bits=4, sparsity=0.5, mode="exact_int")
    x = synth.make_x(82, 1, 4096, mode="exact_int")
    L = gqsa.Layer(bsr)
    y = L.gemv(torch.from_numpy(x).view(torch.float16).cuda()[0]).cpu().numpy()
    assert np.array_equal(y.astype(np.float64), O.gemv(bsr, x)[0])


@pytest.mark.parametrize("mask", ["row_balanced", "skewed"])
def test_slice_k_full_shape_sampled(mask):
    """The data-centric partition at a LLaMA shape, in the sweep's launch configuration."""
    name = f"llama3-8b/14336x4096/4/0.5/16/{mask}"
    seed = synth.seed_for(name)
    bsr = synth.make_layer(seed, 14336, 4096, bits=4, sparsity=0.5, mask=mask)
    L = gqsa.Layer(bsr)
    x = synth.make_x(seed + 1, 1, 4096)
    y = L.gemm(torch.from_numpy(x).view(torch.float16).cuda(), partition=gqsa.PARTITION_SLICE_K).cpu().numpy()
    rs = _sample_rows(14336, 192, seed)
    check_gates(y[:, rs], O.gemv_rows(bsr, x, rs), abs_bound(bsr, x, rs), name + " slice-k")
