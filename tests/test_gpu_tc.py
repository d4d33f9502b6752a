"""GPU parity of the small-batch tensor-core path (LAYOUT-TC + gqsa_tc.cu,
mma.sync.m16n8k16 over 16-row blocks) against the fp64
oracle: bit-exact in exact-integer mode for every batch 1..8 (all partial
sums are exact in fp32, whatever order the tensor core adds the products
in), Stream-K and Slice-K, ragged shapes (last block partial, blocks with no
kept group, K at its maximum, column sums from the mma when the X_c table does
not fit beside x, batch split when x itself does not fit); the gates
G1-G3 on realistic values; fp16 output with bias; bit-identical reruns."""
import numpy as np
import pytest

from oracle import gqsa_oracle as O
from paper_2412_17560_b200 import gqsa, synth
from tests.parity import abs_bound, check_gates

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.init()


def _run(L, x, part=gqsa.PARTITION_STREAM_K, out_dtype=None, bias=None):
    X = torch.from_numpy(np.ascontiguousarray(x)).view(torch.float16).cuda()
    b = None if bias is None else torch.from_numpy(bias).cuda()
    y = L.gemm(X, partition=part, out_dtype=out_dtype, bias=b)
    torch.cuda.synchronize()
    assert int(L.ws.count_nonzero()) == 0, "workspace left zero"
    return y.cpu().numpy()


TC_EXACT = [
    # rows, cols, sparsity, mask, B
    (256, 256, 0.5, "uniform", 8),
    (1024, 4096, 0.5, "uniform", 4),
    (1000, 4096, 0.5, "uniform", 8),     # last block partial
    (333, 1024, 0.3, "row_balanced", 5),
    (512, 2048, 0.5, "skewed", 2),       # whole blocks without a kept group
    (77, 208, 0.2, "uniform", 3),
    (4096, 16, 0.5, "uniform", 1),       # K = G
    (5, 64, 0.5, "uniform", 7),
    (640, 512, 0.9, "uniform", 6),
    (64, 32736, 0.5, "uniform", 8),      # K at its maximum: batch split (3 x 3 rows, X_c by mma)
    (2048, 14336, 0.5, "uniform", 8),    # LLaMA down_proj width: one launch, X_c by mma
]


def test_tc_launch_plan_x_only_at_down_proj_width():
    """B = 8 at K = 14336: x (8 x (2K + 32) B) fits the 225-KB budget only
    without the X_c table -- one launch, weights streamed once."""
    bsr = synth.make_layer(5, 64, 14336, bits=4, sparsity=0.5)
    blob, desc = gqsa.pack(bsr, layout=gqsa.LAYOUT_TC)
    plan = gqsa.launch_plan(desc, 8)
    assert plan.launches == 1 and plan.batch_per_launch == 8
    assert plan.smem_bytes == 8 * (2 * 14336 + 32)
    plan = gqsa.launch_plan(desc, 4)  # the table fits: the cheaper staging
    assert plan.smem_bytes == 4 * (2 * 14336 + 32) + (14336 // 16 + 1) * 32


@pytest.mark.parametrize("rows,cols,sp,mask,B", TC_EXACT)
def test_tc_exact_integer_bit_exact(rows, cols, sp, mask, B):
    seed = synth.seed_for(f"tc/{rows}/{cols}/{sp}/{mask}/{B}")
    bsr = synth.make_layer(seed, rows, cols, bits=4, sparsity=sp, mask=mask, mode="exact_int")
    x = synth.make_x(seed + 1, B, cols, mode="exact_int")
    ref = O.gemv(bsr, x)
    L = gqsa.Layer(bsr, layout=gqsa.LAYOUT_TC)
    for part in (gqsa.PARTITION_STREAM_K, gqsa.PARTITION_SLICE_K):
        y = _run(L, x, part)
        assert np.array_equal(y.astype(np.float64), ref), (part, np.argwhere(y != ref)[:5])


@pytest.mark.parametrize("rows,cols,B", [(4096, 4096, 8), (14336, 4096, 4), (4096, 14336, 8), (2048, 5120, 2)])
def test_tc_realistic_gates_and_determinism(rows, cols, B):
    seed = synth.seed_for(f"tcreal/{rows}/{cols}/{B}")
    bsr = synth.make_layer(seed, rows, cols, bits=4, sparsity=0.5)
    x = synth.make_x(seed + 1, B, cols)
    rs = np.sort(np.random.default_rng(1).choice(rows, size=min(rows, 512), replace=False))
    L = gqsa.Layer(bsr, layout=gqsa.LAYOUT_TC)
    y = _run(L, x)
    check_gates(y[:, rs], O.gemv_rows(bsr, x, rs), abs_bound(bsr, x, rs), f"tc {rows}x{cols} B{B}")
    for _ in range(3):
        assert np.array_equal(_run(L, x), y)


def test_tc_fp16_output_bias_and_onehot():
    bsr = synth.make_layer(71, 700, 1024, bits=4, sparsity=0.5, mask="skewed", mode="exact_int")
    x = synth.make_x(72, 8, 1024, mode="exact_int")
    bias = (np.arange(700, dtype=np.float32) * 0.25 - 40.0).astype(np.float32)
    L = gqsa.Layer(bsr, layout=gqsa.LAYOUT_TC)
    y = _run(L, x, out_dtype=torch.float16, bias=bias)
    assert np.array_equal(y.view(np.uint16), O.gemv(bsr, x, bias=bias).astype(np.float16).view(np.uint16))
    bsr = synth.make_layer(73, 512, 1024, bits=4, sparsity=0.5, mode="onehot_safe")
    W = O.decompress(bsr)
    x = synth.make_x(74, 8, 1024, mode="onehot")
    y = _run(gqsa.Layer(bsr, layout=gqsa.LAYOUT_TC), x)
    cols = np.argmax(x.view(np.float16) != 0, axis=1)
    for b in range(8):
        assert np.array_equal(y[b].astype(np.float64), W[:, cols[b]])
