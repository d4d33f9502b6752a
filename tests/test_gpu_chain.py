"""GPU parity of the persistent chain launch (gqsa_gemm_chain):
several GEMVs in one launch must give, item by item, what the fp64 oracle
gives -- bit-exact in exact-integer mode, within the gates G1/G2/G3
otherwise -- including true data dependencies (item j reads item j-1's fp16
output) and buffer reuse across items (write-after-read)."""
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


def _dev_blob(bsr):
    blob, desc = gqsa.pack(bsr)
    return desc, torch.from_numpy(blob).cuda()


def _x(xbits):
    return torch.from_numpy(np.ascontiguousarray(xbits)).view(torch.float16).cuda()


def run_chain(items, ws=None):
    ws = ws if ws is not None else torch.zeros(gqsa.chain_workspace_size(items, items[0][2].shape[0]),
                                               dtype=torch.uint8, device="cuda")
    gqsa.gemm_chain(items, ws)
    torch.cuda.synchronize()
    assert int(ws.count_nonzero()) == 0 or _flags_clear(ws), "workspace must be left reset"
    return ws


def _flags_clear(ws):
    w = ws.view(torch.int32)
    return int(w[0]) == 0 and int(w[64:].view(-1, 2)[:, 1].count_nonzero()) == 0


CHAIN_CASES = [
    # list of (rows, cols, sparsity, mask), bits, B, wait_prev
    ([(256, 256, 0.5, "uniform"), (1024, 4096, 0.5, "uniform"), (512, 2048, 0.5, "skewed")], 4, 1, 1),
    ([(1024, 4096, 0.5, "uniform"), (4096, 1024, 0.5, "uniform")], 4, 2, 1),
    ([(77, 208, 0.2, "uniform"), (5, 64, 0.5, "uniform"), (4096, 16, 0.5, "uniform"),
      (3, 16384, 0.5, "uniform")], 4, 1, 0),
    ([(640, 512, 0.9, "uniform"), (300, 1024, 0.3, "row_balanced")], 2, 2, 1),
    ([(2048, 14336, 0.5, "uniform"), (1024, 4096, 0.5, "uniform"), (1, 32768, 0.5, "uniform")], 2, 1, 1),
    ([(64, 128, 1.0, "uniform"), (256, 256, 0.5, "uniform")], 4, 1, 1),   # an all-empty layer first
]


@pytest.mark.parametrize("shapes,bits,B,wait", CHAIN_CASES)
def test_chain_exact_integer_bit_exact(shapes, bits, B, wait):
    items, refs = [], []
    for i, (rows, cols, sp, mask) in enumerate(shapes):
        seed = synth.seed_for(f"chain/{i}/{rows}/{cols}/{bits}/{sp}/{mask}/{B}")
        bsr = synth.make_layer(seed, rows, cols, bits=bits, sparsity=sp, mask=mask, mode="exact_int")
        x = synth.make_x(seed + 1, B, cols, mode="exact_int")
        desc, d_blob = _dev_blob(bsr)
        Y = torch.full((B, rows), float("nan"), dtype=torch.float32, device="cuda")
        items.append((desc, d_blob, _x(x), Y, None, wait))
        refs.append(O.gemv(bsr, x))
    ws = run_chain(items)
    for (_, _, _, Y, _, _), ref in zip(items, refs):
        y = Y.cpu().numpy().astype(np.float64)
        assert np.array_equal(y, ref), np.argwhere(y != ref)[:5]
    # reruns on the same workspace are bit-identical (the launch reset it)
    first = [it[3].clone() for it in items]
    for _ in range(5):
        run_chain(items, ws)
        for it, f in zip(items, first):
            assert torch.equal(it[3], f)


def test_chain_true_dependency_fp16_activations():
    """A decode-like dependent chain: item j reads item j-1's fp16 output, and
    the buffers ping-pong (item 2 overwrites item 0's input).  Items after the
    first are checked against the oracle run on the SAME fp16 activations the
    previous GPU item produced (fp16 rounding of a result that differs from
    the oracle's by fp32 rounding can differ in the last bit)."""
    dims = [4096, 1024, 4096, 2048, 4096]
    bsrs = [synth.make_layer(synth.seed_for(f"dep/{i}"), dims[i + 1], dims[i], sparsity=0.5)
            for i in range(4)]
    x0 = synth.make_x(synth.seed_for("dep/x"), 1, dims[0])
    A = torch.zeros(1, 4096, dtype=torch.float16, device="cuda")
    Bf = torch.zeros(1, 4096, dtype=torch.float16, device="cuda")
    A[:, :dims[0]] = _x(x0)
    bufs = [A, Bf, A, Bf, A]
    items = []
    for i, bsr in enumerate(bsrs):
        desc, d_blob = _dev_blob(bsr)
        Xi = bufs[i][:, :dims[i]]
        Yi = bufs[i + 1][:, :dims[i + 1]]
        items.append((desc, d_blob, Xi, Yi, None, 1))
    # reference inputs: recompute with the oracle step by step, feeding each
    # item the GPU's previous fp16 output (captured by running prefixes)
    xin = [x0]
    outs = []
    for n in range(1, 5):
        A[:, :dims[0]] = _x(x0)
        run_chain(items[:n])
        outs.append(bufs[n][:, :dims[n]].clone().cpu().numpy().view(np.uint16))
        if n < 4:
            xin.append(outs[-1])
    for i, bsr in enumerate(bsrs):
        ref = O.gemv(bsr, xin[i])
        y = outs[i].view(np.float16).astype(np.float64)
        # fp16 output: compare within the gates widened by the fp16 rounding
        err = np.abs(y - ref)
        assert np.all(err <= 2.0 ** -10 * np.abs(ref) + 1e-5 * abs_bound(bsr, xin[i])), i


REAL_CHAINS = [
    # the bench's step: LLaMA-3-8B q/o, gate/up, down (W4S50, B = 1)
    ([(4096, 4096), (14336, 4096), (4096, 14336)], 4, 0.5, 1),
    ([(4096, 4096), (1024, 4096), (1024, 4096), (4096, 4096), (14336, 4096), (14336, 4096),
      (4096, 14336)], 4, 0.5, 1),
    ([(4096, 4096), (14336, 4096), (4096, 14336)], 2, 0.5, 2),
]


@pytest.mark.parametrize("shapes,bits,sp,B", REAL_CHAINS)
def test_chain_realistic_gates_llama_shapes(shapes, bits, sp, B):
    items, cases = [], []
    for i, (rows, cols) in enumerate(shapes):
        seed = synth.seed_for(f"chainreal/{i}/{rows}/{cols}/{bits}")
        bsr = synth.make_layer(seed, rows, cols, bits=bits, sparsity=sp)
        x = synth.make_x(seed + 1, B, cols)
        desc, d_blob = _dev_blob(bsr)
        Y = torch.empty(B, rows, dtype=torch.float32, device="cuda")
        items.append((desc, d_blob, _x(x), Y, None, 1))
        cases.append((bsr, x))
    ws = run_chain(items)
    first = [it[3].clone() for it in items]
    for (bsr, x), it in zip(cases, items):
        check_gates(it[3].cpu().numpy(), O.gemv(bsr, x), abs_bound(bsr, x), f"chain {bsr['rows']}x{bsr['cols']}")
    run_chain(items, ws)
    for it, f in zip(items, first):
        assert torch.equal(it[3], f), "chain reruns must be bit-identical"


def test_chain_shared_input_reuse():
    """Items reading the SAME X without waiting (q/k/v, gate/up of a decoder
    layer) reuse the staged activations; results stay exact."""
    x = synth.make_x(31, 2, 4096, mode="exact_int")
    X = _x(x)
    items, refs = [], []
    for i, (rows, wait) in enumerate(((512, 1), (128, 0), (128, 0), (700, 1), (300, 0))):
        bsr = synth.make_layer(40 + i, rows, 4096, sparsity=0.5, mode="exact_int")
        desc, d_blob = _dev_blob(bsr)
        Y = torch.full((2, rows), float("nan"), dtype=torch.float32, device="cuda")
        items.append((desc, d_blob, X, Y, None, wait))
        refs.append(O.gemv(bsr, x))
    run_chain(items)
    for it, ref in zip(items, refs):
        assert np.array_equal(it[3].cpu().numpy().astype(np.float64), ref)


def test_chain_bias_and_fp16_output():
    bsr = synth.make_layer(7, 1000, 2048, sparsity=0.5, mode="exact_int")
    x = synth.make_x(8, 2, 2048, mode="exact_int")
    bias = (np.arange(1000) % 7 - 3).astype(np.float32)
    desc, d_blob = _dev_blob(bsr)
    b = torch.from_numpy(bias).cuda()
    Y32 = torch.empty(2, 1000, dtype=torch.float32, device="cuda")
    Y16 = torch.empty(2, 1000, dtype=torch.float16, device="cuda")
    run_chain([(desc, d_blob, _x(x), Y32, b, 1), (desc, d_blob, _x(x), Y16, b, 0)])
    ref = O.gemv(bsr, x, bias=bias.astype(np.float64))
    assert np.array_equal(Y32.cpu().numpy().astype(np.float64), ref)
    assert np.array_equal(Y16.cpu().numpy(), ref.astype(np.float16))


def test_chain_argument_errors():
    bsr = synth.make_layer(3, 256, 256, sparsity=0.5)
    desc, d_blob = _dev_blob(bsr)
    bsr2 = synth.make_layer(4, 256, 256, bits=2, sparsity=0.5)
    desc2, d_blob2 = _dev_blob(bsr2)
    X = torch.zeros(1, 256, dtype=torch.float16, device="cuda")
    Y = torch.zeros(1, 256, dtype=torch.float32, device="cuda")
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device="cuda")
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.gemm_chain([(desc, d_blob, X, Y, None, 1), (desc2, d_blob2, X, Y, None, 1)], ws)
    assert e.value.status == -3  # mixed bits
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.gemm_chain([(desc, d_blob, X, Y, None, 1)] * 17, ws)
    assert e.value.status == -1
    X3 = torch.zeros(3, 256, dtype=torch.float16, device="cuda")
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.gemm_chain([(desc, d_blob, X3, Y, None, 1)], ws)
    assert e.value.status == -1  # B = 3 is not a chain batch
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.gemm_chain([(desc, d_blob, X, Y, None, 1)], ws[:64])
    assert e.value.status == -4


def test_chain_max_items_and_ws_reuse():
    """16 items (GQSA_MAX_CHAIN), alternating dependent / independent, reused
    workspace over several launches: exact results every time."""
    items, refs = [], []
    for i in range(16):
        rows, cols = (128 + 64 * (i % 5), 256 * (1 + i % 3))
        bsr = synth.make_layer(100 + i, rows, cols, sparsity=0.5, mode="exact_int")
        x = synth.make_x(200 + i, 1, cols, mode="exact_int")
        desc, d_blob = _dev_blob(bsr)
        items.append((desc, d_blob, _x(x), torch.empty(1, rows, dtype=torch.float32, device="cuda"), None, i % 2))
        refs.append(O.gemv(bsr, x))
    ws = run_chain(items)
    for _ in range(3):
        for it in items:
            it[3].fill_(float("nan"))
        run_chain(items, ws)
        for it, ref in zip(items, refs):
            assert np.array_equal(it[3].cpu().numpy().astype(np.float64), ref)
