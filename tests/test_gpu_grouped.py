"""GPU parity of the grouped launch (gqsa_gemm_grouped): several
independent GEMVs in ONE launch -- their tile streams concatenated and cut
into equal per-warp ranges that cross item boundaries -- must give, item by
item, what the fp64 oracle gives: bit-exact in exact-integer mode, within the
gates G1/G2/G3 otherwise, bit-identical across reruns, workspace left zero."""
import os
import subprocess
import sys

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


def _ws(B):
    return torch.zeros(gqsa.workspace_size(gqsa.pack(synth.make_layer(1, 8, 16))[1], B), dtype=torch.uint8,
                       device="cuda")


def run_grouped(items, ws=None, **kw):
    B = items[0][2].shape[0]
    ws = ws if ws is not None else _ws(B)
    n0 = gqsa.launch_count()
    gqsa.gemm_grouped(items, ws, **kw)
    torch.cuda.synchronize()
    assert int(ws.count_nonzero()) == 0, "workspace must be left zero"
    return ws, gqsa.launch_count() - n0


GROUP_CASES = [
    # list of (rows, cols, sparsity, mask), bits, B
    ([(256, 256, 0.5, "uniform"), (1024, 4096, 0.5, "uniform"), (512, 2048, 0.5, "skewed")], 4, 1),
    ([(1024, 4096, 0.5, "uniform"), (4096, 1024, 0.5, "uniform")], 4, 2),
    ([(77, 208, 0.2, "uniform"), (5, 64, 0.5, "uniform"), (4096, 16, 0.5, "uniform"),
      (3, 16384, 0.5, "uniform")], 4, 1),
    ([(640, 512, 0.9, "uniform"), (300, 1024, 0.3, "row_balanced")], 2, 2),
    ([(2048, 14336, 0.5, "uniform"), (1024, 4096, 0.5, "uniform"), (1, 32736, 0.5, "uniform")], 2, 1),
    ([(64, 128, 1.0, "uniform"), (256, 256, 0.5, "uniform"), (64, 128, 1.0, "uniform")], 4, 1),  # empty items
    ([(1024, 4096, 0.5, "uniform"), (512, 1024, 0.5, "skewed"), (300, 2048, 0.3, "uniform")], 4, 4),
    ([(300, 1024, 0.5, "uniform"), (77, 208, 0.2, "uniform")], 8, 3),
    ([(100, 256, 0.5, "uniform")] * 8, 4, 1),  # GQSA_MAX_ITEMS small items: ranges span many items
]


@pytest.mark.parametrize("shapes,bits,B", GROUP_CASES)
def test_grouped_exact_integer_bit_exact(shapes, bits, B):
    items, refs = [], []
    for i, (rows, cols, sp, mask) in enumerate(shapes):
        seed = synth.seed_for(f"grouped/{i}/{rows}/{cols}/{bits}/{sp}/{mask}/{B}")
        bsr = synth.make_layer(seed, rows, cols, bits=bits, sparsity=sp, mask=mask, mode="exact_int")
        x = synth.make_x(seed + 1, B, cols, mode="exact_int")
        desc, d_blob = _dev_blob(bsr)
        Y = torch.full((B, rows), float("nan"), dtype=torch.float32, device="cuda")
        items.append((desc, d_blob, _x(x), Y, None))
        refs.append(O.gemv(bsr, x))
    for part in (gqsa.PARTITION_STREAM_K, gqsa.PARTITION_SLICE_K):
        for x_ready in (False, True):  # x_ready at B <= 2: the pipelined half-SM launch
            for it in items:
                it[3].fill_(float("nan"))
            _, launches = run_grouped(items, partition=part, x_ready=x_ready)
            assert launches == 1
            for it, ref in zip(items, refs):
                assert np.array_equal(it[3].cpu().numpy().astype(np.float64), ref), (part, x_ready)


@pytest.mark.parametrize("x_ready", [False, True])  # True: the bench's pipelined launch
@pytest.mark.parametrize("shapes,bits,sp,B", [
    ([(4096, 4096), (14336, 4096), (4096, 14336)], 4, 0.5, 1),   # the bench step
    ([(4096, 4096), (14336, 4096), (4096, 14336)], 2, 0.5, 2),
    ([(4096, 4096), (1024, 4096), (1024, 4096)], 4, 0.3, 1),     # LLaMA-3-8B q/k/v
    ([(13824, 5120), (13824, 5120)], 4, 0.5, 1),                 # Qwen2.5-14B gate/up
])
def test_grouped_realistic_gates_llama_shapes(shapes, bits, sp, B, x_ready):
    items, data = [], []
    for i, (rows, cols) in enumerate(shapes):
        seed = synth.seed_for(f"groupedreal/{i}/{rows}/{cols}/{bits}/{sp}")
        bsr = synth.make_layer(seed, rows, cols, bits=bits, sparsity=sp)
        x = synth.make_x(seed + 1, B, cols)
        desc, d_blob = _dev_blob(bsr)
        items.append((desc, d_blob, _x(x), torch.empty(B, rows, dtype=torch.float32, device="cuda"), None))
        data.append((bsr, x))
    ws, _ = run_grouped(items, x_ready=x_ready)
    first = [it[3].clone() for it in items]
    for it, (bsr, x) in zip(items, data):
        rs = np.random.default_rng(0).choice(bsr["rows"], size=min(bsr["rows"], 512), replace=False)
        ref = O.gemv_rows(bsr, x, rs)
        check_gates(it[3].cpu().numpy()[:, rs], ref, abs_bound(bsr, x, rs), f"grouped {bsr['rows']}x{bsr['cols']}")
    for _ in range(3):
        run_grouped(items, ws, x_ready=x_ready)
        for it, f in zip(items, first):
            assert torch.equal(it[3], f), "grouped reruns must be bit-identical"


def test_grouped_matches_single_launches_within_gates_and_x_ready():
    """Each item of a grouped launch agrees with its own single launch (the
    fp32 order may differ); x_ready = 1 (at B <= 2 the pipelined launch over
    half of every SM: another grid, so another fp32 order) agrees within the
    gates and is bit-identical across reruns."""
    shapes = [(1024, 4096), (2048, 2048), (512, 14336)]
    items, singles, data = [], [], []
    for i, (rows, cols) in enumerate(shapes):
        bsr = synth.make_layer(synth.seed_for(f"gvs/{i}"), rows, cols, sparsity=0.5)
        x = synth.make_x(i, 2, cols)
        L = gqsa.Layer(bsr)
        items.append((L.desc, L.blob, _x(x), torch.empty(2, rows, dtype=torch.float32, device="cuda"), None))
        singles.append(L.gemm(_x(x)))
        data.append((bsr, x))
    run_grouped(items)
    for it, s, (bsr, x) in zip(items, singles, data):
        check_gates(it[3].cpu().numpy(), s.cpu().numpy().astype(np.float64), abs_bound(bsr, x), "grouped vs single")
    run_grouped(items, x_ready=True)
    base = [it[3].clone() for it in items]
    for it, s, (bsr, x) in zip(items, singles, data):
        check_gates(it[3].cpu().numpy(), s.cpu().numpy().astype(np.float64), abs_bound(bsr, x), "x_ready vs single")
    for _ in range(3):
        run_grouped(items, x_ready=True)
        for it, b in zip(items, base):
            assert torch.equal(it[3], b), "x_ready reruns must be bit-identical"


@pytest.mark.parametrize("use_graph", [False, True])
def test_pipelined_back_to_back_launches(use_graph):
    """Consecutive x_ready launches on one stream overlap (each takes half of
    every SM; the next one streams and stages while this one drains) and share
    ONE workspace: every launch's results stay exact, also interleaved with a
    dependent x_ready = 0 launch that reads the previous launch's fp16 output,
    and when the whole sequence is replayed from a CUDA graph."""
    B = 1
    sets = []
    for k in range(4):
        shapes = [(1024, 4096), (3000, 1024), (512, 2048)][: 1 + k % 3]
        items, refs = [], []
        for i, (rows, cols) in enumerate(shapes):
            seed = synth.seed_for(f"pipe/{k}/{i}")
            bsr = synth.make_layer(seed, rows, cols, sparsity=0.5, mode="exact_int")
            x = synth.make_x(seed + 1, B, cols, mode="exact_int")
            desc, d_blob = _dev_blob(bsr)
            items.append((desc, d_blob, _x(x), torch.empty(B, rows, dtype=torch.float32, device="cuda"), None))
            refs.append(O.gemv(bsr, x))
        sets.append((items, refs))
    # a dependent pair: A writes fp16 y (exact: small integers), B reads it as its x
    bA = synth.make_layer(7001, 2048, 1024, sparsity=0.5, mode="exact_int")
    xA = synth.make_x(7002, B, 1024, mode="exact_int")
    yA_ref = O.gemv(bA, xA)
    bB = synth.make_layer(7003, 512, 2048, sparsity=0.5, mode="exact_int")
    assert np.all(np.abs(yA_ref) < 2048)
    yB_ref = O.gemv(bB, yA_ref.astype(np.float16).view(np.uint16))
    dA, blobA = _dev_blob(bA)
    dB, blobB = _dev_blob(bB)
    YA = torch.empty(B, 2048, dtype=torch.float16, device="cuda")
    YB = torch.empty(B, 512, dtype=torch.float32, device="cuda")
    ws = _ws(B)
    s = torch.cuda.Stream()

    def seq():
        for rep in range(3):
            for items, _ in sets:
                gqsa.gemm_grouped(items, ws, x_ready=True, stream=s)
            gqsa.gemm_grouped([(dA, blobA, _xA, YA, None)], ws, x_ready=True, stream=s)
            gqsa.gemm_grouped([(dB, blobB, YA, YB, None)], ws, x_ready=False, stream=s)

    _xA = _x(xA)
    for items, _ in sets:
        for it in items:
            it[3].fill_(float("nan"))
    YB.fill_(float("nan"))
    torch.cuda.synchronize()
    if use_graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            seq()
        g.replay()
        g.replay()
    else:
        seq()
    torch.cuda.synchronize()
    assert int(ws.count_nonzero()) == 0, "workspace must be left zero"
    for items, refs in sets:
        for it, ref in zip(items, refs):
            assert np.array_equal(it[3].cpu().numpy().astype(np.float64), ref)
    assert np.array_equal(YA.cpu().numpy().astype(np.float64), yA_ref.astype(np.float16).astype(np.float64))
    assert np.array_equal(YB.cpu().numpy().astype(np.float64), yB_ref)


def test_grouped_bias_and_fp16_output():
    bsr = synth.make_layer(31, 700, 1024, sparsity=0.5, mask="skewed", mode="exact_int")
    bsr2 = synth.make_layer(32, 96, 512, sparsity=0.5, mode="exact_int")
    x, x2 = synth.make_x(33, 1, 1024, mode="exact_int"), synth.make_x(34, 1, 512, mode="exact_int")
    b = np.arange(700, dtype=np.float32) * 0.25 - 40.0
    b2 = np.arange(96, dtype=np.float32) * -0.5
    (d, db), (d2, db2) = _dev_blob(bsr), _dev_blob(bsr2)
    Y16 = torch.empty(1, 700, dtype=torch.float16, device="cuda")
    Y16b = torch.empty(1, 96, dtype=torch.float16, device="cuda")
    run_grouped([(d, db, _x(x), Y16, torch.from_numpy(b).cuda()), (d2, db2, _x(x2), Y16b, torch.from_numpy(b2).cuda())])
    assert np.array_equal(Y16.cpu().numpy(), O.gemv(bsr, x, bias=b).astype(np.float16))
    assert np.array_equal(Y16b.cpu().numpy(), O.gemv(bsr2, x2, bias=b2).astype(np.float16))


def test_grouped_argument_errors():
    bsr = synth.make_layer(41, 64, 256, sparsity=0.5)
    desc, d_blob = _dev_blob(bsr)
    X = torch.zeros(1, 256, dtype=torch.float16, device="cuda")
    Y = torch.empty(1, 64, dtype=torch.float32, device="cuda")
    ws = _ws(1)
    bsr2 = synth.make_layer(42, 64, 256, bits=2, sparsity=0.5)
    desc2, d_blob2 = _dev_blob(bsr2)
    with pytest.raises(gqsa.GQSAError) as e:  # mixed bit widths
        gqsa.gemm_grouped([(desc, d_blob, X, Y, None), (desc2, d_blob2, X, Y, None)], ws)
    assert e.value.status == -3
    with pytest.raises(gqsa.GQSAError) as e:  # more than GQSA_MAX_ITEMS
        gqsa.gemm_grouped([(desc, d_blob, X, Y, None)] * 9, ws)
    assert e.value.status == -1
    with pytest.raises(gqsa.GQSAError) as e:  # workspace too small
        gqsa.gemm_grouped([(desc, d_blob, X, Y, None)], ws[:1024])
    assert e.value.status == -4
    with pytest.raises(gqsa.GQSAError) as e:  # ldy < rows
        gqsa.gemm_grouped([(desc, d_blob, X, torch.empty(1, 32, device="cuda"), None)], ws)
    assert e.value.status == -1


def test_grouped_item_split_when_activations_exceed_smem():
    """Eight one-tile items of K = 32736 land in one CTA, whose shared memory
    cannot hold all eight activation vectors: the library splits the item
    list into several launches, results exact.  (Runs with GQSA_MIN_TPW=0:
    by default a launch this small gets one-warp CTAs, each touching one item,
    and needs no split.)"""
    if os.environ.get("GQSA_MIN_TPW") != "0":
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu",
                            f"{os.path.abspath(__file__)}::test_grouped_item_split_when_activations_exceed_smem"],
                           env={**os.environ, "GQSA_MIN_TPW": "0"}, capture_output=True, text=True, timeout=600,
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
        return
    items, refs = [], []
    for i in range(8):
        bsr = synth.make_layer(synth.seed_for(f"gsplit/{i}"), 1, 32736, sparsity=0.99, mode="exact_int")
        x = synth.make_x(i, 1, 32736, mode="exact_int")
        desc, d_blob = _dev_blob(bsr)
        assert desc.num_tiles == 1
        items.append((desc, d_blob, _x(x), torch.empty(1, 1, dtype=torch.float32, device="cuda"), None))
        refs.append(O.gemv(bsr, x))
    _, launches = run_grouped(items)
    assert launches > 1
    for it, ref in zip(items, refs):
        assert np.array_equal(it[3].cpu().numpy().astype(np.float64), ref)
