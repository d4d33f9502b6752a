"""GPU parity: the sm_100a path (through the C ABI) against the fp64 oracle on
the same seeded inputs.  Bit-exact in exact-integer and one-hot modes,
tolerance gates G1/G2/G3 (tests/parity.py) otherwise."""
import json
import os

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


def run(bsr, xbits, bias=None, layer=None, partition=gqsa.PARTITION_STREAM_K, **kw):
    """Pack, upload, run gqsa_gemm_smallbatch (B = rows of x), return y [B][N] float32."""
    L = layer or gqsa.Layer(bsr)
    X = torch.from_numpy(np.ascontiguousarray(xbits)).view(torch.float16).cuda()
    if X.ndim == 1:
        X = X[None]
    b = None if bias is None else torch.from_numpy(bias).cuda()
    if X.shape[0] == 1 and not kw.get("force_gemm") and partition == gqsa.PARTITION_STREAM_K:
        y = L.gemv(X[0], bias=b)[None]
    else:
        y = L.gemm(X, bias=b, partition=partition)
    torch.cuda.synchronize()
    assert int(L.ws.count_nonzero()) == 0, "the workspace (fix-up counters and records) must be left zero"
    return y.cpu().numpy()


# ------------------------------------------------------------------ paper fixture
def test_paper_fixture_embedded_g16():
    """PAPER.md:95-101 listing (tests/golden/paper_fig3.json) embedded in G=16:
    each 4-wide group sits in the first 4 slots of a 16-wide group whose other
    codes equal z (dequantize to exactly 0).  y must equal the paper-derived
    values exactly."""
    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_fig3.json")))
    codes = np.array(fx["codes"]).reshape(-1, 4)
    z = np.array(fx["zeros"])
    full = np.repeat(z[:, None], 16, 1).astype(np.int64)
    full[:, :4] = codes
    keep = np.zeros((4, 2), bool)
    ri = fx["row_index"]
    for r in range(4):
        for g in range(ri[r], ri[r + 1]):
            keep[r, fx["group_cols"][g]] = True
    bsr = synth.bsr_from_parts(4, 32, 16, 4, keep, full, np.array(fx["scales"]), z)
    for case in fx["cases"]:
        x = np.zeros(32)
        for j, v in enumerate(case["x"]):
            x[(j // 4) * 16 + j % 4] = v
        x[4:16] = 7.0  # multiplied by exact zeros
        x[20:32] = -3.0
        y = run(bsr, x.astype(np.float16).view(np.uint16))[0]
        assert list(y) == [float(v) for v in case["y"]]


# ------------------------------------------------------------------ exact modes
EXACT_CASES = [
    # rows, cols, bits, sparsity, mask, B
    (256, 256, 4, 0.5, "uniform", 1),
    (256, 256, 2, 0.5, "uniform", 1),
    (1024, 4096, 4, 0.5, "uniform", 1),
    (1024, 4096, 2, 0.5, "uniform", 3),
    (512, 2048, 4, 0.5, "skewed", 1),
    (300, 1024, 4, 0.3, "row_balanced", 4),
    (77, 208, 4, 0.2, "uniform", 8),      # ragged tile tail, odd rows
    (77, 208, 2, 0.5, "uniform", 3),      # x + column sums of 1560 B: ring alignment (sanitizer find)
    (41, 48, 4, 0.5, "uniform", 5),       # K = 48: 3 column groups, odd batch
    (3, 16384, 4, 0.5, "uniform", 2),     # few long rows: rows span many warps
    (1, 32736, 4, 0.5, "uniform", 1),     # one row over 32 lanes (S = 32), max K
    (4096, 16, 4, 0.5, "uniform", 1),     # K = G: many empty rows, 1-group rows
    (5, 64, 4, 0.5, "uniform", 1),        # nnzg < one tile
    (640, 512, 2, 0.9, "uniform", 5),     # mostly-empty rows
    (2048, 28672, 4, 0.5, "uniform", 4),  # x of 4 columns exceeds an SM: 2 launches of 2
    (1024, 14336, 4, 0.5, "uniform", 8),  # x of 8 columns exceeds an SM: 2 launches of 4
    (512, 14336, 2, 0.5, "skewed", 3),    # half the rows empty, long rows
    # W8 (exact-int needs 255*2*4*K < 2^23: K <= 4096)
    (1024, 4096, 8, 0.5, "uniform", 1),
    (300, 1024, 8, 0.3, "row_balanced", 4),
    (77, 208, 8, 0.2, "uniform", 8),
    (512, 2048, 8, 0.5, "skewed", 2),
]


@pytest.mark.parametrize("rows,cols,bits,sp,mask,B", EXACT_CASES)
def test_exact_integer_mode_bit_exact(rows, cols, bits, sp, mask, B):
    seed = synth.seed_for(f"exact/{rows}/{cols}/{bits}/{sp}/{mask}/{B}")
    bsr = synth.make_layer(seed, rows, cols, bits=bits, sparsity=sp, mask=mask, mode="exact_int")
    x = synth.make_x(seed + 1, B, cols, mode="exact_int")
    y = run(bsr, x)
    ref = O.gemv(bsr, x)
    assert np.array_equal(y.astype(np.float64), ref), np.argwhere(y != ref)[:5]


SLICE_K_CASES = [
    # rows, cols, bits, sparsity, mask, B
    (1024, 4096, 4, 0.5, "uniform", 1),
    (1024, 4096, 2, 0.5, "uniform", 3),
    (512, 2048, 4, 0.5, "skewed", 1),
    (300, 1024, 4, 0.3, "row_balanced", 4),
    (77, 208, 4, 0.2, "uniform", 8),
    (3, 16384, 4, 0.5, "uniform", 2),     # fewer slices than warps
    (4096, 16, 4, 0.5, "uniform", 1),
    (640, 512, 2, 0.9, "uniform", 5),
]


@pytest.mark.parametrize("rows,cols,bits,sp,mask,B", SLICE_K_CASES)
def test_slice_k_partition_bit_exact(rows, cols, bits, sp, mask, B):
    """Data-centric partition (App. J baseline): whole slices per warp, no fix-up."""
    seed = synth.seed_for(f"slicek/{rows}/{cols}/{bits}/{sp}/{mask}/{B}")
    bsr = synth.make_layer(seed, rows, cols, bits=bits, sparsity=sp, mask=mask, mode="exact_int")
    x = synth.make_x(seed + 1, B, cols, mode="exact_int")
    y = run(bsr, x, partition=gqsa.PARTITION_SLICE_K)
    assert np.array_equal(y.astype(np.float64), O.gemv(bsr, x))


@pytest.mark.parametrize("mask", ["uniform", "skewed"])
def test_slice_k_realistic_and_deterministic(mask):
    bsr = synth.make_layer(81, 4096, 4096, sparsity=0.5, mask=mask)
    x = synth.make_x(82, 2, 4096)
    L = gqsa.Layer(bsr)
    y = run(bsr, x, layer=L, partition=gqsa.PARTITION_SLICE_K)
    check_gates(y, O.gemv(bsr, x), abs_bound(bsr, x), f"slice-k {mask}")
    assert np.array_equal(run(bsr, x, layer=L, partition=gqsa.PARTITION_SLICE_K), y)
    with pytest.raises(gqsa.GQSAError) as e:
        X = torch.zeros(1, 4096, dtype=torch.float16, device="cuda")
        gqsa.gemm_ex(L.desc, L.blob, X, torch.empty(1, 4096, device="cuda"), 7, ws=L.ws)
    assert e.value.status == -1


@pytest.mark.parametrize("bits,B", [(4, 1), (2, 3), (8, 8)])
def test_fp16_output_exact(bits, B):
    """fp16 y (RNE of the fp32 result + bias): in exact-integer mode the fp32
    value is exact, so y16 == fp16(oracle) bit for bit; empty rows get fp16(bias)."""
    bsr = synth.make_layer(91 + bits, 700, 1024, bits=bits, sparsity=0.5, mask="skewed", mode="exact_int")
    x = synth.make_x(92, B, 1024, mode="exact_int")
    bias = (np.arange(700, dtype=np.float32) * 0.25 - 40.0).astype(np.float32)
    L = gqsa.Layer(bsr)
    X = torch.from_numpy(x).view(torch.float16).cuda()
    for part in (gqsa.PARTITION_STREAM_K, gqsa.PARTITION_SLICE_K):
        y = L.gemm(X, bias=torch.from_numpy(bias).cuda(), partition=part, out_dtype=torch.float16)
        torch.cuda.synchronize()
        ref = O.gemv(bsr, x, bias=bias).astype(np.float16)
        assert np.array_equal(y.cpu().numpy().view(np.uint16), ref.view(np.uint16))


def test_empty_layer_and_bias():
    bsr = synth.make_layer(5, 100, 64, sparsity=1.0)
    bias = np.linspace(-1, 1, 100).astype(np.float32)
    y = run(bsr, synth.make_x(6, 1, 64), bias=bias)[0]
    assert np.array_equal(y, bias)
    bsr = synth.make_layer(7, 333, 512, sparsity=0.5, mask="skewed", mode="exact_int")
    x = synth.make_x(8, 2, 512, mode="exact_int")
    bias = np.arange(333, dtype=np.float32) * 0.5
    assert np.array_equal(run(bsr, x, bias=bias).astype(np.float64), O.gemv(bsr, x, bias=bias))


@pytest.mark.parametrize("bits", [4, 2])
def test_onehot_columns_exact(bits):
    """x = e_j: y = W_hat[:, j] exactly (z multiple of 1/128, |z| < 16)."""
    bsr = synth.make_layer(21 + bits, 512, 1024, bits=bits, sparsity=0.5, mode="onehot_safe")
    W = O.decompress(bsr)
    L = gqsa.Layer(bsr)
    x = synth.make_x(31, 8, 1024, mode="onehot")
    y = run(bsr, x, layer=L)
    cols = np.argmax(x.view(np.float16) != 0, axis=1)
    for b in range(8):
        assert np.array_equal(y[b].astype(np.float64), W[:, cols[b]])


# ------------------------------------------------------------------ realistic
REAL_CASES = [
    (4096, 4096, 4, 0.5, "uniform", 1),
    (1024, 4096, 4, 0.5, "uniform", 2),
    (4096, 4096, 2, 0.5, "uniform", 1),
    (4096, 4096, 4, 0.3, "uniform", 8),
    (2048, 5120, 4, 0.5, "row_balanced", 4),
    (1024, 2048, 4, 0.5, "skewed", 1),
    (4096, 4096, 8, 0.5, "uniform", 1),
    (2048, 14336, 8, 0.5, "uniform", 2),
]


@pytest.mark.parametrize("rows,cols,bits,sp,mask,B", REAL_CASES)
def test_realistic_tolerance_gates(rows, cols, bits, sp, mask, B):
    seed = synth.seed_for(f"real/{rows}/{cols}/{bits}/{sp}/{mask}/{B}")
    bsr = synth.make_layer(seed, rows, cols, bits=bits, sparsity=sp, mask=mask)
    x = synth.make_x(seed + 1, B, cols)
    y = run(bsr, x)
    check_gates(y, O.gemv(bsr, x), abs_bound(bsr, x), f"{rows}x{cols} W{bits} S{sp} {mask} B{B}")


def test_determinism_and_batch_consistency():
    bsr = synth.make_layer(41, 4096, 4096, sparsity=0.5)
    x = synth.make_x(42, 4, 4096)
    L = gqsa.Layer(bsr)
    first = run(bsr, x, layer=L)
    for _ in range(20):
        assert np.array_equal(run(bsr, x, layer=L), first)
    # the batch-1 GEMV (its own grid, hence its own fp32 summation order)
    # agrees with row 0 of the batched GEMM within the gates
    y1 = run(bsr, x[:1], layer=L)
    check_gates(y1, O.gemv(bsr, x[:1]), abs_bound(bsr, x[:1]), "B1 vs oracle")
    check_gates(y1, first[:1].astype(np.float64), abs_bound(bsr, x[:1]), "B1 vs B4 row 0")


def test_hostio_end_to_end_path():
    bsr = synth.make_layer(51, 1024, 2048, sparsity=0.5, mode="exact_int")
    x = synth.make_x(52, 3, 2048, mode="exact_int")
    L = gqsa.Layer(bsr)
    hX = torch.from_numpy(x).view(torch.float16).pin_memory()
    hY = torch.empty(3, 1024, dtype=torch.float32).pin_memory()
    stage = torch.empty(gqsa.hostio_stage_size(L.desc, 3), dtype=torch.uint8, device="cuda")
    n0 = gqsa.launch_count()
    gqsa.gemm_hostio(L.desc, L.blob, hX, hY, stage, L.ws)
    torch.cuda.synchronize()
    assert gqsa.launch_count() == n0 + 1
    assert np.array_equal(hY.numpy().astype(np.float64), O.gemv(bsr, x))


def test_multi_hostio_end_to_end_path():
    """gqsa_gemm_multi_hostio: one H2D copy of concatenated inputs, ONE grouped
    launch for the layers, one D2H copy of concatenated outputs (bench.py's e2e path)."""
    shapes = [(300, 1024), (77, 208), (1024, 4096)]
    for B in (1, 2):
        layers, xs, refs, xs2, refs2 = [], [], [], [], []
        for i, (n, k) in enumerate(shapes):
            seed = synth.seed_for(f"multi/{i}/{n}/{k}/{B}")
            bsr = synth.make_layer(seed, n, k, sparsity=0.5, mode="exact_int")
            x = synth.make_x(seed + 1, B, k, mode="exact_int")
            x2 = synth.make_x(seed + 2, B, k, mode="exact_int")
            layers.append(gqsa.Layer(bsr))
            xs.append(x.reshape(-1))
            xs2.append(x2.reshape(-1))
            refs.append(O.gemv(bsr, x))
            refs2.append(O.gemv(bsr, x2))
        descs = [L.desc for L in layers]
        hX = torch.from_numpy(np.concatenate(xs)).view(torch.float16).pin_memory()
        hY = torch.full((sum(B * n for n, _ in shapes),), float("nan"), dtype=torch.float32).pin_memory()
        stage = torch.empty(gqsa.multi_hostio_stage_size(descs, B), dtype=torch.uint8, device="cuda")
        # default stream once, then a side stream three times (fresh host inputs each time)
        side = torch.cuda.Stream()
        for k, st in enumerate([None, side, side, side]):
            hX.copy_(torch.from_numpy(np.concatenate(xs) if k % 2 == 0 else np.concatenate(xs2)).view(torch.float16))
            hY.fill_(float("nan"))
            n0 = gqsa.launch_count()
            gqsa.gemm_multi_hostio(descs, [L.blob for L in layers], hX, hY, stage, [layers[0].ws], batch=B,
                                   stream=st)
            assert gqsa.launch_count() == n0 + 1
            torch.cuda.synchronize()
            got = hY.numpy().astype(np.float64)
            off = 0
            for (n, _), ref, ref2 in zip(shapes, refs, refs2):
                assert np.array_equal(got[off:off + B * n].reshape(B, n), ref if k % 2 == 0 else ref2), (k, n)
                off += B * n


def test_argument_errors():
    bsr = synth.make_layer(61, 64, 256, sparsity=0.5)
    L = gqsa.Layer(bsr)
    X = torch.zeros(9, 256, dtype=torch.float16, device="cuda")
    with pytest.raises(gqsa.GQSAError) as e:
        L.gemm(X)  # B = 9 > 8
    assert e.value.status == -1
    small = torch.zeros(8, dtype=torch.uint8, device="cuda")
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.gemv(L.desc, L.blob, X[0], torch.empty(64, device="cuda"), None, small)
    assert e.value.status == -4
    with pytest.raises(gqsa.GQSAError) as e:  # misaligned x
        gqsa.gemv(L.desc, L.blob, X.view(-1)[1:257], torch.empty(64, device="cuda"), None, L.ws)
    assert e.value.status == -4


def test_launch_plan_batch_split():
    """x (+ column sums + zero block) must fit in shared memory: larger batches
    split into several launches; one CTA per SM."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for rows, cols, B, launches in ((4096, 4096, 1, 1), (4096, 4096, 8, 1), (4096, 14336, 1, 1),
                                    (4096, 14336, 4, 1), (4096, 14336, 8, 2), (64, 28672, 4, 2)):
        bsr = synth.make_layer(rows + cols + B, rows, cols, sparsity=0.5)
        _, d = gqsa.pack(bsr)
        p = gqsa.launch_plan(d, B)
        assert p.launches == launches, (rows, cols, B, p.launches)
        assert p.batch_per_launch * p.launches >= B and p.smem_bytes <= 227 * 1024
        assert p.grid <= sms and p.ctas_per_sm == 1 and p.coresident == 0
    n0 = gqsa.launch_count()
    L = gqsa.Layer(synth.make_layer(5, 256, 14336, sparsity=0.5))
    L.gemm(torch.zeros(8, 14336, dtype=torch.float16, device="cuda"))
    torch.cuda.synchronize()
    assert gqsa.launch_count() == n0 + 2


def test_launch_plan_is_persistent_stream_k():
    bsr = synth.make_layer(71, 14336, 4096, sparsity=0.5)
    _, d = gqsa.pack(bsr)
    p = gqsa.launch_plan(d, 1)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert p.active_warps == min(d.num_tiles, p.grid * p.warps_per_cta)
    assert p.grid <= sms and p.x_in_smem == 1


@pytest.mark.parametrize("rows,cols,B,P,f16", [(1000, 2048, 1, 2, False), (4096, 4096, 2, 4, False),
                                               (2048, 14336, 8, 2, False), (512, 1024, 3, 8, True)])
def test_fused_allgather_epilogue_simulated_ranks(rows, cols, B, P, f16):
    """gqsa_gemm_allgather on one GPU with P simulated ranks: each rank's row
    shard stores its rows into ALL P full-length outputs (here local buffers
    standing for the peers' NVLink-mapped y); every output must equal the
    oracle's full result exactly (exact-integer mode; fp16 output = RNE)."""
    seed = synth.seed_for(f"allgather/{rows}/{cols}/{B}/{P}")
    bsr = synth.make_layer(seed, rows, cols, sparsity=0.5, mode="exact_int")
    x = synth.make_x(seed + 1, B, cols, mode="exact_int")
    X = torch.from_numpy(x).view(torch.float16).cuda()
    dt = torch.float16 if f16 else torch.float32
    Ys = [torch.full((B, rows), float("nan"), dtype=dt, device="cuda") for _ in range(P)]
    for r in range(P):
        lo, hi = synth.shard_rows(rows, P, r)
        blob, desc = gqsa.pack(bsr, lo, hi)
        ws = torch.zeros(gqsa.workspace_size(desc, B), dtype=torch.uint8, device="cuda")
        gqsa.gemm_allgather(desc, torch.from_numpy(blob).cuda(), X, Ys, row_offset=lo, ws=ws)
    torch.cuda.synchronize()
    ref = O.gemv(bsr, x)
    for Y in Ys:
        got = Y.cpu().numpy()
        if f16:
            assert np.array_equal(got, ref.astype(np.float16))
        else:
            assert np.array_equal(got.astype(np.float64), ref)


def test_multicast_allgather_argument_contract():
    """gqsa_gemm_allgather_multicast (NVLS multimem.st epilogue) validates its
    arguments like gqsa_gemm_allgather and refuses fp16 output (multimem.st
    has no 16-bit scalar form).  Its stores need a real multicast object of
    >= 2 GPUs, which a one-GPU box cannot create, so only the
    contract is exercised here."""
    bsr = synth.make_layer(91, 256, 512, sparsity=0.5)
    blob, desc = gqsa.pack(bsr)
    d_blob = torch.from_numpy(blob).cuda()
    X = torch.zeros(1, 512, dtype=torch.float16, device="cuda")
    ws = torch.zeros(gqsa.workspace_size(desc, 1), dtype=torch.uint8, device="cuda")
    fake_mc = torch.zeros(1, 256, dtype=torch.float32, device="cuda").data_ptr()
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.gemm_allgather_multicast(desc, d_blob, X, fake_mc, ldy=256, row_offset=0, out_f16=True, ws=ws)
    assert e.value.status == -3
    with pytest.raises(gqsa.GQSAError) as e:  # shard rows beyond ldy
        gqsa.gemm_allgather_multicast(desc, d_blob, X, fake_mc, ldy=255, row_offset=0, ws=ws)
    assert e.value.status == -1
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.gemm_allgather_multicast(desc, d_blob, X, 0, ldy=256, row_offset=0, ws=ws)
    assert e.value.status == -4
    with pytest.raises(gqsa.GQSAError) as e:  # misaligned multicast address
        gqsa.gemm_allgather_multicast(desc, d_blob, X, fake_mc + 2, ldy=256, row_offset=0, ws=ws)
    assert e.value.status == -4


def test_pdl_dependent_launch_chain_reads_producer_output():
    """Back-to-back launches where launch k reads, as its x, the fp16 output
    launch k-1 just wrote (Programmatic Dependent Launch: weights are
    prefetched before griddepcontrol.wait, x only after it).  Inputs start as
    NaN, so a launch that read x early would produce NaN; every layer must
    match the oracle on the activations its producer left, in a CUDA graph
    replayed several times."""
    dims = [4096, 1024, 4096, 2048, 4096, 14336, 4096]
    bsrs = [synth.make_layer(synth.seed_for(f"pdl/{i}"), dims[i + 1], dims[i], sparsity=0.5)
            for i in range(len(dims) - 1)]
    layers = [gqsa.Layer(b) for b in bsrs]
    bufs = [torch.full((1, d), float("nan"), dtype=torch.float16, device="cuda") for d in dims]
    x0 = synth.make_x(77, 1, dims[0])
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i, L in enumerate(layers):
            gqsa.gemm_ex(L.desc, L.blob, bufs[i], bufs[i + 1], ws=L.ws, stream=s)
    for rep in range(3):
        for b in bufs[1:]:
            b.fill_(float("nan"))
        bufs[0].copy_(torch.from_numpy(x0).view(torch.float16))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        for i, b in enumerate(bsrs):
            xin = bufs[i].cpu().numpy().view(np.uint16)
            y = bufs[i + 1].cpu().numpy().astype(np.float64)
            assert np.isfinite(y).all(), (rep, i)
            ref = O.gemv(b, xin)
            assert np.all(np.abs(y - ref) <= 2.0 ** -10 * np.abs(ref) + 1e-5 * abs_bound(b, xin)), (rep, i)


def test_concurrent_streams_share_one_blob():
    """One packed blob used by two streams at once, each with its own
    workspace (include/gqsa.h ownership rules): results stay bit-exact."""
    bsr = synth.make_layer(91, 2048, 4096, sparsity=0.5, mode="exact_int")
    blob, desc = gqsa.pack(bsr)
    d_blob = torch.from_numpy(blob).cuda()
    xs = [synth.make_x(92 + k, 2, 4096, mode="exact_int") for k in range(2)]
    X = [torch.from_numpy(x).view(torch.float16).cuda() for x in xs]
    refs = [O.gemv(bsr, x) for x in xs]
    streams = [torch.cuda.Stream() for _ in range(2)]
    wss = [torch.zeros(gqsa.workspace_size(desc, 2), dtype=torch.uint8, device="cuda") for _ in range(2)]
    Ys = [[torch.empty(2, 2048, dtype=torch.float32, device="cuda") for _ in range(20)] for _ in range(2)]
    torch.cuda.synchronize()
    for it in range(20):
        for k in range(2):
            gqsa.gemm_smallbatch(desc, d_blob, X[k], Ys[k][it], None, wss[k], stream=streams[k])
    torch.cuda.synchronize()
    for k in range(2):
        for Y in Ys[k]:
            assert np.array_equal(Y.cpu().numpy().astype(np.float64), refs[k])


G_EXACT = [
    # rows, cols, G, sparsity, mask, B
    (300, 1024, 8, 0.5, "uniform", 1),
    (77, 264, 8, 0.2, "uniform", 2),
    (512, 2048, 8, 0.5, "skewed", 3),
    (1024, 4096, 8, 0.5, "uniform", 8),
    (300, 1024, 32, 0.5, "uniform", 1),
    (77, 224, 32, 0.2, "uniform", 2),
    (512, 2048, 32, 0.5, "row_balanced", 4),
    (1024, 4096, 32, 0.5, "uniform", 8),
    (3, 16384, 32, 0.5, "uniform", 1),
    (2048, 14336, 32, 0.5, "uniform", 2),
]


@pytest.mark.parametrize("rows,cols,G,sp,mask,B", G_EXACT)
def test_group_size_8_32_exact(rows, cols, G, sp, mask, B):
    """W4 at G = 8 and G = 32 (the group-size sweep): bit-exact in exact-integer
    mode, Stream-K and Slice-K."""
    seed = synth.seed_for(f"gexact/{rows}/{cols}/{G}/{sp}/{mask}/{B}")
    bsr = synth.make_layer(seed, rows, cols, G=G, bits=4, sparsity=sp, mask=mask, mode="exact_int")
    x = synth.make_x(seed + 1, B, cols, mode="exact_int")
    ref = O.gemv(bsr, x)
    L = gqsa.Layer(bsr)
    X = torch.from_numpy(x).view(torch.float16).cuda()
    for part in (gqsa.PARTITION_STREAM_K, gqsa.PARTITION_SLICE_K):
        y = L.gemm(X, partition=part)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy().astype(np.float64), ref), part


@pytest.mark.parametrize("G", [8, 32])
def test_group_size_realistic_gates(G):
    bsr = synth.make_layer(synth.seed_for(f"greal/{G}"), 4096, 4096, G=G, bits=4, sparsity=0.5)
    x = synth.make_x(3, 2, 4096)
    y = run(bsr, x)
    check_gates(y, O.gemv(bsr, x), abs_bound(bsr, x), f"G{G}")
