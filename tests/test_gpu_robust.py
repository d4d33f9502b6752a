"""Forward progress and isolation of the cross-warp fix-up: the
last-arriver protocol never waits for a warp that has not already published,
so launches complete -- bit-exactly -- whatever else occupies the SMs:

three streams run GEMVs and grouped launches concurrently (each stream with
its own workspace) while a fourth stream runs long dense matmuls that hold
SMs, so the GEMV grids are not all co-resident; every result equals the fp64
oracle bit for bit (exact-integer mode) and every workspace is left zero.
"""
import numpy as np
import pytest

from oracle import gqsa_oracle as O
from paper_2412_17560_b200 import gqsa, synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.init()


@pytest.mark.parametrize("x_ready", [False, True])
def test_three_streams_and_a_side_kernel_bit_exact(x_ready):
    """x_ready: every launch is a pipelined one (part of every SM, deferred
    writes, consecutive launches of a stream overlapping and sharing its
    workspace) -- the same guarantees must hold."""
    shapes = [(4096, 4096), (1024, 4096), (2048, 14336)]
    layers, xs, refs = [], [], []
    for i, (n, k) in enumerate(shapes):
        bsr = synth.make_layer(synth.seed_for(f"robust/{i}"), n, k, sparsity=0.5, mode="exact_int")
        x = synth.make_x(i, 2, k, mode="exact_int")
        layers.append(gqsa.Layer(bsr))
        xs.append(torch.from_numpy(x).view(torch.float16).cuda())
        refs.append(O.gemv(bsr, x))
    streams = [torch.cuda.Stream() for _ in range(3)]
    side = torch.cuda.Stream()
    wss = [torch.zeros_like(L.ws) for L in layers]
    A = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    outs = [[torch.empty(2, n, dtype=torch.float32, device="cuda") for _ in range(12)] for n, _ in shapes]
    grouped_out = [[torch.empty(2, n, dtype=torch.float32, device="cuda") for n, _ in shapes] for _ in range(4)]
    gws = torch.zeros_like(layers[0].ws)
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        for _ in range(4):
            A = A @ A  # holds most SMs for milliseconds while the GEMVs run
            A = A / A.abs().amax()
    for it in range(12):
        for k in range(3):
            gqsa.gemm_ex(layers[k].desc, layers[k].blob, xs[k], outs[k][it], ws=wss[k], stream=streams[k],
                         x_ready=x_ready)
        if it % 3 == 0:
            with torch.cuda.stream(streams[it % 3]):
                gqsa.gemm_grouped([(L.desc, L.blob, xs[k], grouped_out[it // 3][k], None)
                                   for k, L in enumerate(layers)], gws, stream=streams[it % 3], x_ready=x_ready)
    torch.cuda.synchronize()
    for k in range(3):
        for Y in outs[k]:
            assert np.array_equal(Y.cpu().numpy().astype(np.float64), refs[k])
        assert int(wss[k].count_nonzero()) == 0
    for go in grouped_out:
        for k in range(3):
            assert np.array_equal(go[k].cpu().numpy().astype(np.float64), refs[k])
    assert int(gws.count_nonzero()) == 0
