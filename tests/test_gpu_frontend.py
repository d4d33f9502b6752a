"""GPU parity on layers produced by the method's own compression front-end
(Eq. 4 saliency + exact-count group pruning + Eq. 1-2, frontend.compress):
row-skewed masks with empty and full rows.  The GEMV must meet the gates
against the fp64 oracle on the same BSR (Stream-K and Slice-K)."""
import numpy as np
import pytest

from oracle import gqsa_oracle as O
from paper_2412_17560_b200 import frontend, gqsa, synth
from tests.parity import abs_bound, check_gates

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("rows,cols,bits,sp,B", [(2048, 4096, 4, 0.5, 1), (1024, 14336, 2, 0.5, 2),
                                                 (4096, 1024, 8, 0.3, 1), (512, 4096, 4, 0.8, 4)])
def test_saliency_masks_gates(rows, cols, bits, sp, B):
    seed = synth.seed_for(f"gpu-frontend/{rows}x{cols}/{bits}/{sp}")
    W = synth.make_dense(seed, rows, cols)
    d = frontend.hessian_inv_diag(synth.make_calib(seed + 1, 128, cols), device="cuda")
    bsr = frontend.compress(W, d, sp, bits)
    lens = np.diff(bsr["row_index"])
    assert lens.max() >= 1.4 * lens.mean()  # the saliency masks are row-skewed
    x = synth.make_x(seed + 2, B, cols)
    L = gqsa.Layer(bsr)
    X = torch.from_numpy(x).view(torch.float16).cuda()
    ref = O.gemv(bsr, x)
    A = abs_bound(bsr, x)
    for part in (gqsa.PARTITION_STREAM_K, gqsa.PARTITION_SLICE_K):
        y = L.gemm(X, partition=part)
        torch.cuda.synchronize()
        check_gates(y.cpu().numpy(), ref, A, f"saliency {rows}x{cols} W{bits} S{sp} part{part}")
