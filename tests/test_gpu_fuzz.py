"""Randomised exact-integer parity (GPU): many small random shapes, batches,
bit widths, sparsities, masks and both partitions, each bit-exact against the
oracle.  Seeded, so a failure is reproducible from its parameters."""
import numpy as np
import pytest

from oracle import gqsa_oracle as O
from paper_2412_17560_b200 import gqsa, synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        bits = int(rng.choice([2, 4, 8]))
        kmax = 4096 if bits == 8 else 12288  # exact-int needs the partial sums < 2^23 (W8: 255*2*4*K)
        out.append((int(rng.integers(1, 1500)), 16 * int(rng.integers(1, kmax // 16 + 1)), bits,
                    float(rng.choice([0.0, 0.2, 0.5, 0.8, 0.95])), str(rng.choice(["uniform", "row_balanced", "skewed"])),
                    int(rng.integers(1, 9)), int(rng.integers(0, 2))))
    return out


@pytest.mark.parametrize("rows,cols,bits,sp,mask,B,part", _cases(60, 2024) + _cases(90, 7))
def test_fuzz_exact_integer(rows, cols, bits, sp, mask, B, part):
    seed = synth.seed_for(f"fuzz/{rows}/{cols}/{bits}/{sp}/{mask}/{B}")
    bsr = synth.make_layer(seed, rows, cols, bits=bits, sparsity=sp, mask=mask, mode="exact_int")
    x = synth.make_x(seed + 1, B, cols, mode="exact_int")
    L = gqsa.Layer(bsr)
    X = torch.from_numpy(x).view(torch.float16).cuda()
    y = L.gemm(X, partition=part)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy().astype(np.float64), O.gemv(bsr, x))
