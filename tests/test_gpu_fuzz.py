"""Randomised exact-integer parity (GPU): many small random shapes, batches,
bit widths, group sizes (W4: 8 / 16 / 32), sparsities, masks and both partitions, each bit-exact against the
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
        G = int(rng.choice([8, 16, 16, 32])) if bits == 4 else 16
        out.append((int(rng.integers(1, 1500)), 32 * int(rng.integers(1, kmax // 32 + 1)), bits,
                    float(rng.choice([0.0, 0.2, 0.5, 0.8, 0.95])), str(rng.choice(["uniform", "row_balanced", "skewed"])),
                    int(rng.integers(1, 9)), int(rng.integers(0, 2)), G))
    return out


@pytest.mark.parametrize("rows,cols,bits,sp,mask,B,part,G", _cases(60, 2024) + _cases(90, 7))
def test_fuzz_exact_integer(rows, cols, bits, sp, mask, B, part, G):
    seed = synth.seed_for(f"fuzz/{rows}/{cols}/{bits}/{sp}/{mask}/{B}/{G}")
    bsr = synth.make_layer(seed, rows, cols, G=G, bits=bits, sparsity=sp, mask=mask, mode="exact_int")
    x = synth.make_x(seed + 1, B, cols, mode="exact_int")
    L = gqsa.Layer(bsr)
    X = torch.from_numpy(x).view(torch.float16).cuda()
    y = L.gemm(X, partition=part)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy().astype(np.float64), O.gemv(bsr, x))
