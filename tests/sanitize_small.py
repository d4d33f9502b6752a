"""Small launches of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): gemv, small-batch GEMM (batch split), Slice-K,
fp16 output, grouped launch (whole-SM and pipelined), LAYOUT-TC, fused
all-gather, whole-GPU launches (CTA-level fix-up, slice-aligned CTA ranges).  Exits non-zero on a
mismatch against the oracle (exact-integer mode)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import gqsa_oracle as O  # noqa: E402
from paper_2412_17560_b200 import gqsa, synth  # noqa: E402

ok = True
for rows, cols, bits, B, mask in ((300, 1024, 4, 1, "uniform"), (77, 208, 2, 3, "uniform"),
                                  (512, 2048, 4, 2, "skewed"), (64, 4096, 8, 1, "uniform"),
                                  (128, 14336, 4, 8, "uniform"), (5, 64, 4, 1, "uniform"),
                                  # every CTA busy: slices cross CTA boundaries (CTA-level fix-up at
                                  # B = 1, slice-aligned CTA ranges at B >= 2)
                                  (4096, 4096, 4, 1, "uniform"), (2048, 4096, 4, 3, "skewed")):
    bsr = synth.make_layer(rows + cols, rows, cols, bits=bits, sparsity=0.5, mask=mask, mode="exact_int")
    x = synth.make_x(rows, B, cols, mode="exact_int")
    L = gqsa.Layer(bsr)
    X = torch.from_numpy(x).view(torch.float16).cuda()
    ref = O.gemv(bsr, x)
    for part in (gqsa.PARTITION_STREAM_K, gqsa.PARTITION_SLICE_K):
        y = L.gemm(X, partition=part).cpu().numpy().astype(np.float64)
        ok &= np.array_equal(y, ref)
    y16 = L.gemm(X, out_dtype=torch.float16, partition=gqsa.PARTITION_SLICE_K).cpu().numpy()
    ok &= np.array_equal(y16, ref.astype(np.float16))
    Y = torch.empty(B, rows, dtype=torch.float32, device="cuda")
    Y2 = torch.empty(B, rows, dtype=torch.float32, device="cuda")
    for x_ready in (False, True):  # x_ready, B <= 2: the pipelined launch (deferred writes)
        Y.fill_(float("nan"))
        Y2.fill_(float("nan"))
        for _ in range(3):  # back to back on one stream, sharing the workspace
            gqsa.gemm_grouped([(L.desc, L.blob, X, Y, None), (L.desc, L.blob, X, Y2, None)], L.ws, x_ready=x_ready)
        ok &= np.array_equal(Y.cpu().numpy().astype(np.float64), ref)
        ok &= np.array_equal(Y2.cpu().numpy().astype(np.float64), ref)
    if bits == 4 and B >= 2:  # LAYOUT-TC (tensor-core small batch)
        Lt = gqsa.Layer(bsr, layout=gqsa.LAYOUT_TC)
        ok &= np.array_equal(Lt.gemm(X).cpu().numpy().astype(np.float64), ref)
    Ys = [torch.zeros(B, rows, dtype=torch.float32, device="cuda") for _ in range(2)]
    for r in range(2):
        lo, hi = synth.shard_rows(rows, 2, r)
        blob, desc = gqsa.pack(bsr, lo, hi)
        wsr = torch.zeros(gqsa.workspace_size(desc, B), dtype=torch.uint8, device="cuda")
        gqsa.gemm_allgather(desc, torch.from_numpy(blob).cuda(), X, Ys, row_offset=lo, ws=wsr)
    for Yk in Ys:
        ok &= np.array_equal(Yk.cpu().numpy().astype(np.float64), ref)
    torch.cuda.synchronize()
print("sanitize_small:", "ok" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
