"""Offline compression front-end (product side): dense layer -> plain BSR.

PAPER.md:74-93 [§3.1 Eq. 4, §3.2 / Fig. 3] and 50-63 [Eq. 1-2]; SURVEY §8(f)
NEXT-4.  Two steps:

* :func:`hessian_inv_diag` -- the layer-wise Hessian proxy H = (2/N) X^T X
  + lambda I (lambda = damping * mean diag; the paper does not define H,
  DESIGN.md reading R16) and the diagonal of its inverse, with torch's dense
  fp64 Cholesky (a library factorisation, on the GPU when one is given);
* :func:`compress` -- Eq. 4 saliency, group means, exact-count pruning and the
  Eq. 1-2 quantizer, all in the C ABI (``gqsa_compress``, csrc/gqsa_compress.cpp).

The result feeds :func:`paper_2412_17560_b200.gqsa.pack` unchanged.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import gqsa


def hessian_inv_diag(X, damping: float = 0.01, device=None) -> np.ndarray:
    """diag(H^-1), H = (2/N) X^T X + damping * mean(diag) * I, in fp64.

    X: calibration inputs [N][K] (numpy or torch).  Returns float64 [K].
    """
    import torch
    Xt = torch.as_tensor(np.asarray(X) if not isinstance(X, torch.Tensor) else X)
    Xt = Xt.to(device=device or "cpu", dtype=torch.float64)
    if Xt.ndim != 2 or Xt.shape[0] < 1:
        raise ValueError("hessian_inv_diag needs >= 1 calibration sample [N][K]")
    n = Xt.shape[0]
    H = (2.0 / n) * (Xt.T @ Xt)
    H = H + damping * torch.diagonal(H).mean() * torch.eye(H.shape[0], dtype=H.dtype, device=H.device)
    L = torch.linalg.cholesky(H)
    return torch.diagonal(torch.cholesky_inverse(L)).cpu().numpy().copy()


def compress(W, hinv_diag, sparsity: float, bits: int = 4, G: int = 16,
             return_saliency: bool = False):
    """gqsa_compress: plain-BSR dict of the kept, quantized groups of W.

    W: float32 [rows][cols]; hinv_diag: float64 [cols].  With
    ``return_saliency`` also returns the group scores [rows][cols/G] (fp64).
    """
    W = np.ascontiguousarray(W, dtype=np.float32)
    d = np.ascontiguousarray(hinv_diag, dtype=np.float64)
    rows, cols = W.shape
    if d.shape != (cols,):
        raise ValueError("hinv_diag must have cols entries")
    L = gqsa.lib()
    nnzg = ctypes.c_int64(0)
    gqsa._check(L.gqsa_compress_nnzg(rows, cols, G, float(sparsity), ctypes.byref(nnzg)), "gqsa_compress_nnzg")
    n = nnzg.value
    out = {
        "row_index": np.zeros(rows + 1, np.int32),
        "group_cols": np.zeros(max(n, 1), np.uint16),
        "codes": np.zeros(max((n * G * bits + 7) // 8, 1), np.uint8),
        "scales_f16": np.zeros(max(n, 1), np.uint16),
        "zeros_f16": np.zeros(max(n, 1), np.uint16),
    }
    b = gqsa.BSR(rows, cols, G, bits, n, out["row_index"].ctypes.data, out["group_cols"].ctypes.data,
                 out["codes"].ctypes.data, out["scales_f16"].ctypes.data, out["zeros_f16"].ctypes.data)
    sal = np.zeros((rows, cols // G), np.float64) if return_saliency else None
    gqsa._check(L.gqsa_compress(W.ctypes.data, rows, cols, G, bits, d.ctypes.data, float(sparsity),
                                ctypes.byref(b), sal.ctypes.data if sal is not None else None),
                "gqsa_compress")
    bsr = {"rows": rows, "cols": cols, "group_size": G, "bits": bits, "nnzg": n,
           "row_index": out["row_index"], "group_cols": out["group_cols"][:n],
           "codes": out["codes"][:(n * G * bits + 7) // 8],
           "scales_f16": out["scales_f16"][:n], "zeros_f16": out["zeros_f16"][:n]}
    return (bsr, sal) if return_saliency else bsr


def concat_rows(bsrs) -> dict:
    """Stack plain-BSR layers with the same K, G and bits along the output
    dimension (rows of bsrs[0] first): the merged q/k/v or gate/up matrix of a
    decoder layer, so one GEMV launch serves what were several (production
    servers merge them the same way; tools/stack_bench.py "merged").  Pure
    data movement: codes are re-packed bit-exactly, row offsets rebased."""
    b0 = bsrs[0]
    G, n, K = int(b0["group_size"]), int(b0["bits"]), int(b0["cols"])
    for b in bsrs:
        if (int(b["group_size"]), int(b["bits"]), int(b["cols"])) != (G, n, K):
            raise ValueError("concat_rows: layers differ in K, G or bits")
    rows = sum(int(b["rows"]) for b in bsrs)
    ri = [np.zeros(1, np.int64)]
    off = 0
    bits = []
    for b in bsrs:
        r = np.asarray(b["row_index"], np.int64)
        ri.append(r[1:] + off)
        off += int(r[-1])
        nb = int(b["nnzg"]) * G * n
        bits.append(np.unpackbits(np.asarray(b["codes"], np.uint8), bitorder="little")[:nb])
    allbits = np.concatenate(bits) if bits else np.zeros(0, np.uint8)
    pad = (-allbits.size) % 8
    if pad:
        allbits = np.concatenate([allbits, np.zeros(pad, np.uint8)])
    return {
        "rows": rows, "cols": K, "group_size": G, "bits": n, "nnzg": off,
        "row_index": np.concatenate(ri).astype(np.int32),
        "group_cols": np.concatenate([np.asarray(b["group_cols"], np.uint16) for b in bsrs]),
        "codes": np.packbits(allbits, bitorder="little"),
        "scales_f16": np.concatenate([np.asarray(b["scales_f16"], np.uint16) for b in bsrs]),
        "zeros_f16": np.concatenate([np.asarray(b["zeros_f16"], np.uint16) for b in bsrs]),
    }
