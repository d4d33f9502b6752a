"""GQSA compression front-end oracle -- TEST INFRASTRUCTURE ONLY.

Plain fp64 reference for the upstream step of the method that turns a dense
layer into the BSR the hot path consumes (SURVEY §8(a) row a0 and §8(f)
NEXT-4): Hessian saliency, group ranking, exact-count group pruning and
per-group quantization.  Only ``tests/`` may import this module; it shares no
code with the product front-end (``paper_2412_17560_b200/frontend.py`` and
``csrc/gqsa_compress.cpp``) and imports only numpy, the standard library and
its sibling ``gqsa_oracle`` (for the Eq. 1-2 quantizer).

Steps, in the paper's order (PAPER.md:74-93 [§3.1 Eq. 4, §3.2, Fig. 3]):

  1. estimate_hessian  H = (2/N) sum_k x_k x_k^T + lambda I,
                       lambda = 0.01 * mean(diag) before damping
                       (the paper does not define H: DESIGN.md reading R16,
                       SPEC.md:191 / 226-227)
  2. weight_saliency   s_{r,c} = W[r,c]^2 / ([H^-1]_{cc})^2           (Eq. 4)
  3. group_saliency    mean of s over each run of G columns of a row,
                       summed in ascending t (Fig. 3 caption "average
                       saliency metrics within each group")
  4. select_groups     prune exactly floor(S * total) groups with the lowest
                       score in the layer; ties -> lower (row, group) index
                       pruned first (reading R13/R17)
  5. build_gqs         Eq. 1-2 per kept group (gqsa_oracle.compute_qparams,
                       quantize_group, fp64), codes packed low bits first;
                       s and z stored as fp16 (RNE of the fp64 values,
                       reading R7); row_index / group_cols as in PAPER.md:95-101.

Pins (tests/test_frontend.py): SPEC.md:197 (x = e_1 -> H = [[2,0],[0,0]]
before damping), SPEC.md:206 (H = diag(a, b) -> s = W^2 a^2)
(group mean [1,1,3,3], G = 2 -> [1, 3]), SPEC.md:339 ([[1,2],[3,4]] at S = 0.5
prunes row 0), tie rule, brute-force selection by exhaustive ranking,
nestedness across sparsities, Eq. 4 homogeneity, the PAPER.md:101 topology,
and the all-kept round trip |W_hat - W| <= s/2.
"""
from __future__ import annotations

import math

import numpy as np

from oracle import gqsa_oracle as O

__all__ = ["estimate_hessian", "hessian_inv_diag", "weight_saliency", "group_saliency",
           "select_groups", "build_gqs", "compress_layer"]


def estimate_hessian(X, damping: float = 0.01) -> np.ndarray:
    """H = (2/N) sum_k x_k x_k^T + lambda I with lambda = damping * mean(diag(H0)).

    X: calibration inputs [N][K] (any float dtype), N >= 1.
    """
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] < 1:
        raise ValueError("estimate_hessian needs >= 1 calibration sample")
    n, k = X.shape
    H = np.zeros((k, k))
    for i in range(n):                 # sum of outer products, sample by sample
        H += np.outer(X[i], X[i])
    H *= 2.0 / n
    lam = damping * float(np.mean(np.diag(H)))
    return H + lam * np.eye(k)


def hessian_inv_diag(H) -> np.ndarray:
    """diag(H^-1) via a dense inverse (a library routine)."""
    return np.diag(np.linalg.inv(np.asarray(H, dtype=np.float64))).copy()


def weight_saliency(W, hinv_diag) -> np.ndarray:
    """Eq. 4: s_i = w_i^2 / [H^-1]_ii^2 (denominator squared as printed)."""
    W = np.asarray(W, dtype=np.float64)
    d = np.asarray(hinv_diag, dtype=np.float64)
    if W.shape[1] != d.shape[0]:
        raise ValueError("W.cols != dim(H)")
    return (W * W) / (d * d)[None, :]


def group_saliency(per_weight, G: int) -> np.ndarray:
    """Mean over each contiguous run of G columns, summed t = 0..G-1 in order."""
    s = np.asarray(per_weight, dtype=np.float64)
    rows, cols = s.shape
    if cols % G:
        raise ValueError("cols % G != 0")
    g = s.reshape(rows, cols // G, G)
    acc = np.zeros((rows, cols // G))
    for t in range(G):
        acc = acc + g[:, :, t]
    return acc / G


def select_groups(per_group, sparsity: float) -> np.ndarray:
    """keep[r][g]: prune exactly floor(sparsity * total) lowest-score groups of
    the layer, ties by (row, group) lexicographic order (lower index first)."""
    sc = np.asarray(per_group, dtype=np.float64)
    if not (0.0 <= sparsity < 1.0):
        raise ValueError("sparsity must be in [0, 1)")
    flat = sc.reshape(-1)
    n_prune = int(math.floor(sparsity * flat.size))
    order = np.lexsort((np.arange(flat.size), flat))  # by score, then index
    keep = np.ones(flat.size, dtype=bool)
    keep[order[:n_prune]] = False
    return keep.reshape(sc.shape)


def build_gqs(W, keep, G: int, bits: int) -> dict:
    """Plain BSR of the kept groups, Eq. 1-2 per group, fp16 s/z (RNE)."""
    W = np.asarray(W, dtype=np.float32).astype(np.float64)
    rows, cols = W.shape
    keep = np.asarray(keep, dtype=bool)
    if keep.shape != (rows, cols // G) or cols % G:
        raise ValueError("shape mismatch")
    if bits not in (2, 4, 8):
        raise ValueError("bits must be 2, 4 or 8")
    row_index = [0]
    group_cols, codes, s16, z16 = [], [], [], []
    for r in range(rows):
        for g in range(cols // G):
            if not keep[r, g]:
                continue
            grp = W[r, g * G:(g + 1) * G]
            s, z = O.compute_qparams(grp, bits)
            codes.extend(O.quantize_group(grp, s, z, bits))
            s16.append(s)
            z16.append(z)
            group_cols.append(g)
        row_index.append(len(group_cols))
    with np.errstate(over="ignore"):
        sh = np.array(s16, dtype=np.float64).astype(np.float16)
        zh = np.array(z16, dtype=np.float64).astype(np.float16)
    if not (np.all(np.isfinite(sh)) and np.all(np.isfinite(zh)) and np.all(sh > 0)):
        raise ValueError("scale/zero not representable in fp16 (reading R8)")
    # low bits first: element e of the stream at bits [e*n, e*n+n)
    per = 8 // bits                         # bits in {2, 4, 8}: whole codes per byte
    c = np.array(codes, dtype=np.uint32)
    c = np.concatenate([c, np.zeros((-len(c)) % per, dtype=np.uint32)]).reshape(-1, per)
    code_bytes = np.zeros(c.shape[0], dtype=np.uint32)
    for j in range(per):
        code_bytes |= c[:, j] << (j * bits)
    code_bytes = code_bytes.astype(np.uint8)
    return {
        "rows": rows, "cols": cols, "group_size": G, "bits": bits, "nnzg": len(group_cols),
        "row_index": np.array(row_index, dtype=np.int32),
        "group_cols": np.array(group_cols, dtype=np.uint16),
        "codes": code_bytes,
        "scales_f16": sh.view(np.uint16), "zeros_f16": zh.view(np.uint16),
    }


def compress_layer(W, hinv_diag, sparsity: float, bits: int, G: int = 16):
    """Steps 2-5 on one layer; returns (bsr, keep, per_group)."""
    per_group = group_saliency(weight_saliency(W, hinv_diag), G)
    keep = select_groups(per_group, sparsity)
    return build_gqs(W, keep, G, bits), keep, per_group
