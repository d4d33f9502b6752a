"""GQSA CPU oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 reference for the GQSA decode hot path
(arXiv 2412.17560).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with the CUDA path (``paper_2412_17560_b200``):
no kernels, headers, helpers, tables or pre/post-processing.  It imports only
numpy and the standard library.

Citations are ``PAPER.md:L [section / equation]`` into /root/reference/PAPER.md
(the paper's LaTeX) and ``SPEC.md:L [module / op]``.

What the hot path computes (PAPER.md:64-69 [Eq. 3], PAPER.md:95-101 [§3.2 BSR
listing], PAPER.md:134 [§3.5 "GEMV task of shape 1xNxK"]):

    y[b][r] = sum_{g in [rowIndex[r], rowIndex[r+1])}
                  sum_{t < G} (q[g][t] - z[g]) * s[g] * x[b][groups[g]*G + t]
              (+ bias[r])

This is an exact-result method: the kernel reaches the plain definition
y = W_hat @ x with W_hat = decompress(BSR).  The oracle therefore *is* that
definition written out, in fp64.  Every product (q - z) * s * x of
fp16-derived values is exact in fp64 (<= 50 significand bits),
so only the additions round.

Pins (tests/test_oracle.py):
  * unpack_codes ........ SPEC.md:149 worked example (0x15 <-> [5, 1]), brute
                          bit-by-bit definition on random streams.
  * decompress .......... PAPER.md:95-101 listing (golden fixture), zeros at
                          pruned positions, placement example SPEC.md:272.
  * gemv ................ PAPER.md:95-101 fixture exact outputs
                          (tests/golden/paper_fig3.json); exact Fraction
                          brute force over every mask of tiny grids; S=0
                          equals the dense int64 matmul in exact-integer mode;
                          linearity; empty rows == bias.
  * compute_qparams /
    quantize_group ...... SPEC.md:122-124, 131 worked examples (Eq. 1-2).
  * dequantize_group .... SPEC.md:140 worked example (Eq. 3).
  * partition_stream_k .. SPEC.md:508-509 worked examples.
  * footprint ........... SPEC.md:293 worked example; ratio in [4.0, 5.0]
                          bracketing PAPER.md:399 "4.3x compression ratio".
"""
from __future__ import annotations

import math
from typing import Optional

import numpy as np

__all__ = [
    "unpack_codes",
    "f16_bits_to_f64",
    "decompress",
    "gemv",
    "gemv_rows",
    "compute_qparams",
    "quantize_group",
    "dequantize_group",
    "partition_stream_k",
    "footprint_bytes",
    "validate_bsr",
]


# --------------------------------------------------------------------------
# Storage decoding
# --------------------------------------------------------------------------

def unpack_codes(packed: np.ndarray, count: int, bits: int) -> np.ndarray:
    """Unpack ``count`` unsigned ``bits``-bit codes from a little-endian bit stream.

    Element e occupies bits [e*bits, e*bits + bits) of the byte stream, least
    significant bit first ("code 2k in low nibble of byte
    k"; reading R10).  For bits=4 this is "low nibble first".

    Written as the definition: expand every byte into its 8 bits (LSB first),
    then read each code as sum_i bit_i * 2^i.
    """
    packed = np.asarray(packed, dtype=np.uint8)
    nbits = count * bits
    if packed.size * 8 < nbits:
        raise ValueError("packed stream too short")
    allbits = np.unpackbits(packed, bitorder="little")[:nbits].astype(np.int64)
    allbits = allbits.reshape(count, bits)
    weights = (1 << np.arange(bits, dtype=np.int64))
    return (allbits * weights).sum(axis=1)


def f16_bits_to_f64(bits_u16: np.ndarray) -> np.ndarray:
    """IEEE binary16 bit patterns -> float64 (exact widening).

    s and z are stored as fp16 (reading R7: "Parity is defined on the
    stored fp16 values"; PAPER.md:134 says only "along with scaling factors and
    zero points").
    """
    return np.asarray(bits_u16, dtype=np.uint16).view(np.float16).astype(np.float64)


def validate_bsr(bsr: dict) -> None:
    """Layer invariants: raises ValueError.

    row_index[0] == 0, non-decreasing, row_index[rows] == nnzg; group columns
    strictly increasing within a row and < cols/G; cols % G == 0.
    """
    rows, cols, G = int(bsr["rows"]), int(bsr["cols"]), int(bsr["group_size"])
    ri = np.asarray(bsr["row_index"], dtype=np.int64)
    gc = np.asarray(bsr["group_cols"], dtype=np.int64)
    if cols % G != 0:
        raise ValueError("cols % G != 0")
    if ri.shape != (rows + 1,) or ri[0] != 0:
        raise ValueError("row_index shape / row_index[0]")
    if np.any(np.diff(ri) < 0):
        raise ValueError("row_index not monotone")
    if ri[-1] != gc.size:
        raise ValueError("row_index[rows] != nnzg")
    for r in range(rows):
        seg = gc[ri[r]:ri[r + 1]]
        if seg.size and (np.any(np.diff(seg) <= 0) or seg[-1] >= cols // G or seg[0] < 0):
            raise ValueError(f"group_cols invalid in row {r}")


def _dequant_groups(bsr: dict) -> np.ndarray:
    """Eq. 3: W_hat = (W_tilde - z) * s, per kept group, fp64.

    Returns an array [nnzg, G] of dequantized weights in CSR (storage) order.
    """
    G, n = int(bsr["group_size"]), int(bsr["bits"])
    nnzg = int(np.asarray(bsr["group_cols"]).size)
    q = unpack_codes(bsr["codes"], nnzg * G, n).reshape(nnzg, G).astype(np.float64)
    s = f16_bits_to_f64(bsr["scales_f16"]).reshape(nnzg, 1)
    z = f16_bits_to_f64(bsr["zeros_f16"]).reshape(nnzg, 1)
    return (q - z) * s


def decompress(bsr: dict) -> np.ndarray:
    """Dense W_hat [rows][cols] in fp64 from the plain BSR.

    BSR semantics: row r owns kept groups
    [rowIndex[r], rowIndex[r+1]) (reading R1: the paper's "rowIndex[r+1] -
    rowIndex[i]" is a typo); group g sits at columns groups[g]*G ... +G
    ("in terms of group units", reading R4); values are group-major, G
    consecutive columns per group (reading R2).  Pruned positions are exactly 0.
    """
    rows, cols, G = int(bsr["rows"]), int(bsr["cols"]), int(bsr["group_size"])
    ri = np.asarray(bsr["row_index"], dtype=np.int64)
    gc = np.asarray(bsr["group_cols"], dtype=np.int64)
    wg = _dequant_groups(bsr)
    W = np.zeros((rows, cols), dtype=np.float64)
    for r in range(rows):
        for g in range(ri[r], ri[r + 1]):
            c0 = gc[g] * G
            W[r, c0:c0 + G] = wg[g]
    return W


def _x_to_f64(x) -> np.ndarray:
    x = np.asarray(x)
    if x.dtype == np.uint16:
        x = x.view(np.float16)
    return x.astype(np.float64)


def gemv_rows(bsr: dict, x, row_ids, bias: Optional[np.ndarray] = None) -> np.ndarray:
    """The oracle GEMV restricted to the rows ``row_ids`` -> y [B][len(row_ids)].

    Same arithmetic as :func:`gemv`; lets tests and the bench's CPU baseline
    evaluate sampled outputs of full-size layers one by one.
    """
    G = int(bsr["group_size"])
    n = int(bsr["bits"])
    X = _x_to_f64(x)
    if X.ndim == 1:
        X = X[None, :]
    if X.shape[1] != int(bsr["cols"]):
        raise ValueError("x length != cols")
    ri = np.asarray(bsr["row_index"], dtype=np.int64)
    gc = np.asarray(bsr["group_cols"], dtype=np.int64)
    s_all = f16_bits_to_f64(bsr["scales_f16"])
    z_all = f16_bits_to_f64(bsr["zeros_f16"])
    codes = np.asarray(bsr["codes"], dtype=np.uint8)
    row_ids = np.asarray(row_ids, dtype=np.int64)
    B = X.shape[0]
    y = np.zeros((B, row_ids.size), dtype=np.float64)
    t = np.arange(G, dtype=np.int64)
    for j, r in enumerate(row_ids):
        g0, g1 = int(ri[r]), int(ri[r + 1])
        if g1 > g0:
            # codes of groups g0..g1-1: elements [g0*G, g1*G) of the bit stream.
            e0, e1 = g0 * G, g1 * G
            b0, b1 = (e0 * n) // 8, -(-(e1 * n) // 8)
            off = (e0 * n) - b0 * 8           # bit offset inside the first byte
            sub = np.unpackbits(codes[b0:b1], bitorder="little")[off:off + (e1 - e0) * n]
            q = (sub.reshape(-1, n).astype(np.int64) * (1 << np.arange(n))).sum(1)
            q = q.reshape(g1 - g0, G).astype(np.float64)
            # Eq. 3: (q - z) * s, then times the activation gathered "according to
            # the real group index of each group".
            w_hat = (q - z_all[g0:g1, None]) * s_all[g0:g1, None]
            cols_idx = (gc[g0:g1, None] * G + t[None, :]).reshape(-1)
            for b in range(B):
                terms = (w_hat.reshape(-1) * X[b, cols_idx])
                # accumulate left to right, CSR order, t = 0..G-1 (cumsum is a
                # strictly sequential running sum).
                y[b, j] = np.cumsum(terms)[-1]
        if bias is not None:
            y[:, j] += np.float64(np.asarray(bias)[r])
    return y


def gemv(bsr: dict, x, bias: Optional[np.ndarray] = None) -> np.ndarray:
    """y = W_hat @ x for every row, fp64.  x: [K] or [B][K] (fp16 bits or floats).

    Returns [B][rows] (B = 1 for a 1-D x).  Empty rows yield exactly bias[r]
    (or 0).  Batch rows are independent (small-batch GEMM
    = B independent GEMVs, "TensorCores (MMA) or CudaCores (FMA)").
    """
    return gemv_rows(bsr, x, np.arange(int(bsr["rows"])), bias)


# --------------------------------------------------------------------------
# Quantizer (upstream of the hot path; pinned by SPEC worked examples)
# --------------------------------------------------------------------------

def _round_half_away(v: float) -> float:
    """The paper's rounding operator with ties away from zero (reading R5;
    SPEC.md:128, 160)."""
    return math.copysign(math.floor(abs(v) + 0.5), v)


def compute_qparams(group, bits: int):
    """Eq. 1: s = (max W - min W) / (2^n - 1); z = -round(min W / s).

    Degenerate group (max == min == c), reading R9: s = |c| (1 if c == 0),
    z = -sign(c), so that code 0 dequantizes to c exactly.
    """
    w = [float(v) for v in group]
    if not w or any(not math.isfinite(v) for v in w):
        raise ValueError("empty or non-finite group")
    lo, hi = min(w), max(w)
    if hi == lo:
        c = lo
        if c == 0.0:
            return 1.0, 0.0
        return abs(c), -math.copysign(1.0, c)
    s = (hi - lo) / (2 ** bits - 1)
    z = -_round_half_away(lo / s)
    return s, z


def quantize_group(group, s: float, z: float, bits: int):
    """Eq. 2: clamp(round(W / s) + z, 0, 2^n - 1)."""
    qmax = 2 ** bits - 1
    return [int(min(max(_round_half_away(float(v) / s) + z, 0), qmax)) for v in group]


def dequantize_group(codes, s: float, z: float):
    """Eq. 3: W_hat = (W_tilde - z) * s."""
    return [(float(q) - z) * s for q in codes]


# --------------------------------------------------------------------------
# Work partition and footprint
# --------------------------------------------------------------------------

def partition_stream_k(total: int, parts: int):
    """Task-centric split (PAPER.md:161 [§3.5 Stream-K]).

    Contiguous ranges over 0..total whose sizes differ by at most one; the
    first ``total % parts`` ranges get the extra unit (SPEC.md:508 example
    nnzg=10, P=3 -> {4, 3, 3}).  Returns a list of (lo, hi).
    """
    q, r = divmod(total, parts)
    out, lo = [], 0
    for c in range(parts):
        hi = lo + q + (1 if c < r else 0)
        out.append((lo, hi))
        lo = hi
    return out


def footprint_bytes(rows: int, cols: int, nnzg: int, G: int, bits: int, batch: int = 1) -> dict:
    """Algorithmic (compressed) bytes of one GEMV call, SURVEY §8(d).

    Per kept group: n*G/8 code bytes + 2 (fp16 s) + 2 (fp16 z) + 2 (u16 group
    column); 4*(rows+1) B of row offsets; per call 2*B*K bytes of fp16 x and
    4*B*N bytes of fp32 y.  (SPEC.md:293 counts codes, scales, zeros,
    group_cols and (rows+1) row offsets for the file payload.)
    """
    codes = nnzg * G * bits // 8
    weights = codes + 6 * nnzg + 4 * (rows + 1)
    act = 2 * batch * cols + 4 * batch * rows
    payload_file = codes + 6 * nnzg + 4 * (rows + 1)
    return {
        "codes": codes,
        "scales": 2 * nnzg,
        "zeros": 2 * nnzg,
        "group_cols": 2 * nnzg,
        "row_index": 4 * (rows + 1),
        "weight_bytes": weights,
        "act_bytes": act,
        "total": weights + act,
        "payload_file_bytes": payload_file,
        "ratio_vs_fp16": (2.0 * rows * cols) / payload_file,
    }
