"""Parity helpers shared by the GPU tests (test infrastructure)."""
import numpy as np

from oracle import gqsa_oracle as O


def abs_bound(bsr: dict, x_bits: np.ndarray, rows=None) -> np.ndarray:
    """A_r = sum_g |s_g| (sum_t |q_t x_t| + |z_g| sum_t |x_t|) per row (and
    batch): the magnitude the fp32 kernel's rounding errors scale with
    (DESIGN.md §7).  Returns [B][len(rows)]."""
    G, n = int(bsr["group_size"]), int(bsr["bits"])
    X = np.asarray(x_bits).view(np.float16).astype(np.float64)
    if X.ndim == 1:
        X = X[None]
    ri = np.asarray(bsr["row_index"], np.int64)
    gc = np.asarray(bsr["group_cols"], np.int64)
    s = np.abs(O.f16_bits_to_f64(bsr["scales_f16"]))
    z = np.abs(O.f16_bits_to_f64(bsr["zeros_f16"]))
    rows = np.arange(int(bsr["rows"])) if rows is None else np.asarray(rows)
    out = np.zeros((X.shape[0], rows.size))
    t = np.arange(G)
    codes = np.asarray(bsr["codes"], np.uint8)
    for j, r in enumerate(rows):
        g0, g1 = int(ri[r]), int(ri[r + 1])
        if g1 == g0:
            continue
        e0, e1 = g0 * G * n, g1 * G * n
        bits = np.unpackbits(codes[e0 // 8:-(-e1 // 8)], bitorder="little")[e0 % 8:e0 % 8 + (e1 - e0)]
        q = (bits.reshape(-1, n) * (1 << np.arange(n))).sum(1).reshape(g1 - g0, G)
        idx = gc[g0:g1, None] * G + t
        for b in range(X.shape[0]):
            ax = np.abs(X[b][idx])
            out[b, j] = np.sum(s[g0:g1] * ((q * ax).sum(1) + z[g0:g1] * ax.sum(1)))
    return out


def check_gates(y_gpu: np.ndarray, y_ref: np.ndarray, A: np.ndarray, what: str = "") -> None:
    """G1 (north star, literal): max|dy| <= 1e-3 ||y||_2;  G2 (per row, sees a
    dropped group): |dy_r| <= 1e-5 A_r;  G3: ||dy||_2 <= 1e-4 ||y||_2."""
    y_gpu = np.asarray(y_gpu, np.float64)
    d = np.abs(y_gpu - y_ref)
    nrm = np.linalg.norm(y_ref)
    assert np.all(np.isfinite(y_gpu)), what
    assert d.max(initial=0.0) <= 1e-3 * nrm + 1e-30, f"G1 {what}: {d.max()} vs {nrm}"
    bad = d > 1e-5 * A + 1e-30
    assert not bad.any(), f"G2 {what}: {np.argwhere(bad)[:5]} d={d[bad][:5]} A={A[bad][:5]}"
    assert np.linalg.norm(d) <= 1e-4 * nrm + 1e-30, f"G3 {what}"
