"""Parity helpers shared by the GPU tests (test infrastructure)."""
import numpy as np

from oracle import gqsa_oracle as O


# Offset each element carries through the kernel's folded dot products before
# it is removed once per group (DESIGN.md §6 step 4, §7): W4 even t 1024, odd
# t 1024/16; W2 t mod 4 = j: 1024/4^j; W8 1024.
def _fold_offsets(bits: int, G: int) -> np.ndarray:
    t = np.arange(G)
    if bits == 4:
        return np.where(t % 2 == 0, 1024.0, 64.0)
    if bits == 2:
        return 1024.0 / 4.0 ** (t % 4)
    return np.full(G, 1024.0)


FOLD_REL = 2.0 ** -23 / 1e-5  # fold error: 2 roundings (2^-24) of o_t|x_t| per group, in G2 units
# G2x: the worst-case recursive-summation bound of the folded
# chains, for inputs whose |x| spans the fp16 range.  A W4 group's two FHFMA
# chains each add G/2 = 8 exact products, every addition rounding at most
# 2^-24 |partial| <= 2^-24 F_group, plus the fold and scale roundings: (8 + 2)
# roundings of F per group (W2: 4 chains of 4 adds; W8: 2 chains of 8).
FOLD_REL_WORST = 10 * 2.0 ** -24 / 1e-5


def abs_bound(bsr: dict, x_bits: np.ndarray, rows=None, fold_rel: float = FOLD_REL) -> np.ndarray:
    """G2's scale per row (and batch): A_r + fold_rel * F_r with
    A_r = sum_g |s_g| (sum_t |q_t x_t| + |z_g| sum_t |x_t|), the magnitude of
    the terms the fp32 kernel adds, and F_r = sum_g |s_g| sum_t o_t |x_t|, the
    magnitude of the fold offsets o_t it carries and removes once per group
    (so |dy_r| <= 1e-5 A_r + 2^-23 F_r).  fold_rel =
    FOLD_REL_WORST gives G2x, the worst-case bound for extreme |x|.
    Returns [B][len(rows)]."""
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
    off = _fold_offsets(n, G)
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
            out[b, j] += fold_rel * np.sum(s[g0:g1] * (ax * off).sum(1))
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
