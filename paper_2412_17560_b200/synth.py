"""Seeded synthetic inputs for the GQSA hot path (shared by tests, bench and smoke).

This module holds NONE of the method's arithmetic: it never dequantizes,
multiplies or reduces.  It only draws random codes / scales / zeros / masks /
activations with the shapes and statistics of the paper's workloads and
writes them in the plain BSR storage format: row offsets,
kept-group column indices, n-bit packed codes (element e at bits
[e*n, e*n+n), low bits first -- SPEC.md:146) and fp16 scale / zero bit
patterns.  The recipe is stated in DESIGN.md §4.

Value modes:
  * ``realistic``   codes ~ round(N((2^n-1)/2, (2^n-1)/4.5)) clipped -- the
                    histogram of Eq. 2 applied to Gaussian groups; per-row
                    scale sigma_r = 0.02 * 10^U(-1,1) (SPEC.md:64 channel
                    imbalance), s = sigma_r * U(3,5)/(2^n-1) * (1+U(-.01,.01));
                    z = round(U(.3,.7)*(2^n-1)) + U(-.5,.5) (continuous z after
                    E2E-OQP).  s, z rounded to fp16.
  * ``exact_int``   codes uniform, s in {0.5, 1, 2}, integer z in [0, 2^n-1]
                    (every term and partial sum a multiple of 0.5; fp32 is
                    exact -> bit-exact parity).
  * ``onehot_safe`` realistic, but z rounded to a multiple of 1/128 with
                    |z| < 16 (y = W_hat[:, j] exact in fp32).
  * ``extreme``     reading R6's full range (any finite fp16 z):
                    uniform codes; s log-uniform over [2^-24, 1] (fp16
                    subnormals included); z a mixture of uniform [-1000, 1000],
                    integers in [-2^n, 2^(n+1)] (outside [0, 2^n-1] too) and
                    tiny values of either sign (fp16 subnormals included).

Masks (exactly floor(S * N*K/G) groups pruned):
  * ``uniform``      chosen uniformly without replacement over the layer;
  * ``row_balanced`` each row prunes exactly floor(S * K/G);
  * ``skewed``       a random half of the rows keeps everything, the rest
                     keeps nothing (S=0.5; the Slice-K stress case SPEC.md:630).
"""
from __future__ import annotations

import zlib
from typing import Optional

import numpy as np

__all__ = ["seed_for", "make_layer", "make_x", "pack_bits", "bsr_from_parts", "shard_rows",
           "make_dense", "make_calib"]


def seed_for(name: str) -> int:
    """seed = crc32(name) -- e.g. ``"llama3-8b/q/4/0.5/16/uniform"``."""
    return zlib.crc32(name.encode()) & 0xFFFFFFFF


def pack_bits(codes: np.ndarray, bits: int) -> np.ndarray:
    """Write unsigned codes into the little-endian n-bit stream (storage format)."""
    codes = np.asarray(codes).reshape(-1)
    if codes.size and (int(codes.min()) < 0 or int(codes.max()) >= (1 << bits)):
        raise ValueError("code out of range")
    c = codes.astype(np.uint8)
    if bits in (1, 2, 4, 8):
        per = 8 // bits
        pad = (-c.size) % per
        if pad:
            c = np.concatenate([c, np.zeros(pad, np.uint8)])
        c = c.reshape(-1, per)
        out = np.zeros(c.shape[0], np.uint8)
        for i in range(per):
            out |= (c[:, i] << (i * bits)).astype(np.uint8)
        return out
    b = ((codes.astype(np.int64)[:, None] >> np.arange(bits)) & 1).astype(np.uint8).reshape(-1)
    pad = (-b.size) % 8
    if pad:
        b = np.concatenate([b, np.zeros(pad, np.uint8)])
    return np.packbits(b, bitorder="little")


def _f16_bits(v: np.ndarray) -> np.ndarray:
    return np.asarray(v, dtype=np.float64).astype(np.float16).view(np.uint16)


def _keep_mask(rng, rows: int, gpr: int, sparsity: float, mask: str) -> np.ndarray:
    total = rows * gpr
    if mask == "uniform":
        n_prune = int(np.floor(sparsity * total + 1e-9))
        keep = np.ones(total, dtype=bool)
        if n_prune:
            keep[rng.choice(total, size=n_prune, replace=False)] = False
        return keep.reshape(rows, gpr)
    if mask == "row_balanced":
        n_prune = int(np.floor(sparsity * gpr + 1e-9))
        keep = np.ones((rows, gpr), dtype=bool)
        for r in range(rows):
            keep[r, rng.choice(gpr, size=n_prune, replace=False)] = False
        return keep
    if mask == "skewed":
        keep = np.zeros((rows, gpr), dtype=bool)
        full = rng.choice(rows, size=rows - int(np.floor(sparsity * rows + 1e-9)), replace=False)
        keep[full] = True
        return keep
    raise ValueError(f"unknown mask kind {mask!r}")


def bsr_from_parts(rows, cols, G, bits, keep, codes, s, z) -> dict:
    """Assemble a plain-BSR dict from a keep mask [rows][K/G] and per-kept-group
    codes (either [nnzg][G] integers or an already packed n-bit byte stream),
    s [nnzg] and z [nnzg] (CSR order = row-major over the mask)."""
    keep = np.asarray(keep, dtype=bool)
    counts = keep.sum(axis=1)
    row_index = np.zeros(rows + 1, dtype=np.int32)
    np.cumsum(counts, out=row_index[1:])
    group_cols = np.nonzero(keep)[1].astype(np.uint16)
    codes = np.asarray(codes)
    packed = codes if codes.dtype == np.uint8 and codes.ndim == 1 else pack_bits(codes, bits)
    return {
        "rows": int(rows), "cols": int(cols), "group_size": int(G), "bits": int(bits),
        "nnzg": int(row_index[-1]),
        "row_index": row_index,
        "group_cols": group_cols,
        "codes": packed,
        "scales_f16": _f16_bits(s),
        "zeros_f16": _f16_bits(z),
    }


def make_layer(seed: int, rows: int, cols: int, G: int = 16, bits: int = 4,
               sparsity: float = 0.5, mask: str = "uniform",
               mode: str = "realistic") -> dict:
    """A seeded synthetic GQS layer in plain BSR form (see module docstring)."""
    if cols % G:
        raise ValueError("cols % G != 0")
    rng = np.random.default_rng(seed)
    gpr = cols // G
    keep = _keep_mask(rng, rows, gpr, sparsity, mask)
    nnzg = int(keep.sum())
    qmax = (1 << bits) - 1
    row_of = np.repeat(np.arange(rows), keep.sum(axis=1))
    chunk = 1 << 20  # groups per generation chunk (bounded host memory)
    packed = []
    if mode in ("realistic", "onehot_safe"):
        for g0 in range(0, nnzg, chunk):
            m = min(chunk, nnzg - g0)
            c = np.clip(np.rint(rng.normal(qmax / 2.0, qmax / 4.5, size=(m, G))), 0, qmax)
            packed.append(pack_bits(c.astype(np.uint8), bits))
        sigma_r = 0.02 * 10.0 ** rng.uniform(-1.0, 1.0, size=rows)
        s = sigma_r[row_of] * rng.uniform(3.0, 5.0, size=nnzg) / qmax
        s = s * (1.0 + rng.uniform(-0.01, 0.01, size=nnzg))
        z = np.rint(rng.uniform(0.3, 0.7, size=nnzg) * qmax) + rng.uniform(-0.5, 0.5, size=nnzg)
        if mode == "onehot_safe":
            z = np.clip(np.rint(z * 128.0) / 128.0, -15.9921875, 15.9921875)
    elif mode == "extreme":
        for g0 in range(0, nnzg, chunk):
            m = min(chunk, nnzg - g0)
            packed.append(pack_bits(rng.integers(0, qmax + 1, size=(m, G), dtype=np.uint8), bits))
        s = 2.0 ** rng.uniform(-24.0, 0.0, size=nnzg)
        kind = rng.integers(0, 3, size=nnzg)
        z = np.where(kind == 0, rng.uniform(-1000.0, 1000.0, size=nnzg),
                     np.where(kind == 1, rng.integers(-(qmax + 1), 2 * (qmax + 1) + 1, size=nnzg).astype(np.float64),
                              rng.choice([-1.0, 1.0], size=nnzg) * 2.0 ** rng.uniform(-24.0, -10.0, size=nnzg)))
    elif mode == "exact_int":
        for g0 in range(0, nnzg, chunk):
            m = min(chunk, nnzg - g0)
            packed.append(pack_bits(rng.integers(0, qmax + 1, size=(m, G), dtype=np.uint8), bits))
        s = rng.choice(np.array([0.5, 1.0, 2.0]), size=nnzg)
        z = rng.integers(0, qmax + 1, size=nnzg).astype(np.float64)
    else:
        raise ValueError(f"unknown value mode {mode!r}")
    codes = np.concatenate(packed) if packed else np.zeros(0, np.uint8)
    return bsr_from_parts(rows, cols, G, bits, keep, codes, s, z)


def make_x(seed: int, batch: int, cols: int, mode: str = "realistic") -> np.ndarray:
    """Activations as fp16 bit patterns, shape [batch][cols] (uint16).

    realistic: N(0,1) with 0.5 % of channels scaled x20 (activation outliers);
    exact_int: integers in [-4, 4];  onehot: row b is e_{j_b};
    extreme: N(0,1) with 1 % of entries of magnitude 10^U(3, 4.8) (up to the
    fp16 maximum 65504), 1 % fp16 subnormals/tiny (2^U(-24, -14)) and 1 %
    exact zeros, signs random.
    """
    rng = np.random.default_rng(seed)
    if mode == "realistic":
        x = rng.normal(0.0, 1.0, size=(batch, cols))
        n_out = max(1, int(round(0.005 * cols)))
        ch = rng.choice(cols, size=n_out, replace=False)
        x[:, ch] *= 20.0
    elif mode == "exact_int":
        x = rng.integers(-4, 5, size=(batch, cols)).astype(np.float64)
    elif mode == "extreme":
        x = rng.normal(0.0, 1.0, size=(batch, cols))
        u = rng.uniform(size=(batch, cols))
        sign = rng.choice([-1.0, 1.0], size=(batch, cols))
        x = np.where(u < 0.01, sign * np.minimum(10.0 ** rng.uniform(3.0, 4.8, size=(batch, cols)), 65504.0), x)
        x = np.where((u >= 0.01) & (u < 0.02), sign * 2.0 ** rng.uniform(-24.0, -14.0, size=(batch, cols)), x)
        x = np.where((u >= 0.02) & (u < 0.03), 0.0, x)
    elif mode == "onehot":
        x = np.zeros((batch, cols))
        x[np.arange(batch), rng.integers(0, cols, size=batch)] = 1.0
    else:
        raise ValueError(f"unknown x mode {mode!r}")
    return x.astype(np.float16).view(np.uint16)


def make_dense(seed: int, rows: int, cols: int) -> np.ndarray:
    """A dense fp32 weight matrix [rows][cols] for the compression front-end:
    W[r, :] ~ N(0, sigma_r^2), sigma_r = 0.02 * 10^U(-1,1) (per-row channel
    imbalance), plus 0.1 % of input columns x4 (salient input
    channels, the structure Fig. 1 shows)."""
    rng = np.random.default_rng(seed)
    sigma = 0.02 * 10.0 ** rng.uniform(-1.0, 1.0, size=rows)
    W = rng.standard_normal((rows, cols)) * sigma[:, None]
    ch = rng.choice(cols, size=max(1, cols // 1000), replace=False)
    W[:, ch] *= 4.0
    return W.astype(np.float32)


def make_calib(seed: int, n: int, cols: int) -> np.ndarray:
    """Calibration activations [n][cols] fp32: N(0,1) with 0.5 % of the
    channels x20 (activation outliers, as make_x)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, cols))
    ch = rng.choice(cols, size=max(1, int(round(0.005 * cols))), replace=False)
    X[:, ch] *= 20.0
    return X.astype(np.float32)


def shard_rows(rows: int, world: int, rank: int) -> tuple:
    """Row range [lo, hi) owned by ``rank`` under output-row sharding."""
    return (rows * rank) // world, (rows * (rank + 1)) // world


def slice_rows(bsr: dict, lo: int, hi: int) -> dict:
    """Plain BSR of rows [lo, hi) with rebased row offsets (pure data movement)."""
    ri = np.asarray(bsr["row_index"], dtype=np.int64)
    g0, g1 = int(ri[lo]), int(ri[hi])
    G, n = int(bsr["group_size"]), int(bsr["bits"])
    e0, e1 = g0 * G * n, g1 * G * n  # bit offsets
    allbits = np.unpackbits(np.asarray(bsr["codes"], np.uint8), bitorder="little")[e0:e1]
    pad = (-allbits.size) % 8
    if pad:
        allbits = np.concatenate([allbits, np.zeros(pad, np.uint8)])
    return {
        "rows": hi - lo, "cols": int(bsr["cols"]), "group_size": G, "bits": n,
        "nnzg": g1 - g0,
        "row_index": (ri[lo:hi + 1] - g0).astype(np.int32),
        "group_cols": np.asarray(bsr["group_cols"])[g0:g1].copy(),
        "codes": np.packbits(allbits, bitorder="little"),
        "scales_f16": np.asarray(bsr["scales_f16"])[g0:g1].copy(),
        "zeros_f16": np.asarray(bsr["zeros_f16"])[g0:g1].copy(),
    }
