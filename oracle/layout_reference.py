"""Independent Python implementation of the packed-blob LAYOUT v1 -- TEST
INFRASTRUCTURE ONLY (same import rules as gqsa_oracle.py).

Written from the prose specification in DESIGN.md §5, not from the C++
packer, so that `gqsa_pack` bytes == `pack_reference` bytes is a check of two
implementations of one document.  Uses only struct / numpy.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = 0x41535147
VERSION = 1
T = 128          # groups per tile
LANES = 32
HDR = 256
ALIGN = 256


def _align(v: int, a: int = ALIGN) -> int:
    return -(-v // a) * a


def tile_bytes(bits: int) -> int:
    # 32 B tile header + codes (T*G*n/8) + s/z (T*4) + columns (T*2)
    return 32 + T * 16 * bits // 8 + T * 4 + T * 2


def pack_reference(bsr: dict, row_begin: int = 0, row_end=None) -> bytes:
    rows_all = int(bsr["rows"])
    row_end = rows_all if row_end is None else int(row_end)
    G, n, K = int(bsr["group_size"]), int(bsr["bits"]), int(bsr["cols"])
    ri_all = [int(v) for v in np.asarray(bsr["row_index"])]
    g0, g1 = ri_all[row_begin], ri_all[row_end]
    rows = row_end - row_begin
    nnzg = g1 - g0
    ri = [v - g0 for v in ri_all[row_begin:row_end + 1]]
    counts = [ri[r + 1] - ri[r] for r in range(rows)]
    nzrows = [r for r in range(rows) if counts[r] > 0]
    empty = [r for r in range(rows) if counts[r] == 0]
    ordinal = {r: i for i, r in enumerate(nzrows)}
    row_of = []
    for r in range(rows):
        row_of += [r] * counts[r]
    num_tiles = -(-nnzg // T)
    tb = tile_bytes(n)
    off_ri = HDR
    off_nz = _align(off_ri + 4 * (rows + 1))
    off_em = _align(off_nz + 4 * len(nzrows))
    off_tiles = _align(off_em + 4 * len(empty))
    total = _align(off_tiles + num_tiles * tb)

    out = bytearray(total)
    struct.pack_into("<IIiiiiqiiiiiiiiQQQQQ", out, 0,
                     MAGIC, VERSION, rows, K, G, n, nnzg, T, num_tiles, len(nzrows), len(empty),
                     tb, 1, row_begin, row_end, off_ri, off_nz, off_em, off_tiles, total)
    struct.pack_into(f"<{rows + 1}i", out, off_ri, *ri)
    if nzrows:
        struct.pack_into(f"<{len(nzrows)}i", out, off_nz, *nzrows)
    if empty:
        struct.pack_into(f"<{len(empty)}i", out, off_em, *empty)

    cb = G * n // 8                       # code bytes per group
    codes = np.asarray(bsr["codes"], np.uint8)
    gcols = np.asarray(bsr["group_cols"], np.uint16)
    sc = np.asarray(bsr["scales_f16"], np.uint16)
    zr = np.asarray(bsr["zeros_f16"], np.uint16)
    per_plane = 16 // cb                  # groups of one lane in a 16-B code vector
    codes_total = T * cb
    for t in range(num_tiles):
        base = off_tiles + t * tb
        masks = [0, 0, 0, 0]
        for j in range(T):                # j = u*32 + lane
            pos = t * T + j
            if pos >= nnzg:
                continue
            u, lane = divmod(j, LANES)
            g = g0 + pos
            if pos == 0 or row_of[pos] != row_of[pos - 1]:
                masks[u] |= 1 << lane
            swap = lane & 1
            gb = bytes(codes[g * cb:(g + 1) * cb])
            if swap:
                gb = gb[cb // 2:] + gb[:cb // 2]
            off_c = base + 32 + (u // per_plane) * 512 + lane * 16 + (u % per_plane) * cb
            out[off_c:off_c + cb] = gb
            off_sz = base + 32 + codes_total + lane * 16 + u * 4
            struct.pack_into("<HH", out, off_sz, int(sc[g]), int(zr[g]))
            off_col = base + 32 + codes_total + T * 4 + lane * 8 + u * 2
            struct.pack_into("<H", out, off_col, (int(gcols[g]) << 1) | swap)
        m0 = ordinal[row_of[t * T]]
        struct.pack_into("<IIIIi", out, base, *masks, m0)
    return bytes(out)
