"""Independent Python implementation of the packed-blob LAYOUT v3 -- TEST
INFRASTRUCTURE ONLY (same import rules as gqsa_oracle.py).

Written from the prose specification in DESIGN.md §5, not from the C++
packer, so that `gqsa_pack` bytes == `pack_reference` bytes is a check of two
implementations of one document.  Uses only struct / numpy.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = 0x41535147
VERSION = 3
T = 128          # groups per tile (4 slots x 32 lanes)
LANES = 32
SLOTS = 4
HDR = 256
ALIGN = 256


def _align(v: int, a: int = ALIGN) -> int:
    return -(-v // a) * a


def tile_bytes(bits: int, G: int = 16) -> int:
    # codes (T*G*n/8) + s/z (T*4) + columns (T*2); no per-tile header
    return T * G * bits // 8 + T * 4 + T * 2


def target_slots(nnzg: int) -> int:
    """Slots per lane of the longest slice: 16 when the layer
    has under 1.6 tiles (of 128 groups) per warp of a 148 x 16-warp grid, 128
    under 4, else 256."""
    tpw = nnzg / 128.0 / (148.0 * 16.0)
    return 16 if tpw < 1.6 else 128 if tpw < 4.0 else 256


def lanes_per_row(n_nz: int, max_len: int, target: int = 256) -> int:
    """S = the larger of (a) the smallest power of two with
    ceil(max_len / S) <= target slots per lane and (b) 32 / (next power of
    two >= n_nz) when fewer than 32 rows are non-empty; capped at 32."""
    if n_nz <= 0:
        return 1
    s = 1
    while s < LANES and -(-max_len // s) > target:
        s *= 2
    p = 1
    while p < n_nz and p < LANES:
        p *= 2
    return max(s, LANES // p)


def deal_row(cols_of_row, lanes, slots):
    """Bank-aware dealing of one row's kept groups (CSR positions 0..n-1 with
    group columns cols_of_row) over its lanes: slot by slot j, lane l takes
    the first remaining group whose column c has c mod 8 == want =
    (((l mod 8) // 2 + j) mod 4) + 4 * ((l // 8) mod 2), else c mod 8 ==
    want ^ 4, else the first remaining group of the fullest bucket (lowest
    bucket index on ties).  Returns {(lane, slot): position}."""
    buckets = [[] for _ in range(8)]
    for k, c in enumerate(cols_of_row):
        buckets[int(c) % 8].append(k)
    heads = [0] * 8
    left = len(cols_of_row)
    out = {}
    for j in range(slots):
        for lane in lanes:
            if left == 0:
                return out
            want = (((lane % 8) // 2 + j) % 4) + 4 * ((lane // 8) % 2)
            b = want
            if heads[b] == len(buckets[b]):
                b = want ^ 4
            if heads[b] == len(buckets[b]):
                b = max(range(8), key=lambda i: (len(buckets[i]) - heads[i], -i))
            out[(lane, j)] = buckets[b][heads[b]]
            heads[b] += 1
            left -= 1
    return out


def pack_reference(bsr: dict, row_begin: int = 0, row_end=None) -> bytes:
    row_end = int(bsr["rows"]) if row_end is None else int(row_end)
    G, n, K = int(bsr["group_size"]), int(bsr["bits"]), int(bsr["cols"])
    ri_all = [int(v) for v in np.asarray(bsr["row_index"])]
    g0 = ri_all[row_begin]
    rows = row_end - row_begin
    nnzg = ri_all[row_end] - g0
    counts = [ri_all[row_begin + r + 1] - ri_all[row_begin + r] for r in range(rows)]
    nz = [r for r in range(rows) if counts[r] > 0]
    nz.sort(key=lambda r: (-counts[r], r))          # count descending, then row
    empty = [r for r in range(rows) if counts[r] == 0]
    S = lanes_per_row(len(nz), counts[nz[0]] if nz else 0, target_slots(nnzg))
    rps = LANES // S                                # rows per slice
    n_slices = -(-len(nz) // rps)
    slice_tiles = []
    for s in range(n_slices):
        slots = -(-counts[nz[s * rps]] // S)        # the slice's longest row sets its length
        slice_tiles.append(-(-slots // SLOTS))
    num_tiles = sum(slice_tiles)
    tb = tile_bytes(n, G)
    off_ri = HDR
    off_perm = _align(off_ri + 4 * (rows + 1))
    off_em = _align(off_perm + 4 * LANES * n_slices)
    off_st0 = _align(off_em + 4 * len(empty))
    off_ts = _align(off_st0 + 4 * (n_slices + 1))
    off_tiles = _align(off_ts + 4 * num_tiles)
    total = _align(off_tiles + num_tiles * tb)

    out = bytearray(total)
    struct.pack_into("<IIiiiiqiiiiiiiiiiQQQQQQQ", out, 0,
                     MAGIC, VERSION, rows, K, G, n, nnzg, T, num_tiles, len(nz), len(empty),
                     tb, (4 if G == 16 else 0) | (S << 8), row_begin, row_end, n_slices, 0,
                     off_ri, off_perm, off_em, off_st0, off_ts, off_tiles, total)
    struct.pack_into(f"<{rows + 1}i", out, off_ri, *[v - g0 for v in ri_all[row_begin:row_end + 1]])
    if empty:
        struct.pack_into(f"<{len(empty)}i", out, off_em, *empty)
    # slice tables: first tile of each slice (+ the total), and the slice of each tile
    first = [sum(slice_tiles[:s]) for s in range(n_slices + 1)]
    struct.pack_into(f"<{n_slices + 1}i", out, off_st0, *first)
    if num_tiles:
        struct.pack_into(f"<{num_tiles}i", out, off_ts, *[s for s in range(n_slices) for _ in range(slice_tiles[s])])

    cb = G * n // 8
    codes = np.asarray(bsr["codes"], np.uint8)
    gcols = np.asarray(bsr["group_cols"], np.uint16)
    sc = np.asarray(bsr["scales_f16"], np.uint16)
    zr = np.asarray(bsr["zeros_f16"], np.uint16)
    per_plane = 16 // cb
    codes_total = T * cb
    t = 0
    for s in range(n_slices):
        lane_row = []
        for lane in range(LANES):
            k = s * rps + lane // S
            lane_row.append(nz[k] if k < len(nz) else -1)
        struct.pack_into(f"<{LANES}i", out, off_perm + 4 * LANES * s, *lane_row)
        nt = slice_tiles[s]
        deal = {}
        for l0 in range(0, LANES, S):
            row = lane_row[l0]
            if row >= 0:
                gr = ri_all[row_begin + row]
                if G == 16:
                    dealt = deal_row(gcols[gr:gr + counts[row]], range(l0, l0 + S), nt * SLOTS)
                else:  # G = 8 / 32: CSR order, round robin over the row's S lanes
                    dealt = {(l0 + p % S, p // S): p for p in range(counts[row])}
                for key, pos in dealt.items():
                    deal[key] = gr + pos
        for tau in range(nt):
            base = off_tiles + t * tb
            for u in range(SLOTS):
                for lane in range(LANES):
                    g = deal.get((lane, tau * SLOTS + u))
                    off_col = base + codes_total + T * 4 + lane * 8 + u * 2
                    if g is None:  # padding: s = z = 0, codes 0, reads the zero block after x (byte 2K)
                        struct.pack_into("<H", out, off_col, 2 * K)
                        continue
                    swap = lane % 2 if G == 16 else lane % 4 if G == 32 else 0
                    gb = bytes(codes[g * cb:(g + 1) * cb])
                    if G == 32:   # the lane reads chunks rot, rot+1, .. (mod 4): words in that order
                        gb = b"".join(gb[4 * ((k + swap) % 4):4 * ((k + swap) % 4) + 4] for k in range(4))
                    elif swap:
                        gb = gb[cb // 2:] + gb[:cb // 2]
                    off_c = base + (u // per_plane) * 512 + lane * 16 + (u % per_plane) * cb
                    out[off_c:off_c + cb] = gb
                    struct.pack_into("<HH", out, base + codes_total + lane * 16 + u * 4,
                                     int(sc[g]), int(zr[g]))
                    # byte offset of the group's first 16-B x chunk: 2c + swap (G = 16), c (G = 8), 4c (G = 32)
                    field = (((int(gcols[g]) << 1) | swap) << 4 if G == 16 else
                             (int(gcols[g]) << 4) if G == 8 else (((int(gcols[g]) << 2) | swap) << 4))
                    struct.pack_into("<H", out, off_col, field)
            t += 1
    return bytes(out)


# ---------------------------------------------------------------- LAYOUT-TC
TC_ROWS = 16
TC_ITEMS = 4
TC_TILE = 768
FLAG_TC = 2


def pack_reference_tc(bsr: dict, row_begin: int = 0, row_end=None) -> bytes:
    """LAYOUT-TC, written from its description: rows in
    blocks of 16; a block's items are the group columns kept by any of its
    rows, ascending (a block with none gets one padding item at column K/16);
    tiles of 4 items: codes at lane * 16 + item * 4 (lane L's 32-bit word,
    nibble j = A[(L >> 2) + 8 (j & 1)][2 (L & 3) + 8 ((j >> 1) & 1) + (j >> 2)]),
    then (s, z) of rows g and g + 8 at 512 + g * 32 + item * 8; side arrays:
    item columns u16 [tile][4], first tile of each block, block of each tile."""
    row_end = int(bsr["rows"]) if row_end is None else int(row_end)
    G, n, K = int(bsr["group_size"]), int(bsr["bits"]), int(bsr["cols"])
    assert G == 16 and n == 4
    ri_all = [int(v) for v in np.asarray(bsr["row_index"])]
    g0 = ri_all[row_begin]
    rows = row_end - row_begin
    nnzg = ri_all[row_end] - g0
    gcols = np.asarray(bsr["group_cols"], np.int64)
    codes = np.asarray(bsr["codes"], np.uint8)
    sc = np.asarray(bsr["scales_f16"], np.uint16)
    zr = np.asarray(bsr["zeros_f16"], np.uint16)
    nb = -(-rows // TC_ROWS)
    pad_col = K // G
    block_cols, empty = [], []
    for blk in range(nb):
        cs = set()
        for r in range(blk * TC_ROWS, min(rows, (blk + 1) * TC_ROWS)):
            a, b = ri_all[row_begin + r], ri_all[row_begin + r + 1]
            if a == b:
                empty.append(r)
            cs.update(int(c) for c in gcols[a:b])
        block_cols.append(sorted(cs) if cs else [pad_col])
    block_tiles = [-(-len(c) // TC_ITEMS) for c in block_cols]
    first = [sum(block_tiles[:b]) for b in range(nb + 1)]
    num_tiles = first[nb]
    off_ri = HDR
    off_tc = _align(off_ri + 4 * (rows + 1))
    off_em = _align(off_tc + 2 * TC_ITEMS * num_tiles)
    off_bt0 = _align(off_em + 4 * len(empty))
    off_tb = _align(off_bt0 + 4 * (nb + 1))
    off_tiles = _align(off_tb + 4 * num_tiles)
    total = _align(off_tiles + num_tiles * TC_TILE)
    out = bytearray(total)
    struct.pack_into("<IIiiiiqiiiiiiiiiiQQQQQQQ", out, 0,
                     MAGIC, VERSION, rows, K, G, n, nnzg, TC_ITEMS * TC_ROWS, num_tiles, rows - len(empty),
                     len(empty), TC_TILE, FLAG_TC | (1 << 8), row_begin, row_end, nb, 0,
                     off_ri, off_tc, off_em, off_bt0, off_tb, off_tiles, total)
    struct.pack_into(f"<{rows + 1}i", out, off_ri, *[v - g0 for v in ri_all[row_begin:row_end + 1]])
    if empty:
        struct.pack_into(f"<{len(empty)}i", out, off_em, *empty)
    struct.pack_into(f"<{nb + 1}i", out, off_bt0, *first)
    if num_tiles:
        struct.pack_into(f"<{num_tiles}i", out, off_tb, *[b for b in range(nb) for _ in range(block_tiles[b])])
    for blk in range(nb):
        cols = block_cols[blk]
        # (block row, column) -> group index
        where = {}
        for rr in range(TC_ROWS):
            r = blk * TC_ROWS + rr
            if r >= rows:
                break
            for g in range(ri_all[row_begin + r], ri_all[row_begin + r + 1]):
                where[(rr, int(gcols[g]))] = g
        for k in range(block_tiles[blk]):
            t = first[blk] + k
            base = off_tiles + t * TC_TILE
            for u in range(TC_ITEMS):
                item = k * TC_ITEMS + u
                col = cols[item] if item < len(cols) else pad_col
                struct.pack_into("<H", out, off_tc + 2 * (t * TC_ITEMS + u), col)
                if item >= len(cols):
                    continue
                for lane in range(LANES):
                    w = 0
                    for j in range(8):
                        rr = (lane >> 2) + 8 * (j & 1)
                        kk = 2 * (lane & 3) + 8 * ((j >> 1) & 1) + (j >> 2)
                        g = where.get((rr, col))
                        if g is None:
                            continue
                        e = g * G + kk
                        w |= ((int(codes[e // 2]) >> (4 * (e % 2))) & 0xF) << (4 * j)
                    struct.pack_into("<I", out, base + lane * 16 + u * 4, w)
                for gp in range(8):
                    vals = []
                    for h in range(2):
                        g = where.get((gp + 8 * h, col))
                        vals += [int(sc[g]), int(zr[g])] if g is not None else [0, 0]
                    struct.pack_into("<4H", out, base + 512 + gp * 32 + u * 8, *vals)
    return bytes(out)
