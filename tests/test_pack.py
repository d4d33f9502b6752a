"""Host-side boundary tests (CPU): the C-ABI library loads and exports every
symbol include/gqsa.h declares; gqsa_pack / gqsa_unpack round-trip bit-exactly;
the C++ packer's bytes equal the independent Python LAYOUT implementation;
validation rejects malformed BSR with the documented status."""
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import gqsa_oracle as O
from oracle.layout_reference import pack_reference, pack_reference_tc
from paper_2412_17560_b200 import gqsa, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "gqsa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gqsa_\w+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = _header_functions()
    assert "gqsa_gemv" in names and "gqsa_pack" in names and "gqsa_gemm_smallbatch" in names
    L = gqsa.lib()
    for n in names:
        assert hasattr(L, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", gqsa.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (gqsa_\w+)", out))
    assert set(names) <= exported
    assert set(gqsa.EXPORTS) == set(names)
    assert gqsa.lib().gqsa_version() == 3
    assert gqsa.status_string(-2) == "validation error"


def _eq_bsr(a, b):
    for k in ("rows", "cols", "group_size", "bits"):
        assert int(a[k]) == int(b[k]), k
    for k in ("row_index", "group_cols", "codes", "scales_f16", "zeros_f16"):
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k


CASES = [
    # rows, cols, bits, sparsity, mask, seed
    (256, 256, 4, 0.5, "uniform", 1),
    (256, 256, 2, 0.5, "uniform", 2),
    (64, 512, 4, 0.5, "skewed", 3),       # half the rows empty
    (37, 208, 4, 0.3, "row_balanced", 4),  # ragged last tile, odd rows
    (5, 16, 4, 0.0, "uniform", 5),         # K = G: one group per row
    (300, 32, 2, 0.8, "uniform", 6),       # many empty rows, tiny rows
    (8, 64, 4, 1.0, "uniform", 7),         # nnzg = 0
    (1, 4096, 4, 0.5, "uniform", 8),       # all groups in one row
    (256, 256, 8, 0.5, "uniform", 9),      # W8: four 512-B code planes per tile
    (37, 208, 8, 0.3, "row_balanced", 10),
]
# W4 at group sizes 8 and 32 (SURVEY §8(f) NEXT-1 group-size sweep)
G_CASES = [
    # rows, cols, G, sparsity, mask, seed
    (256, 512, 8, 0.5, "uniform", 21),
    (37, 264, 8, 0.3, "row_balanced", 22),
    (64, 1024, 32, 0.5, "skewed", 23),
    (3, 4096, 32, 0.5, "uniform", 24),
    (40, 96, 32, 0.0, "uniform", 25),
]


@pytest.mark.parametrize("rows,cols,bits,sp,mask,seed", CASES)
def test_roundtrip_and_reference_bytes(rows, cols, bits, sp, mask, seed):
    bsr = synth.make_layer(seed, rows, cols, bits=bits, sparsity=sp, mask=mask)
    blob, desc = gqsa.pack(bsr)
    assert desc.blob_bytes == blob.size and desc.nnzg == bsr["nnzg"]
    assert bytes(blob) == pack_reference(bsr)
    _eq_bsr(gqsa.unpack(blob), bsr)


@pytest.mark.parametrize("rows,cols,G,sp,mask,seed", G_CASES)
def test_group_sizes_roundtrip_and_reference_bytes(rows, cols, G, sp, mask, seed):
    bsr = synth.make_layer(seed, rows, cols, G=G, bits=4, sparsity=sp, mask=mask)
    blob, desc = gqsa.pack(bsr)
    assert desc.group_size == G and desc.tile_bytes == 128 * G // 2 + 512 + 256
    assert bytes(blob) == pack_reference(bsr)
    _eq_bsr(gqsa.unpack(blob), bsr)


def test_group_size_rejections():
    bsr = synth.make_layer(26, 16, 128, G=8, bits=2, sparsity=0.5)
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.pack(bsr)
    assert e.value.status == -3
    bsr = synth.make_layer(27, 16, 128, G=64, bits=4, sparsity=0.5)
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.pack(bsr)
    assert e.value.status == -3


def test_shard_ranges_rebase_and_reassemble():
    bsr = synth.make_layer(9, 96, 256, sparsity=0.5, mask="skewed")
    world = 4
    parts = []
    for r in range(world):
        lo, hi = synth.shard_rows(96, world, r)
        blob, d = gqsa.pack(bsr, lo, hi)
        assert (d.row_begin, d.row_end, d.rows) == (lo, hi, hi - lo)
        assert bytes(blob) == pack_reference(bsr, lo, hi)
        sh = gqsa.unpack(blob)
        _eq_bsr(sh, synth.slice_rows(bsr, lo, hi))
        parts.append(sh)
    # concatenating the shards reproduces the layer
    assert np.array_equal(np.concatenate([p["group_cols"] for p in parts]), bsr["group_cols"])
    offs = np.concatenate([[0], np.cumsum([p["nnzg"] for p in parts])])
    ri = np.concatenate([parts[0]["row_index"][:1]] + [p["row_index"][1:] + offs[i] for i, p in enumerate(parts)])
    assert np.array_equal(ri, bsr["row_index"])


def test_tile_fields_match_layout():
    """Spot-check the documented tile fields and slice tables directly."""
    bsr = synth.make_layer(10, 64, 256, sparsity=0.5)
    blob, d = gqsa.pack(bsr)
    assert d.tile_bytes == 1792 and d.tile_bytes % 128 == 0 and d.version == 3 and (d.flags >> 8) & 0xFF == 1
    counts = np.diff(bsr["row_index"])
    perm = blob[d.off_perm:d.off_perm + 4 * 64].view(np.int32)
    # slices hold rows by descending kept-group count
    assert list(counts[perm]) == sorted(counts, reverse=True)
    # slice tables: slice 0 (32 rows) spans ceil(longest / 4) tiles
    st0 = blob[d.off_slice_tile0:d.off_slice_tile0 + 4 * (d.num_slices + 1)].view(np.int32)
    ts = blob[d.off_tile_slice:d.off_tile_slice + 4 * d.num_tiles].view(np.int32)
    assert d.num_slices == 2 and st0[0] == 0 and st0[1] == -(-int(counts.max()) // 4) and st0[2] == d.num_tiles
    assert list(ts) == [0] * int(st0[1]) + [1] * int(st0[2] - st0[1])
    t0 = blob[d.off_tiles:d.off_tiles + d.tile_bytes]
    cols = t0[1024 + 512:].view(np.uint16)
    hit = 0
    for u in range(4):
        for lane in range(32):
            field = int(cols[lane * 4 + u])
            assert field % 16 == 0  # byte offset of the first x chunk
            f = field >> 4          # chunk index 2c + swap
            row = int(perm[lane])
            g0, g1 = bsr["row_index"][row], bsr["row_index"][row + 1]
            assert (f >> 1) in set(bsr["group_cols"][g0:g1].tolist())
            assert f & 1 == lane & 1  # swap = lane parity
            want = (((lane % 8) // 2 + u) % 4) + 4 * ((lane // 8) % 2)
            hit += ((f >> 1) % 4 == want % 4)  # the lane's target bank quad
    # bank-aware dealing: early slots almost always get the lane's target quad
    assert hit >= 0.9 * 128, hit
    # padding entries: s = z = 0, codes 0, column field = the zero block at byte 2K
    last = blob[d.off_tiles + (d.num_tiles - 1) * d.tile_bytes:d.off_tiles + d.num_tiles * d.tile_bytes]
    sz = last[1024:1536].view(np.uint16).reshape(32, 4, 2)
    pad = sz[:, :, 0] == 0
    assert pad.any()
    assert np.all(sz[pad][:, 1] == 0)
    assert np.all(last[1536:].view(np.uint16).reshape(32, 4)[pad] == 2 * 256)


def test_validation_errors():
    bsr = synth.make_layer(11, 16, 128, sparsity=0.5)
    with pytest.raises(gqsa.GQSAError) as e:
        bad = dict(bsr, row_index=bsr["row_index"].copy())
        bad["row_index"][5] = bad["row_index"][6] + 1  # non-monotone
        gqsa.pack(bad)
    assert e.value.status == -2
    bad = dict(bsr, group_cols=bsr["group_cols"].copy())
    bad["group_cols"][0] = 200  # >= K/G
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.pack(bad)
    assert e.value.status == -2
    bad = dict(bsr, scales_f16=bsr["scales_f16"].copy())
    bad["scales_f16"][3] = 0x7C00  # +inf scale
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.pack(bad)
    assert e.value.status == -2
    bad = dict(bsr, zeros_f16=bsr["zeros_f16"].copy())
    bad["zeros_f16"][3] = 0x7E00  # NaN zero
    with pytest.raises(gqsa.GQSAError):
        gqsa.pack(bad)
    bad = dict(bsr, bits=3)
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.pack(bad)
    assert e.value.status == -3
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.pack(bsr, 5, 3)
    assert e.value.status == -1


def test_read_desc_rejects_corruption():
    bsr = synth.make_layer(12, 16, 128, sparsity=0.5)
    blob, _ = gqsa.pack(bsr)
    for off, val in ((0, 0x00), (4, 0x07), (36, 0x7F)):
        b = blob.copy()
        b[off] = val
        with pytest.raises(gqsa.GQSAError):
            gqsa.read_desc(b)
    with pytest.raises(gqsa.GQSAError):
        gqsa.read_desc(blob[:blob.size - 256])
    # a corrupted slice table is caught by read_desc (the kernel trusts it)
    d = gqsa.read_desc(blob)
    b = blob.copy()
    b[d.off_tile_slice + 4 * (d.num_tiles - 1)] ^= 0x01
    with pytest.raises(gqsa.GQSAError):
        gqsa.read_desc(b)
    b = blob.copy()
    b[d.off_slice_tile0 + 4] ^= 0x02
    with pytest.raises(gqsa.GQSAError):
        gqsa.read_desc(b)
    # a padding entry that does not point at the zero block is caught by unpack
    last = d.off_tiles + (d.num_tiles - 1) * d.tile_bytes
    sz = blob[last + 1024:last + 1536].view(np.uint16).reshape(32, 4, 2)
    lane, u = map(int, np.argwhere(sz[:, :, 0] == 0)[0])
    b = blob.copy()
    b[last + 1536 + lane * 8 + u * 2] = 0x20
    with pytest.raises(gqsa.GQSAError):
        gqsa.unpack(b)


def test_lanes_per_row_rule():
    # long rows are dealt over several lanes: the longest slice has at most
    # `target` slots per lane, target = 16 / 128 / 256 for layers under 1.6 /
    # 4 / more tiles per warp of a 148 x 16-warp grid
    for rows, cols in ((256, 4096), (64, 14336), (8, 4096), (3, 256), (64, 512), (1, 32736),
                       (14336, 4096), (4096, 4096)):
        bsr = synth.make_layer(rows + cols, rows, cols, sparsity=0.5)
        _, d = gqsa.pack(bsr)
        S = (d.flags >> 8) & 0xFF
        tpw = d.nnzg / 128 / (148 * 16)
        target = 16 if tpw < 1.6 else 128 if tpw < 4 else 256
        longest = int(np.diff(bsr["row_index"]).max())
        assert -(-longest // S) <= target or S == 32
        assert S == 1 or -(-longest // (S // 2)) > target or S // 2 < 32 // (1 << (rows - 1).bit_length())
    assert target == 128 and S == 2  # 4096 x 4096: 1.7 tiles per warp


def test_workspace_size_is_layer_independent():
    # per launch: 256 B + one u32 arrival counter and two [B][32] 8-B records
    # per possible warp (148 SMs x 32 warps bound), whatever the layer
    _, d = gqsa.pack(synth.make_layer(13, 4096, 4096, sparsity=0.5))
    _, d2 = gqsa.pack(synth.make_layer(14, 64, 256, sparsity=0.3))
    for B in (1, 2, 8):
        want = 256 + 4736 * 4 + 4736 * 2 * B * 32 * 8
        assert gqsa.workspace_size(d, B) == want == gqsa.workspace_size(d2, B)


# ---------------------------------------------------------------- LAYOUT-TC
@pytest.mark.parametrize("rows,cols,sp,mask,seed", [
    (64, 256, 0.5, "uniform", 31), (37, 512, 0.5, "uniform", 32), (40, 96, 0.0, "uniform", 33),
    (100, 1024, 0.9, "uniform", 34), (64, 512, 0.5, "skewed", 35), (5, 64, 0.5, "uniform", 36),
    (48, 2048, 0.3, "row_balanced", 37), (16, 32736, 0.5, "uniform", 38)])
def test_tc_layout_reference_bytes_and_roundtrip(rows, cols, sp, mask, seed):
    """LAYOUT-TC: the C++ packer's bytes equal the independent Python
    implementation of the DESIGN.md §5.2 description, unpack inverts it
    exactly (empty blocks, ragged last block, S0 / S90, K at its maximum)."""
    bsr = synth.make_layer(seed, rows, cols, bits=4, sparsity=sp, mask=mask)
    blob, d = gqsa.pack(bsr, layout=gqsa.LAYOUT_TC)
    assert d.flags & 2 and d.tile_bytes == 768 and d.num_slices == -(-rows // 16)
    assert bytes(blob) == pack_reference_tc(bsr)
    _eq_bsr(gqsa.unpack(blob), bsr)
    lo, hi = rows // 3, rows - rows // 5  # a row shard, rebased
    blob2, d2 = gqsa.pack(bsr, lo, hi, layout=gqsa.LAYOUT_TC)
    assert bytes(blob2) == pack_reference_tc(bsr, lo, hi)
    _eq_bsr(gqsa.unpack(blob2), synth.slice_rows(bsr, lo, hi))


def test_tc_layout_fragment_words_and_errors():
    """Spot-check the fragment order: lane L's word of an item holds, in
    nibble j, A[(L >> 2) + 8 (j & 1)][2 (L & 3) + 8 ((j >> 1) & 1) + (j >> 2)]."""
    bsr = synth.make_layer(41, 16, 64, bits=4, sparsity=0.0, mode="exact_int")
    blob, d = gqsa.pack(bsr, layout=gqsa.LAYOUT_TC)
    q = O.unpack_codes(bsr["codes"], bsr["nnzg"] * 16, 4).reshape(16, 4, 16)  # [row][col][k] (S0: all kept)
    tile = blob[d.off_tiles:d.off_tiles + 768]
    for lane in range(32):
        w = int(tile[lane * 16:lane * 16 + 4].view(np.uint32)[0])  # item 0 = column 0
        for j in range(8):
            r, k = (lane >> 2) + 8 * (j & 1), 2 * (lane & 3) + 8 * ((j >> 1) & 1) + (j >> 2)
            assert (w >> (4 * j)) & 0xF == q[r, 0, k]
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.pack(synth.make_layer(42, 16, 64, bits=2, sparsity=0.5), layout=gqsa.LAYOUT_TC)
    assert e.value.status == -3
    with pytest.raises(gqsa.GQSAError) as e:
        gqsa.pack(bsr, layout=7)
    assert e.value.status == -1
    b = blob.copy()
    b[d.off_tile_slice] ^= 1  # tile 0 claims block 1
    with pytest.raises(gqsa.GQSAError):
        gqsa.read_desc(b)
    b = blob.copy()
    b[d.off_perm:d.off_perm + 2] = np.frombuffer(np.uint16(9).tobytes(), np.uint8)  # column beyond K/16
    with pytest.raises(gqsa.GQSAError):
        gqsa.read_desc(b)
