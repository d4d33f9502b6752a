"""Host-side model check of the Stream-K fix-up protocols (CPU; no kernel runs).

The stream kernel (paper_2412_17560_b200/csrc/gqsa_stream.cu) cuts the
launch's tile stream into equal (+-1 tile) contiguous warp ranges regardless
of slice boundaries (task-centric partition, PAPER.md:161 [§3.5 Stream-K],
PAPER.md:510 [App. J]); a slice split over several ranges is finished by the
fix-up.  This test replays, on random partitions, the
bookkeeping of the CTA-level fix-up of whole-SM launches:

  * every warp keeps at most a head piece (a slice begun upstream and closed
    in its range) and a tail piece (the slice open at its range end; a
    "middle" piece when that slice also began upstream);
  * the first warp of a slice's part inside a CTA (the slice's owner, or warp 0
    for a slice begun in an earlier CTA) walks the following warps' pieces in
    warp order until the slice closes or the CTA ends;
  * a slice that crosses CTA boundaries gets exactly one piece from every CTA
    c0..c1 it touches; c0..c1-1 publish theirs as records and c1, the CTA
    holding the slice's last tile, adds them (it waits only for lower CTAs).

It asserts that every tile of every slice is counted exactly once, that a
crossing slice has one piece per touched CTA, and that its collector is c1.
"""
import random


def _model(total, slice_ends, W, nwarps):
    active = min(total, nwarps)
    q, r = divmod(total, active)

    def rng(w):
        b = w * q + min(w, r)
        return b, b + q + (1 if w < r else 0)

    def warp_of_tile(t):
        big = r * (q + 1)
        return t // (q + 1) if t < big else r + (t - big) // q

    starts = [0] + slice_ends[:-1]

    def slice_of(t):
        return next(i for i, (s, e) in enumerate(zip(starts, slice_ends)) if s <= t < e)

    stores, records = {}, {}
    for c in range((active + W - 1) // W):
        base = c * W
        nw = min(W, active - base)
        meta = []
        for lw in range(nw):
            b, e = rng(base + lw)
            cur = slice_of(b)
            fr = starts[cur] < b
            head = tail = None
            acc = set()
            for t in range(b, e):
                acc.add(t)
                if t + 1 == slice_ends[cur]:
                    if fr:
                        head = (cur, frozenset(acc))
                    else:
                        stores.setdefault(cur, []).append(frozenset(acc))
                    acc, fr = set(), False
                    if t + 1 < e:
                        cur += 1
            if acc:
                tail = (cur, frozenset(acc), fr)
            meta.append((head, tail))
        for lw in range(nw):
            head, tail = meta[lw]
            if lw == 0 and head:  # warp 0's head piece: the CTA's only piece of that slice
                records.setdefault(head[0], []).append((c, head[1]))
            if tail and (not tail[2] or lw == 0):
                s, v, closed = tail[0], set(tail[1]), False
                k = lw + 1
                while k < nw and not closed:
                    h, tt = meta[k]
                    if tt and tt[2]:  # middle piece
                        assert tt[0] == s
                        v |= tt[1]
                    else:
                        assert h and h[0] == s
                        v |= h[1]
                        closed = True
                    k += 1
                if closed and not tail[2]:
                    stores.setdefault(s, []).append(frozenset(v))
                else:
                    records.setdefault(s, []).append((c, frozenset(v)))
    for s, (st, en) in enumerate(zip(starts, slice_ends)):
        full = set(range(st, en))
        if s in records:
            assert s not in stores
            c0, c1 = warp_of_tile(st) // W, warp_of_tile(en - 1) // W
            assert sorted(c for c, _ in records[s]) == list(range(c0, c1 + 1))
            # the collector is c1, the CTA holding the slice's last tile; it waits only for c0..c1-1
            assert [c for c, v in records[s] if en - 1 in v] == [c1]
            seen = set()
            for _, v in records[s]:
                assert not seen & v
                seen |= v
            assert seen == full
        else:
            assert len(stores[s]) == 1 and set(stores[s][0]) == full


def test_cta_fixup_counts_every_tile_once():
    rnd = random.Random(20241217560)
    for _ in range(1500):
        ns = rnd.randint(1, 60)
        ends, a = [], 0
        for _ in range(ns):
            a += rnd.randint(1, rnd.choice([1, 4, 32, 128]))
            ends.append(a)
        W = rnd.randint(1, 20)
        _model(a, ends, W, W * rnd.randint(1, 10))


def test_cta_fixup_llama_shapes():
    # 4096^2 at W4S50 on 148 SMs x 20 warps: 4096 tiles, 32-tile slices
    _model(4096, [32 * (i + 1) for i in range(128)], 20, 148 * 20)
    # one slice spanning every CTA (a single long row block)
    _model(5000, [5000], 20, 148 * 20)
