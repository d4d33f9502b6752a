#!/usr/bin/env python
"""Timeline of GQSA launches from the kernel's %globaltimer stamps (gqsa_debug_trace).

    python tools/trace_layer.py --rows 14336 --cols 4096 [--launches 6]
For a CUDA graph of back-to-back launches (rotating weight copies, PDL on),
prints per launch: start spread, PDL-wait release, activation staging, first
tile arrival, tile-loop end and exit (µs relative to the first launch's
earliest start; percentiles over warps).
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_17560_b200 import gqsa, synth  # noqa: E402

NAMES = ["start", "pdl_wait", "x_staged", "loop0", "loop_end", "exit", "tile0_done"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=14336)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--sparsity", type=float, default=0.5)
    ap.add_argument("--launches", type=int, default=6)
    ap.add_argument("--eager", action="store_true", help="stream launches instead of a CUDA graph")
    a = ap.parse_args()
    seed = synth.seed_for(f"trace/{a.rows}x{a.cols}")
    bsr = synth.make_layer(seed, a.rows, a.cols, bits=a.bits, sparsity=a.sparsity)
    x = synth.make_x(seed + 1, 1, a.cols)
    blob, desc = gqsa.pack(bsr)
    R = max(a.launches, math.ceil(300e6 / blob.size))
    blobs = [torch.from_numpy(blob).cuda() for _ in range(R)]
    ws = torch.zeros(gqsa.workspace_size(desc, 1), dtype=torch.uint8, device="cuda")
    X = torch.from_numpy(x).view(torch.float16).cuda()
    Y = torch.empty(1, a.rows, dtype=torch.float32, device="cuda")
    plan = gqsa.launch_plan(desc, 1)
    W = plan.active_warps
    bufs = [torch.zeros(W * 8, dtype=torch.int64, device="cuda") for _ in range(R)]
    s = torch.cuda.Stream()
    if a.eager:  # plain stream launches (PDL attribute on each)
        for _ in range(2):
            with torch.cuda.stream(s):
                for i in range(R):
                    gqsa.debug_trace(bufs[i])
                    gqsa.gemm_smallbatch(desc, blobs[i], X, Y, None, ws)
            torch.cuda.synchronize()
    else:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(R):
                gqsa.debug_trace(bufs[i])
                gqsa.gemm_smallbatch(desc, blobs[i], X, Y, None, ws)
        for _ in range(3):
            g.replay()
    gqsa.debug_trace(None)
    torch.cuda.synchronize()
    T = np.stack([b.cpu().numpy().reshape(W, 8)[:, :7] for b in bufs])  # [R][W][7]
    t0 = T[0, :, 0].min()
    T = (T - t0) / 1e3
    print(f"{a.rows}x{a.cols} W{a.bits}: grid={plan.grid} warps={W} stages={plan.stages} "
          f"ctas/SM={plan.ctas_per_sm} tiles={plan.num_tiles}")
    print("launch  " + "  ".join(f"{n:>17s}" for n in NAMES) + "   (min/median/max µs)")
    for i in range(min(R, a.launches)):
        cols = []
        for k in range(7):
            v = T[i, :, k]
            cols.append(f"{v.min():5.2f}/{np.median(v):5.2f}/{v.max():5.2f}")
        print(f"{i:6d}  " + "  ".join(f"{c:>17s}" for c in cols))
    per = [(T[i + 1, :, 5].max() - T[i, :, 5].max()) for i in range(min(R, a.launches) - 1)]
    print("exit-to-exit per launch (µs):", " ".join(f"{p:.2f}" for p in per))
    d = T[1:, :, :]
    print("median phase durations (µs): wait=%.2f stage=%.2f first_tile=%.2f loop=%.2f fixup=%.2f" % (
        np.median(d[..., 1] - d[..., 0]), np.median(d[..., 2] - d[..., 1]), np.median(d[..., 6] - d[..., 3]),
        np.median(d[..., 4] - d[..., 3]), np.median(d[..., 5] - d[..., 4])))
    e = d
    q, r = divmod(plan.num_tiles, W)  # Stream-K units are tiles
    ntile = np.array([q + (1 if w < r else 0) for w in range(W)], dtype=float)
    loop = e[..., 4] - e[..., 6]  # steady state: after the first tile
    per = loop / np.maximum(ntile[None, :] - 1, 1)
    print("loop µs per tile (p10/p50/p90/max): %.3f/%.3f/%.3f/%.3f; warps with q+1 tiles: %.0f%%" % (
        np.percentile(per, 10), np.median(per), np.percentile(per, 90), per.max(), 100 * r / W))
    sm = np.arange(W) // plan.warps_per_cta
    per_cta = np.array([np.median(per[:, sm == c]) for c in range(plan.grid)])
    print("per-CTA median µs/tile: min %.3f max %.3f (spread %.0f%%)" % (
        per_cta.min(), per_cta.max(), 100 * (per_cta.max() / per_cta.min() - 1)))
    ex = T[1:, :, 5]  # exit times [launch][warp]
    cta_max = np.stack([ex[:, sm == c].max(axis=1) for c in range(plan.grid)], axis=1)
    cta_med = np.stack([np.median(ex[:, sm == c], axis=1) for c in range(plan.grid)], axis=1)
    print("exit spread (µs, median over launches): within-CTA max-median %.2f; across CTAs "
          "(CTA max) p10/p50/max - launch median %.2f/%.2f/%.2f" % (
              np.median(cta_max - cta_med),
              np.median(np.percentile(cta_max, 10, axis=1) - np.median(ex, axis=1)),
              np.median(np.median(cta_max, axis=1) - np.median(ex, axis=1)),
              np.median(cta_max.max(axis=1) - np.median(ex, axis=1))))
    # the slowest warps: which phase made them late, and their fix-up path
    path = np.stack([b.cpu().numpy().reshape(W, 8)[:, 7] for b in bufs])[1:]
    late = ex - np.median(ex, axis=1, keepdims=True)
    cut = np.percentile(late, 95)
    m = late >= cut
    le = d[..., 4] - np.median(d[..., 4], axis=1, keepdims=True)
    st = d[..., 2] - np.median(d[..., 2], axis=1, keepdims=True)
    print("slowest 5%% of warps (exit >= median + %.2f us): loop end vs median %.2f, staged vs median %.2f, "
          "fix-up (exit - loop end) %.2f us (medians); fix paths %s" % (
              cut, np.median(le[m]), np.median(st[m]), np.median((d[..., 5] - d[..., 4])[m]),
              {int(k): int(v) for k, v in zip(*np.unique(path[m], return_counts=True))}))
    if os.environ.get("GQSA_TRACE_FIX"):  # library built with -DGQSA_TRACE_FIX: slot 6 = arrival returned,
        raw = np.stack([b.cpu().numpy().reshape(W, 8) for b in bufs])[1:]  # slot 2 = re-polls in collect
        arr = (raw[..., 6].astype(np.float64) - t0) / 1e3 - d[..., 4]
        m3 = m & (path == 3)
        if m3.any():
            ent = (raw[..., 2].astype(np.float64) - t0) / 1e3
            b1 = (raw[..., 1].astype(np.float64) - t0) / 1e3
            arr_abs = arr + d[..., 4]
            print("  slow collectors (medians, us): loop end -> arrival returned %.2f -> collect entry %.2f -> "
                  "first batch summed %.2f -> exit %.2f" % (
                      np.median(arr[m3]), np.median((ent - arr_abs)[m3]), np.median((b1 - ent)[m3]),
                      np.median((d[..., 5] - b1)[m3])))
    if os.environ.get("GQSA_TRACE_FIX"):  # CTA-level fix-up: 6 = pieces in smem, 3 = arrival returned
        raw = np.stack([b.cpu().numpy().reshape(W, 8) for b in bufs])[1:].astype(np.float64)
        rel = (raw - t0) / 1e3
        for paths, name in (((5, 15), "cross-CTA reducers"), ((4, 14), "in-CTA reducers")):
            m5 = m & np.isin(path, paths)
            if not m5.any():
                continue
            print("  slow %s (n=%d, medians, us): loop end -> pieces in smem %.2f -> arrival returned %.2f "
                  "-> exit %.2f" % (name, m5.sum(), np.median((rel[..., 6] - d[..., 4])[m5]),
                                    np.median((rel[..., 3] - rel[..., 6])[m5]),
                                    np.median((d[..., 5] - rel[..., 3])[m5])))
        allr = np.isin(path, (5, 15))
        print("  all cross-CTA reducers: pieces->arrival %.2f, arrival->exit %.2f (medians); "
              "exit minus launch-median exit p50/p95 %.2f/%.2f" % (
                  np.median((rel[..., 3] - rel[..., 6])[allr]), np.median((d[..., 5] - rel[..., 3])[allr]),
                  np.median(late[allr]), np.percentile(late[allr], 95)))
    prev_exit = T[:-1, :, 5].max(axis=1)
    rel = T[1:, :, 1].min(axis=1) - prev_exit
    print("PDL release after previous launch's last exit (µs):", " ".join(f"{r:.2f}" for r in rel[:5]))


if __name__ == "__main__":
    main()
