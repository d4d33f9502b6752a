#!/usr/bin/env python
"""Timeline of the bench step as ONE grouped launch (gqsa_gemm_grouped over the
LLaMA-3-8B shapes 4096x4096, 14336x4096, 4096x14336, W4S50, B = 1), from the
kernel's %globaltimer stamps (gqsa_debug_trace), in a CUDA graph of R
back-to-back steps on rotating weight copies (like bench.py).

    python tools/trace_step.py [--x-ready 1] [--steps 4]
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
SHAPES = [(4096, 4096), (14336, 4096), (4096, 14336)]
ORDERS = {"default": [0, 1, 2], "rev": [2, 1, 0], "q": [0], "gate": [1], "down": [2]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--x-ready", type=int, default=0)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--order", default="default", choices=sorted(ORDERS))
    a = ap.parse_args()
    packed, xs, ys = [], [], []
    for rows, cols in [SHAPES[i] for i in ORDERS[a.order]]:
        seed = synth.seed_for(f"llama3-8b/{rows}x{cols}/4/0.5/16/uniform")
        bsr = synth.make_layer(seed, rows, cols, bits=4, sparsity=0.5)
        packed.append(gqsa.pack(bsr))
        xs.append(torch.from_numpy(synth.make_x(seed + 1, 1, cols)).view(torch.float16).cuda())
        ys.append(torch.empty(1, rows, dtype=torch.float32, device="cuda"))
    set_bytes = sum(b.size for b, _ in packed)
    R = max(a.steps + 1, math.ceil(2.2 * 126 * 2**20 / set_bytes) + 1)
    copies = [[torch.from_numpy(b).cuda() for b, _ in packed] for _ in range(R)]
    ws = torch.zeros(gqsa.workspace_size(packed[0][1], 1), dtype=torch.uint8, device="cuda")
    calls = [gqsa.Grouped([(d, copies[r][i], xs[i], ys[i], None) for i, (_, d) in enumerate(packed)], ws,
                          x_ready=bool(a.x_ready)) for r in range(R)]
    total_tiles = sum(d.num_tiles for _, d in packed)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    plan = gqsa.launch_plan(packed[0][1], 1, x_ready=bool(a.x_ready))
    wpc = plan.warps_per_cta
    W = min(total_tiles, sms * wpc)
    bufs = [torch.zeros(W * 8, dtype=torch.int64, device="cuda") for _ in range(R)]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for r in range(R):
            gqsa.debug_trace(bufs[r])
            calls[r]()
    for _ in range(3):
        g.replay()
    gqsa.debug_trace(None)
    torch.cuda.synchronize()
    raw = np.stack([b.cpu().numpy().reshape(W, 8) for b in bufs])
    path = raw[1:, :, 7]
    T = raw[:, :, :7].astype(np.float64)
    t0 = T[0, :, 0].min()
    T = (T - t0) / 1e3
    print(f"grouped step: warps={W} ({wpc} per CTA, pipelined={plan.coresident}) tiles={total_tiles} "
          f"x_ready={a.x_ready} R={R}")
    print("step    " + "  ".join(f"{n:>17s}" for n in NAMES) + "   (min/median/max µs)")
    for i in range(a.steps):
        cols = [f"{T[i, :, k].min():5.2f}/{np.median(T[i, :, k]):5.2f}/{T[i, :, k].max():5.2f}" for k in range(7)]
        print(f"{i:6d}  " + "  ".join(f"{c:>17s}" for c in cols))
    ex = [T[i + 1, :, 5].max() - T[i, :, 5].max() for i in range(R - 1)]
    print("exit-to-exit per step (µs): median %.2f  (%s)" % (np.median(ex), " ".join(f"{e:.2f}" for e in ex[:8])))
    d = T[1:]
    print("median phase durations (µs): wait=%.2f stage=%.2f first_tile=%.2f loop=%.2f fixup=%.2f" % (
        np.median(d[..., 1] - d[..., 0]), np.median(d[..., 2] - d[..., 1]), np.median(d[..., 6] - d[..., 3]),
        np.median(d[..., 4] - d[..., 3]), np.median(d[..., 5] - d[..., 4])))
    q, r = divmod(total_tiles, W)
    ntile = np.array([q + (1 if w < r else 0) for w in range(W)], dtype=float)
    per = (d[..., 4] - d[..., 6]) / np.maximum(ntile[None, :] - 1, 1)
    print("loop µs per tile (p10/p50/p90/max): %.3f/%.3f/%.3f/%.3f; tiles per warp %d(+1 for %.0f%%)" % (
        np.percentile(per, 10), np.median(per), np.percentile(per, 90), per.max(), q, 100 * r / W))
    fx = d[..., 5] - d[..., 4]
    print("fixup (exit - loop end) p10/p50/p90/max: %.2f/%.2f/%.2f/%.2f" % (
        np.percentile(fx, 10), np.median(fx), np.percentile(fx, 90), fx.max()))
    for code, name in ((0, "no open slice"), (1, "fast path"), (2, "published, not last"),
                       (3, "published + collected"), (10, "head collected only"), (11, "fast + head"),
                       (12, "published + head"), (13, "collected + head")):
        m = path == code
        if m.any():
            print("  fixup %-22s %5.1f%% of warps: p50/p90/max %.2f/%.2f/%.2f us" % (
                name, 100 * m.mean(), np.median(fx[m]), np.percentile(fx[m], 90), fx[m].max()))
    if os.environ.get("GQSA_TRACE_PRO"):
        v = d[..., 3] - d[..., 0]
        print("  prologue: start -> tile loads issued p10/p50/p90 %.2f/%.2f/%.2f" % (
            np.percentile(v, 10), np.median(v), np.percentile(v, 90)))
        v = d[..., 1] - d[..., 3]
        print("  prologue: tile loads issued -> stamp 1 p10/p50/p90 %.2f/%.2f/%.2f" % (
            np.percentile(v, 10), np.median(v), np.percentile(v, 90)))
    if os.environ.get("GQSA_TRACE_FIX"):
        m = path == 1
        for k, name in ((3, "ready checked"), (6, "all_sync passed"), (2, "rows stored"), (5, "exit")):
            v = (d[..., k] - d[..., 4])[m]
            print("  fast path: loop end -> %-16s p50/p90 %.2f/%.2f" % (name, np.median(v), np.percentile(v, 90)))
    prev_exit = T[:-1, :, 5].max(axis=1)
    rel = T[1:, :, 1].min(axis=1) - prev_exit
    print("PDL release after previous step's last exit (µs):", " ".join(f"{v:.2f}" for v in rel[:5]))
    lat = T[1:, :, 5].max(axis=1) - np.median(T[1:, :, 5], axis=1)
    print("last exit - median exit (µs):", " ".join(f"{v:.2f}" for v in lat[:5]))
    wid_report(T, W, wpc)



def wid_report(T, W, wpc=16, sms=148):
    """Per warp-in-CTA (wid) and per CTA spread of the tile-loop speed and exit."""
    d = T[1:]
    loop = d[..., 4] - d[..., 3]
    ex = d[..., 5] - np.median(d[..., 5], axis=1, keepdims=True)
    wid = np.arange(W) % wpc
    print("wid : median loop µs / median exit - step median exit")
    print("  " + " ".join(f"{w:2d}:{np.median(loop[:, wid == w]):5.2f}/{np.median(ex[:, wid == w]):+.2f}" for w in range(wpc)))
    cta = np.arange(W) // wpc
    q, r = divmod(W and int(T.shape[1]) and 0 or 0, 1)
    steady = (d[..., 4] - d[..., 6])
    cl = np.array([np.median(loop[:, cta == c]) for c in range(cta.max() + 1)])
    cs = np.array([np.median(steady[:, cta == c]) for c in range(cta.max() + 1)])
    print("per-CTA steady loop (after tile 0) µs by CTA index (blocks of 8):",
          " ".join(f"{np.median(cs[i:i + 8]):.2f}" for i in range(0, len(cs), 8)))
    print("per-CTA median loop µs: p10/p50/p90/max %.2f/%.2f/%.2f/%.2f" % (
        np.percentile(cl, 10), np.median(cl), np.percentile(cl, 90), cl.max()))
    print("per-CTA loop µs by CTA index (blocks of 8):", " ".join(f"{np.median(cl[i:i + 8]):.2f}" for i in range(0, len(cl), 8)))
    sm_tile = d[..., 4] - d[..., 6]
    print("per-CTA exit - median:", " ".join(f"{np.median(ex[:, cta == c]):+.1f}" for c in range(0, cta.max() + 1, 4)))


if __name__ == "__main__":
    main()
