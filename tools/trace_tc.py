#!/usr/bin/env python
"""Timeline of the LAYOUT-TC small-batch kernel (gqsa_tc.cu) from its
%globaltimer stamps (gqsa_debug_trace): start, staged, loop start, loop end,
exit -- per launch in a CUDA graph of back-to-back launches on rotating copies.

    python tools/trace_tc.py --rows 14336 --cols 4096 --batch 8
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=14336)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=8)
    a = ap.parse_args()
    bsr = synth.make_layer(synth.seed_for(f"llama3-8b/{a.rows}x{a.cols}/4/0.5/16/uniform"), a.rows, a.cols)
    blob, desc = gqsa.pack(bsr, layout=gqsa.LAYOUT_TC)
    R = max(4, math.ceil(300e6 / blob.size))
    blobs = [torch.from_numpy(blob).cuda() for _ in range(R)]
    ws = torch.zeros(gqsa.workspace_size(desc, a.batch), dtype=torch.uint8, device="cuda")
    X = torch.from_numpy(synth.make_x(1, a.batch, a.cols)).view(torch.float16).cuda()
    Y = torch.empty(a.batch, a.rows, dtype=torch.float32, device="cuda")
    plan = gqsa.launch_plan(desc, a.batch)
    W = plan.active_warps
    bufs = [torch.zeros(W * 8, dtype=torch.int64, device="cuda") for _ in range(R)]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(R):
            gqsa.debug_trace(bufs[i])
            gqsa.gemm_ex(desc, blobs[i], X, Y, ws=ws, stream=s)
    for _ in range(3):
        g.replay()
    gqsa.debug_trace(None)
    torch.cuda.synchronize()
    T = np.stack([b.cpu().numpy().reshape(W, 8) for b in bufs]).astype(np.float64)
    t0 = T[0, :, 0].min()
    Traw = T.copy()
    T = (T - t0) / 1e3
    d = T[1:]
    print(f"TC {a.rows}x{a.cols} B={a.batch}: warps={W} tiles={desc.num_tiles} blocks={desc.num_slices} "
          f"blob={blob.size / 1e6:.1f} MB, launches={plan.launches}")
    ex = [T[i + 1, :, 5].max() - T[i, :, 5].max() for i in range(R - 1)]
    print("exit-to-exit per launch (µs): median %.2f" % np.median(ex))
    print("median phases (µs): start->staged %.2f  staged->loop %.2f  loop %.2f  fixup %.2f" % (
        np.median(d[..., 2] - d[..., 0]), np.median(d[..., 3] - d[..., 2]), np.median(d[..., 4] - d[..., 3]),
        np.median(d[..., 5] - d[..., 4])))
    q, r = divmod(desc.num_tiles, W)
    per = (d[..., 4] - d[..., 3]) / q
    print("loop µs per tile p10/p50/p90: %.3f/%.3f/%.3f (tiles per warp %d)" % (
        np.percentile(per, 10), np.median(per), np.percentile(per, 90), q))
    print("last exit - median exit (µs): %.2f" % np.median(d[..., 5].max(axis=1) - np.median(d[..., 5], axis=1)))
    # per launch, relative to its median "staged" stamp
    rel = d - np.median(d[..., 2], axis=1)[:, None, None]
    for k, name in ((0, "start"), (2, "staged"), (4, "loop end"), (5, "exit")):
        v = rel[..., k]
        print("  %-8s p1 %.2f  p50 %.2f  p99 %.2f  max %.2f" % (
            name, np.median(np.percentile(v, 1, axis=1)), np.median(np.percentile(v, 50, axis=1)),
            np.median(np.percentile(v, 99, axis=1)), np.median(v.max(axis=1))))
    late = np.argsort(rel[1, :, 5])[-8:]
    print("  latest exits of one launch: warp, start, staged, loop, fixup, exit; fix-up stamps (arrived, tail collect, head collect; -: not reached)")
    for w in late:
        r = rel[1, w]
        raw = Traw[2, w]
        fx = " ".join("%6.2f" % ((raw[k] - raw[4]) / 1e3) if raw[k] > 0 else "     -" for k in (1, 6, 7))
        print("   %5d %6.2f %6.2f %6.2f %6.2f %6.2f | %s | raw7 %d" % (w, r[0], r[2], r[4] - r[3], r[5] - r[4], r[5], fx, raw[7]))


if __name__ == "__main__":
    main()
