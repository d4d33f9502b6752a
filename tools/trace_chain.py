#!/usr/bin/env python
"""Timeline of gqsa_gemm_chain launches from %globaltimer stamps (gqsa_debug_trace).

    python tools/trace_chain.py [--launches 6]
The bench's step (LLaMA-3-8B 4096x4096, 14336x4096, 4096x14336; W4S50, B=1)
as one chain launch, R rotating weight copies in a CUDA graph.  Per launch and
item: barrier passed (staging starts), activations staged, warp done with
the item (min/median/max over warps, µs from the first launch's first stamp).
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

SHAPES = [(4096, 4096), (14336, 4096), (4096, 14336)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", type=int, default=6)
    a = ap.parse_args()
    packed, xs, ys = [], [], []
    for (n, k) in SHAPES:
        seed = synth.seed_for(f"trace/{n}x{k}")
        blob, desc = gqsa.pack(synth.make_layer(seed, n, k, bits=4, sparsity=0.5))
        packed.append((blob, desc))
        xs.append(torch.from_numpy(synth.make_x(seed + 1, 1, k)).view(torch.float16).cuda())
        ys.append(torch.empty(1, n, dtype=torch.float32, device="cuda"))
    set_bytes = sum(b.size for b, _ in packed)
    R = max(a.launches, math.ceil(300e6 / set_bytes))
    copies = [[torch.from_numpy(b).cuda() for b, _ in packed] for _ in range(R)]
    items = [[(packed[i][1], copies[r][i], xs[i], ys[i], None, 1) for i in range(3)] for r in range(R)]
    ws = torch.zeros(gqsa.chain_workspace_size(items[0], 1), dtype=torch.uint8, device="cuda")
    TW = 148 * 16 * 2
    bufs = [torch.zeros(TW * 3 * 4, dtype=torch.int64, device="cuda") for _ in range(R)]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        gqsa.gemm_chain(items[0], ws)  # warm-up (attributes)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for r in range(R):
            gqsa.debug_trace(bufs[r])
            gqsa.gemm_chain(items[r], ws)
    gqsa.debug_trace(None)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    T = [b.cpu().numpy().reshape(-1, 3, 4) for b in bufs]
    W = int((T[0][:, 0, 0] != 0).sum())
    T = np.stack([t[:W] for t in T]).astype(np.float64)  # [R][W][item][4]
    t0 = T[0, :, 0, 0].min()
    T = (T - t0) / 1e3
    names = ["barrier", "staged", "done"]
    for r in range(min(R, a.launches)):
        line = []
        for j in range(3):
            cells = []
            for k in range(3):
                v = T[r, :, j, k]
                cells.append(f"{v.min():6.2f}/{np.median(v):6.2f}/{v.max():6.2f}")
            line.append(" ".join(cells))
        print(f"launch {r}: " + " | ".join(line))
    ends = T[:, :, 2, 2].max(axis=1)
    print("launch end-to-end (last done) deltas µs:", " ".join(f"{d:.2f}" for d in np.diff(ends)[:8]))
    d = T[1:]
    for j in range(3):
        print("item %d: barrier->staged %.2f  staged->median done %.2f  median->max done %.2f  "
              "prev max done -> barrier min %.2f" % (
                  j, np.median(d[:, :, j, 1] - d[:, :, j, 0]),
                  np.median(np.median(d[:, :, j, 2], axis=1) - d[:, :, j, 1].min(axis=1)),
                  np.median(d[:, :, j, 2].max(axis=1) - np.median(d[:, :, j, 2], axis=1)),
                  np.median(d[:, :, j, 0].min(axis=1) - (d[:, :, j - 1, 2].max(axis=1) if j > 0
                                                         else T[:-1, :, 2, 2].max(axis=1)))))


if __name__ == "__main__":
    main()
