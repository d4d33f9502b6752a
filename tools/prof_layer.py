#!/usr/bin/env python
"""Launch the GQSA GEMV on one layer shape a fixed number of times (for ncu).

    python tools/prof_layer.py --rows 14336 --cols 4096 --bits 4 --sparsity 0.5 --launches 12
Weights rotate over enough device copies to exceed L2 (like bench.py).
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2412_17560_b200 import gqsa, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=14336)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--sparsity", type=float, default=0.5)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--mask", default="uniform")
    ap.add_argument("--launches", type=int, default=12)
    ap.add_argument("--time", action="store_true", help="also print CUDA-event µs per launch")
    a = ap.parse_args()
    tag = f"prof/{a.rows}x{a.cols}/{a.bits}/{a.sparsity}/{a.mask}"
    seed = synth.seed_for(tag)
    bsr = synth.make_layer(seed, a.rows, a.cols, bits=a.bits, sparsity=a.sparsity, mask=a.mask)
    x = synth.make_x(seed + 1, a.batch, a.cols)
    blob, desc = gqsa.pack(bsr)
    R = max(1, math.ceil(300e6 / blob.size))
    blobs = [torch.from_numpy(blob).cuda() for _ in range(R)]
    ws = torch.zeros(gqsa.workspace_size(desc, a.batch), dtype=torch.uint8, device="cuda")
    X = torch.from_numpy(x).view(torch.float16).cuda()
    Y = torch.empty(a.batch, a.rows, dtype=torch.float32, device="cuda")
    plan = gqsa.launch_plan(desc, a.batch)
    print(f"plan grid={plan.grid} active_warps={plan.active_warps} tiles={plan.num_tiles} "
          f"smem={plan.smem_bytes} stages={plan.stages} ctas/SM={plan.ctas_per_sm} R={R}", flush=True)
    for i in range(a.launches):
        gqsa.gemm_smallbatch(desc, blobs[i % R], X[:a.batch], Y, None, ws)
    torch.cuda.synchronize()
    if a.time:
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(R):
                gqsa.gemm_smallbatch(desc, blobs[i % R], X[:a.batch], Y, None, ws)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        e0.record(s)
        with torch.cuda.stream(s):
            for _ in range(reps):
                g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * R)
        nb = desc.nnzg * (16 * a.bits // 8 + 6) + 4 * (a.rows + 1) + 2 * a.batch * a.cols + 4 * a.batch * a.rows
        print(f"{a.rows}x{a.cols} W{a.bits}S{a.sparsity} B{a.batch}: {us:.3f} us/launch, "
              f"{nb / us / 1e3:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
