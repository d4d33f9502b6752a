#!/usr/bin/env python
"""Secondary measurements of SURVEY §8(d)/(f) on one GPU (not the bench line).

    python tools/sweep.py --out profiles/r01_sweep [--quick]

A. W4S50 / W4S30 / W2S50 / W8S50 x batch 1, 2, 4, 8 at the LLaMA-3-8B shapes.
B. Partition ablation (App. J): Stream-K versus
   Slice-K on uniform, row-balanced and skewed masks (W4S50, batch 1).
C. Sparsity sweep at 4096x4096 W4 (Fig. 6 trend): S = 0 .. 0.8,
   speed-up over this build's own S = 0 (dense-equivalent) launch.
H. Group size G = 8 / 16 / 32 at W4S50, B = 1.
D. Saliency-selected masks (the method's own front-end, PAPER.md:74-93:
   Eq. 4 + group means + exact-count pruning, frontend.compress) on synthetic
   dense layers with per-row scale imbalance and calibration activations with
   outlier channels: row-length spread, Stream-K vs Slice-K (W4S50, B = 1).

Every number: µs per launch from a CUDA graph of R launches over rotating
device copies of the blob (> 2x L2), PDL on, CUDA events on the launching
stream; GB/s = counted bytes (bench.counted_bytes) / µs.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import counted_bytes, peaks  # noqa: E402
from paper_2412_17560_b200 import frontend, gqsa, synth  # noqa: E402

SHAPES = [(4096, 4096), (14336, 4096), (4096, 14336)]


def measure(bsr, B, partition=gqsa.PARTITION_STREAM_K, reps=20, layout=gqsa.LAYOUT_STREAM):
    rows, cols = int(bsr["rows"]), int(bsr["cols"])
    blob, desc = gqsa.pack(bsr, layout=layout)
    R = max(2, math.ceil(300e6 / blob.size))
    blobs = [torch.from_numpy(blob).cuda() for _ in range(R)]
    ws = torch.zeros(gqsa.workspace_size(desc, B), dtype=torch.uint8, device="cuda")
    seed = synth.seed_for(f"sweep-x/{rows}x{cols}/{B}")
    X = torch.from_numpy(synth.make_x(seed, B, cols)).view(torch.float16).cuda()
    Y = torch.empty(B, rows, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(R):
            gqsa.gemm_ex(desc, blobs[i], X, Y, partition, ws=ws, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(R):
            gqsa.gemm_ex(desc, blobs[i], X, Y, partition, ws=ws, stream=s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * R)
    nb = counted_bytes(rows, cols, int(bsr["nnzg"]), int(bsr["bits"]), B)
    del blobs
    return dict(rows=rows, cols=cols, bits=int(bsr["bits"]), nnzg=int(bsr["nnzg"]), B=B, us=round(us, 3),
                counted_bytes=nb, gbs=round(nb / us / 1e3, 1), tiles=desc.num_tiles,
                blob_bytes=int(desc.blob_bytes))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None, help="write <out>.md and <out>.jsonl")
    ap.add_argument("--quick", action="store_true", help="batch 1 and 8 only")
    ap.add_argument("--sections", default="ABCDH", help="subset of A, B, C, D, H to run")
    a = ap.parse_args()
    peak, src = peaks()
    recs = []
    lines = ["# Secondary sweeps (tools/sweep.py; B200, 1 GPU)", "",
             f"GB/s = counted bytes / µs; frac = GB/s / {peak:.1f} ({src}). "
             "CUDA graph of R launches over rotating blob copies (> 2x L2), PDL on.", ""]

    def emit(section, r):
        r["section"] = section
        r["frac"] = round(r["gbs"] / peak, 4)
        recs.append(r)
        print(json.dumps(r), flush=True)

    if "A" in a.sections:  # quantisation settings x batch
        lines += ["## A. Quantisation setting x batch (Stream-K)", "",
                  "| setting | shape | B=1 µs (GB/s) | B=2 | B=4 | B=8 |", "|---|---|---|---|---|---|"]
        batches = [1, 8] if a.quick else [1, 2, 4, 8]
        for bits, sp in ((4, 0.5), (4, 0.3), (2, 0.5), (8, 0.5)):
            for rows, cols in SHAPES:
                bsr = synth.make_layer(synth.seed_for(f"llama3-8b/{rows}x{cols}/{bits}/{sp}/16/uniform"),
                                       rows, cols, bits=bits, sparsity=sp)
                cells = {}
                for B in batches:
                    r = measure(bsr, B)
                    r["setting"] = f"W{bits}S{int(sp * 100)}"
                    emit("A", r)
                    cells[B] = f"{r['us']:.2f} ({r['gbs']:.0f})"
                lines.append(f"| W{bits}S{int(sp * 100)} | {rows}x{cols} | " +
                             " | ".join(cells.get(B, "-") for B in (1, 2, 4, 8)) + " |")
        lines.append("")

    if "T" in a.sections:  # small-batch tensor-core layout vs the CUDA-core stream
        lines += ["## T. Small batch: LAYOUT-TC (mma.sync) vs the CUDA-core stream, W4S50", "",
                  "GB/s over the counted (BSR) bytes; the TC blob reads about 2x them (blob MB column).", "",
                  "| shape | layout | blob MB | B=1 µs | B=2 | B=4 | B=8 |", "|---|---|---|---|---|---|---|"]
        for rows, cols in SHAPES:
            bsr = synth.make_layer(synth.seed_for(f"llama3-8b/{rows}x{cols}/4/0.5/16/uniform"),
                                   rows, cols, bits=4, sparsity=0.5)
            for lay, name in ((gqsa.LAYOUT_STREAM, "stream"), (gqsa.LAYOUT_TC, "tc")):
                cells, mb = {}, 0.0
                for B in (1, 2, 4, 8):
                    r = measure(bsr, B, layout=lay)
                    r["layout"] = name
                    emit("T", r)
                    cells[B] = f"{r['us']:.2f}"
                    mb = r["blob_bytes"] / 1e6
                lines.append(f"| {rows}x{cols} | {name} | {mb:.1f} | " + " | ".join(cells[B] for B in (1, 2, 4, 8)) + " |")
        lines.append("")

    if "B" in a.sections:  # partition ablation
        lines += ["## B. Partition ablation, W4S50, B = 1 (Stream-K vs Slice-K)", "",
                  "| mask | shape | Stream-K µs | Slice-K µs | Slice-K / Stream-K |", "|---|---|---|---|---|"]
        for mask in ("uniform", "row_balanced", "skewed"):
            for rows, cols in SHAPES:
                bsr = synth.make_layer(synth.seed_for(f"llama3-8b/{rows}x{cols}/4/0.5/16/{mask}"),
                                       rows, cols, bits=4, sparsity=0.5, mask=mask)
                rs = measure(bsr, 1, gqsa.PARTITION_STREAM_K)
                rk = measure(bsr, 1, gqsa.PARTITION_SLICE_K)
                for name, r in (("stream_k", rs), ("slice_k", rk)):
                    r.update(mask=mask, partition=name)
                    emit("B", r)
                lines.append(f"| {mask} | {rows}x{cols} | {rs['us']:.2f} | {rk['us']:.2f} | "
                             f"{rk['us'] / rs['us']:.2f}x |")
        lines.append("")

    if "C" in a.sections:  # sparsity sweep
        lines += ["## C. Sparsity sweep, 4096x4096 W4, B = 1 (Fig. 6 trend)", "",
                  "| S | nnzg | counted MB | µs | GB/s | speed-up vs S=0 |", "|---|---|---|---|---|---|"]
        base = None
        for sp in (0.0, 0.2, 0.3, 0.4, 0.5, 0.6, 0.8):
            bsr = synth.make_layer(synth.seed_for(f"sweep-s/4096/{sp}"), 4096, 4096, bits=4, sparsity=sp)
            r = measure(bsr, 1)
            r["sparsity"] = sp
            emit("C", r)
            base = base or r["us"]
            lines.append(f"| {sp:.1f} | {r['nnzg']} | {r['counted_bytes'] / 1e6:.2f} | {r['us']:.2f} | "
                         f"{r['gbs']:.0f} | {base / r['us']:.2f}x |")
        lines.append("")

    if "D" in a.sections:  # saliency-selected masks (the method's own front-end)
        lines += ["## D. Saliency-selected masks (Eq. 4 front-end), W4S50, B = 1", "",
                  "Dense W: N(0, sigma_r^2), sigma_r = 0.02*10^U(-1,1), 0.1 % of input columns x4; "
                  "calibration X: 256 samples, N(0,1) with 0.5 % channels x20; H = 2/N X^T X + 1 % "
                  "damping; frontend.compress (C ABI). Row spread = kept groups per row (min / mean / max).", "",
                  "| shape | rows kept min/mean/max | empty rows | Stream-K µs (GB/s) | Slice-K µs | "
                  "Slice-K / Stream-K | compress s |", "|---|---|---|---|---|---|---|"]
        import time
        import numpy as np
        for rows, cols in SHAPES:
            seed = synth.seed_for(f"saliency/{rows}x{cols}")
            W = synth.make_dense(seed, rows, cols)
            d = frontend.hessian_inv_diag(synth.make_calib(seed + 1, 256, cols), device="cuda")
            t0 = time.perf_counter()
            bsr = frontend.compress(W, d, 0.5, 4)
            tc = time.perf_counter() - t0
            lens = np.diff(bsr["row_index"])
            rs = measure(bsr, 1, gqsa.PARTITION_STREAM_K)
            rk = measure(bsr, 1, gqsa.PARTITION_SLICE_K)
            for name, r in (("stream_k", rs), ("slice_k", rk)):
                r.update(mask="saliency", partition=name, compress_s=round(tc, 2),
                         row_min=int(lens.min()), row_mean=float(lens.mean()), row_max=int(lens.max()),
                         empty_rows=int((lens == 0).sum()))
                emit("D", r)
            lines.append(f"| {rows}x{cols} | {lens.min()}/{lens.mean():.0f}/{lens.max()} | "
                         f"{int((lens == 0).sum())} | {rs['us']:.2f} ({rs['gbs']:.0f}) | {rk['us']:.2f} | "
                         f"{rk['us'] / rs['us']:.2f}x | {tc:.2f} |")
        lines.append("")

    if "H" in a.sections:  # group size, W4S50, B = 1
        lines += ["## H. Group size G = 8 / 16 / 32, W4S50, B = 1", "",
                  "Counted bytes per kept group: G/2 code bytes + 6 (s, z, column): 1.25 / 0.875 / 0.69 B per "
                  "weight. The paper keeps G = 16 (PAPER.md:170).", "",
                  "| shape | G = 8 µs (GB/s) | G = 16 | G = 32 |", "|---|---|---|---|"]
        for rows, cols in SHAPES:
            cells = []
            for G in (8, 16, 32):
                bsr = synth.make_layer(synth.seed_for(f"sweep-g/{rows}x{cols}/{G}"), rows, cols, G=G, bits=4,
                                       sparsity=0.5)
                r = measure(bsr, 1)
                r["group_size"] = G
                nb = int(bsr["nnzg"]) * (G // 2 + 6) + 4 * (rows + 1) + 2 * cols + 4 * rows
                r["counted_bytes"], r["gbs"] = nb, round(nb / r["us"] / 1e3, 1)
                emit("H", r)
                cells.append(f"{r['us']:.2f} ({r['gbs']:.0f})")
            lines.append(f"| {rows}x{cols} | " + " | ".join(cells) + " |")
        lines.append("")

    if a.out:
        open(a.out + ".md", "w").write("\n".join(lines) + "\n")
        with open(a.out + ".jsonl", "w") as f:
            for r in recs:
                f.write(json.dumps(r) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
