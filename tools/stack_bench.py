#!/usr/bin/env python
"""SURVEY §8(d) configs C3-C5 on one GPU (secondary measurements, not the bench line).

    python tools/stack_bench.py --out profiles/r01_stack

E. LLaMA-3-8B decoder LINEAR STACK per token (32 layers x q, k, v, o, gate,
   up, down = 224 GEMVs) at W4S30 / W4S50 / W2S50, B = 1, 2, 4, 8: one CUDA
   graph of the whole stack (PDL between launches), µs per token, counted GB/s.
   Also the merged form production servers use (vLLM-style fused qkv
   6144x4096 and gate_up 28672x4096: 128 GEMVs per token), and the separate
   matrices as gqsa_gemm_grouped launches of the GEMVs that share an input
   ({q, k, v}, {o}, {gate, up}, {down}: 128 launches per token).  Every launch
   reads the previous launch's output in a real decoder, so none declares
   x_ready (whole-SM launches, PDL between them).
F. Qwen2.5-14B (5120 / 13824, 48 layers) W4S50 and LLaMA-3.1-70B (8192 /
   28672) W4S50 row shards: the per-rank GEMV of a P-way row split
   (N/P x K) measured on this GPU, P = 1, 2, 4, 8 (Qwen) and P = 8 (70B).
   These are per-rank kernel times; the multi-GPU aggregate and all-gather
   need P GPUs (bench.py under torchrun) and are not measured here.

Weights: one synthetic set of layer matrices per setting, replicated into 32
(48) distinct device copies, so every GEMV streams its weights from HBM (the
stack is 2-4 GB, far beyond L2); values do not affect speed, masks are
uniform at the given sparsity.
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
from paper_2412_17560_b200 import gqsa, synth  # noqa: E402

LLAMA3_8B = [("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
             ("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336)]
LLAMA3_8B_MERGED = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]


# groups of GEMVs that share one input (one gqsa_gemm_grouped launch each)
GROUPS = {"q": 0, "k": 0, "v": 0, "o": 1, "gate": 2, "up": 2, "down": 3}


def time_stack(mats, n_layers, bits, sp, B, reps=20, grouped=False):
    """mats: [(name, rows, cols)] of one decoder layer; returns µs per token and bytes.
    grouped: the GEMVs sharing an input as one gqsa_gemm_grouped launch."""
    dev = torch.device("cuda")
    packed = []
    for name, rows, cols in mats:
        bsr = synth.make_layer(synth.seed_for(f"stack/{name}/{rows}x{cols}/{bits}/{sp}"), rows, cols,
                               bits=bits, sparsity=sp)
        blob, desc = gqsa.pack(bsr)
        packed.append((blob, desc))
    copies = [[torch.from_numpy(b).to(dev) for b, _ in packed] for _ in range(n_layers)]
    ws = [torch.zeros(gqsa.workspace_size(d, B), dtype=torch.uint8, device=dev) for _, d in packed]
    # q/k/v (qkv) read the same input, gate/up (gate_up) too
    src = {"q": "attn", "k": "attn", "v": "attn", "qkv": "attn", "o": "o", "gate": "mlp", "up": "mlp",
           "gate_up": "mlp", "down": "down"}
    xin = {}
    for name, _, c in mats:
        if src[name] not in xin:
            xin[src[name]] = torch.from_numpy(synth.make_x(synth.seed_for(f"stack-x/{src[name]}/{c}/{B}"), B, c)
                                              ).view(torch.float16).to(dev)
    xs = [xin[src[name]] for name, _, _ in mats]
    ys = [torch.empty(B, r, dtype=torch.float32, device=dev) for _, r, _ in mats]
    s = torch.cuda.Stream()
    if grouped:
        calls = []
        for L in range(n_layers):
            gs = {}
            for i, (name, _, _) in enumerate(mats):
                gs.setdefault(GROUPS[name], []).append((packed[i][1], copies[L][i], xs[i], ys[i], None))
            calls += [gqsa.Grouped(gs[k], ws[0]) for k in sorted(gs)]

    def token():
        if grouped:
            for c in calls:
                c(s)
            return
        for L in range(n_layers):
            for i, (_, d) in enumerate(packed):
                gqsa.gemm_smallbatch(d, copies[L][i], xs[i], ys[i], None, ws[i], stream=s)

    with torch.cuda.stream(s):
        token()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        token()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    nb = n_layers * sum(counted_bytes(d.rows, d.cols, d.nnzg, bits, B) for _, d in packed)
    launches = len(calls) if grouped else n_layers * len(packed)
    del copies
    torch.cuda.empty_cache()
    return us, nb, launches


def time_layer(rows, cols, bits, sp, B, reps=20):
    bsr = synth.make_layer(synth.seed_for(f"shard/{rows}x{cols}/{bits}/{sp}"), rows, cols, bits=bits, sparsity=sp)
    blob, desc = gqsa.pack(bsr)
    R = max(2, math.ceil(300e6 / blob.size))
    blobs = [torch.from_numpy(blob).cuda() for _ in range(R)]
    ws = torch.zeros(gqsa.workspace_size(desc, B), dtype=torch.uint8, device="cuda")
    X = torch.from_numpy(synth.make_x(7, B, cols)).view(torch.float16).cuda()
    Y = torch.empty(B, rows, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(R):
            gqsa.gemm_smallbatch(desc, blobs[i], X, Y, None, ws, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(R):
            gqsa.gemm_smallbatch(desc, blobs[i], X, Y, None, ws, stream=s)
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
    return us, counted_bytes(rows, cols, desc.nnzg, bits, B)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--batches", default="1,2,4,8")
    ap.add_argument("--settings", default="W4S30,W4S50,W2S50", help="subset of section E's settings")
    ap.add_argument("--forms", default="separate,merged,grouped", help="subset of section E's forms")
    ap.add_argument("--sections", default="EFG")
    a = ap.parse_args()
    peak, src = peaks()
    batches = [int(b) for b in a.batches.split(",")]
    recs = []
    lines = ["# Decoder-stack and shard measurements (tools/stack_bench.py; B200, 1 GPU)", "",
             f"GB/s = counted bytes / µs; frac = GB/s / {peak:.1f} ({src}). One CUDA graph per token, "
             "PDL between launches, weights in 32 (48) distinct device copies (HBM-resident, >> L2).", "",
             "## E. LLaMA-3-8B decoder linear stack per token (SURVEY §8(d) C3)", "",
             "| setting | form | launches | B | µs / token | GB per token | GB/s | frac |", "|---|---|---|---|---|---|---|---|"]
    forms = (("separate", "separate q/k/v, gate/up", LLAMA3_8B, False),
             ("merged", "merged qkv, gate_up", LLAMA3_8B_MERGED, False),
             ("grouped", "separate, grouped {qkv}{o}{gate,up}{down}", LLAMA3_8B, True))
    for bits, sp in ((4, 0.3), (4, 0.5), (2, 0.5)):
        if "E" not in a.sections or f"W{bits}S{int(sp * 100)}" not in a.settings.split(","):
            continue
        for key, form, mats, grouped in forms:
            if key not in a.forms.split(","):
                continue
            for B in batches:
                us, nb, nl = time_stack(mats, 32, bits, sp, B, grouped=grouped)
                r = dict(section="E", setting=f"W{bits}S{int(sp * 100)}", form=form, B=B, us=round(us, 1),
                         bytes=nb, launches=nl, gbs=round(nb / us / 1e3, 1), frac=round(nb / us / 1e3 / peak, 4))
                recs.append(r)
                print(json.dumps(r), flush=True)
                lines.append(f"| W{bits}S{int(sp * 100)} | {form} | {nl} | {B} | {us:.1f} | {nb / 1e9:.3f} | "
                             f"{r['gbs']:.0f} | {r['frac']:.3f} |")
    lines += ["", "## F. Row-shard GEMV per rank (SURVEY §8(d) C4, C5; §8(e)), W4S50, B = 1", "",
              "| model | matrix | full N x K | P | rank shard | µs | GB/s per rank |", "|---|---|---|---|---|---|---|"]
    qwen = [("q/o", 5120, 5120), ("k/v", 1024, 5120), ("gate/up", 13824, 5120), ("down", 5120, 13824)]
    l70 = [("q/o", 8192, 8192), ("k/v", 1024, 8192), ("gate/up", 28672, 8192), ("down", 8192, 28672)]
    for model, mats, Ps in (("Qwen2.5-14B", qwen, (1, 2, 4, 8)), ("LLaMA-3.1-70B", l70, (8,))) if "F" in a.sections else ():
        for name, n, k in mats:
            for P in Ps:
                us, nb = time_layer(n // P, k, 4, 0.5, 1)
                r = dict(section="F", model=model, matrix=name, N=n, K=k, P=P, us=round(us, 3), bytes=nb,
                         gbs=round(nb / us / 1e3, 1))
                recs.append(r)
                print(json.dumps(r), flush=True)
                lines.append(f"| {model} | {name} | {n}x{k} | {P} | {n // P}x{k} | {us:.2f} | {r['gbs']:.0f} |")
    lines += ["", "## G. Qwen2.5-14B full matrices, W4S50, B = 1 / 2 / 4 / 8 on one GPU (SURVEY §8(d) C4, P = 1)", "",
              "| matrix | N x K | B | µs | GB/s |", "|---|---|---|---|---|"]
    for name, n, k in qwen if "G" in a.sections else ():
        for B in batches:
            us, nb = time_layer(n, k, 4, 0.5, B)
            r = dict(section="G", model="Qwen2.5-14B", matrix=name, N=n, K=k, B=B, us=round(us, 3), bytes=nb,
                     gbs=round(nb / us / 1e3, 1))
            recs.append(r)
            print(json.dumps(r), flush=True)
            lines.append(f"| {name} | {n}x{k} | {B} | {us:.2f} | {r['gbs']:.0f} |")
    lines.append("")
    if a.out:
        open(a.out + ".md", "w").write("\n".join(lines) + "\n")
        with open(a.out + ".jsonl", "w") as f:
            for r in recs:
                f.write(json.dumps(r) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
