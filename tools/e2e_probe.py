"""Where the end-to-end (host I/O) step time goes: copies only, launches only, full."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2412_17560_b200 import gqsa, synth

shapes = [(4096, 4096), (14336, 4096), (4096, 14336)]
layers = [gqsa.Layer(synth.make_layer(i, n, k, sparsity=0.5)) for i, (n, k) in enumerate(shapes)]
descs = [L.desc for L in layers]
hX = torch.zeros(sum(k for _, k in shapes), dtype=torch.float16).pin_memory()
hY = torch.zeros(sum(n for n, _ in shapes), dtype=torch.float32).pin_memory()
stage = torch.empty(gqsa.multi_hostio_stage_size(descs, 1), dtype=torch.uint8, device="cuda")
dX = torch.zeros_like(hX, device="cuda"); dY = torch.zeros_like(hY, device="cuda")
s = torch.cuda.current_stream()

def bench(name, fn, n=2000):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n): fn()
    print(f"{name:40s} {(time.perf_counter() - t) / n * 1e6:8.1f} us/step", flush=True)

bench("sync only", lambda: s.synchronize())
bench("H2D+D2H+sync", lambda: (dX.copy_(hX, non_blocking=True), hY.copy_(dY, non_blocking=True), s.synchronize()))
def launches():
    off = 0
    for L, (n, k) in zip(layers, shapes):
        gqsa.gemv(L.desc, L.blob, dX[off:off + k], dY[:n], None, L.ws)
        off += k
bench("3 launches (no sync)", launches, 200)
bench("3 launches + sync", lambda: (launches(), s.synchronize()))
bench("multi_hostio + sync", lambda: (gqsa.gemm_multi_hostio(descs, [L.blob for L in layers], hX, hY, stage, [L.ws for L in layers]), s.synchronize()))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    gqsa.gemm_multi_hostio(descs, [L.blob for L in layers], hX, hY, stage, [L.ws for L in layers])
bench("graph(multi_hostio) + sync", lambda: (g.replay(), s.synchronize()))
t0 = time.perf_counter(); n0 = gqsa.launch_count()
for _ in range(1000): gqsa.gemv(layers[0].desc, layers[0].blob, dX[:4096], dY[:4096], None, layers[0].ws)
print("gemv host call us", (time.perf_counter() - t0) * 1e3)
torch.cuda.synchronize()
L0 = layers[0]
def tm(name, fn, n=2000):
    t = time.perf_counter()
    for _ in range(n): fn()
    print(f"{name:40s} {(time.perf_counter() - t) / n * 1e6:8.2f} us", flush=True)
tm("ctypes gqsa_version", lambda: gqsa.lib().gqsa_version())
tm("launch_plan (ctypes+make_plan)", lambda: gqsa.launch_plan(L0.desc, 1))
tm("current_stream ptr", lambda: gqsa._stream_ptr(None))
tm("data_ptr x5", lambda: (L0.blob.data_ptr(), dX.data_ptr(), dY.data_ptr(), L0.ws.data_ptr(), L0.ws.numel()))
tm("gemv call", lambda: gqsa.gemv(L0.desc, L0.blob, dX[:4096], dY[:4096], None, L0.ws))
torch.cuda.synchronize()
tm("slice dX[:4096]", lambda: dX[:4096])
