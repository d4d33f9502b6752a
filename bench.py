#!/usr/bin/env python
"""GQSA decode hot path benchmark (BASELINE.json metric).

One STEP = one sparse GEMV on each LLaMA-3-8B layer shape of BASELINE.json
configs[1] -- 4096x4096, 14336x4096, 4096x14336 at W4S50, G=16, batch 1 --
i.e. every row of SURVEY §8(a) over one batch of synthetic input.  value =
counted (compressed, algorithmic) bytes of all steps / device time, in GB/s.

The step runs as ONE gqsa_gemm_grouped launch (the three GEMVs are
independent; `--path launches` runs one gqsa_gemv per layer instead).  The
step's activations are inputs that nothing in the timed region writes, so the
launch declares them ready (x_ready, `--x-ready 0` turns it off): the library
then runs it PIPELINED -- half of every SM, all global writes deferred until
the previous step's launch has completed -- so consecutive steps overlap
their start-up and drain.  `layers[]` are standalone
launches of each layer: `us` with x_ready = 0 (the dependent-chain case),
`us_x_ready` as consecutive independent (pipelined) launches.

Timing: the weights rotate over R device copies of the layer set (> 2x the
126 MB L2), so every launch streams from HBM.  K steps are replayed from CUDA
graphs (every graph of the timed region replayed during warm-up), bracketed
by barrier + synchronize, timed with CUDA events on the launching stream (max
over ranks).  Clocks / throttle reasons are sampled through NVML during the
timed region.

N > 1 (torchrun, NCCL): every rank owns rows [N*r/P, N*(r+1)/P) of each layer
(output-row sharding), runs its GEMV, then all-gathers y over
NVLink (torch.distributed.all_gather_into_tensor), all captured in CUDA
graphs.  Total work is fixed: "scaling": "strong".  The line adds the split
of SURVEY §8(e): per-rank kernel µs, all-gather µs, end-to-end µs and the
kernel-only aggregate GB/s.

--impl reference: the CPU fp64 oracle (oracle/), the tier's reference arm,
timed on the host on a bounded row sample of the same workload (rank 0 only).
"""
import os

# the CPU legs (oracle) run single-threaded: set before numpy is imported
for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse
import json
import math
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GQSA W4S50 sparse GEMV µs & achieved HBM GB/s vs ~8 TB/s at LLaMA shapes"
SHAPES = [(4096, 4096, "q_proj/o_proj"), (14336, 4096, "gate_proj/up_proj"), (4096, 14336, "down_proj")]
NOMINAL_HBM_GBS = 8000.0
FALLBACK_HBM_GBS = 6650.0
L2_BYTES = 126 * 1024 * 1024


def counted_bytes(rows, cols, nnzg, bits, batch=1, G=16):
    """n*G/8 + 2 + 2 + 2 bytes per kept group, 4*(rows+1) row
    offsets, 2*B*K of fp16 x, 4*B*N of fp32 y."""
    return nnzg * (G * bits // 8 + 6) + 4 * (rows + 1) + 2 * batch * cols + 4 * batch * rows


def workload_config(batch, world, bits=4, sparsity=0.5):
    """The workload both arms run (identical dicts: the driver compares them)."""
    return {"workload": f"llama3-8b-layer-shapes-w{bits}s{int(round(sparsity * 100))}-b{batch} "
                        "(4096x4096, 14336x4096, 4096x14336)",
            "global_batch": batch, "seq_len": 1, "group_size": 16, "bits": bits, "sparsity": sparsity,
            "parallelism": f"rowshard{world}" if world > 1 else "single",
            "l2": "inputs larger than L2 (weights rotate over device copies > 2x L2)"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy r+w)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def read_peak(achieved):
    """The third denominator: the best read-only stream this build's
    calibration kernel (tools/stream_bench.cu) measured on a B200, from
    profiles/r02_stream_bench.jsonl: the same 59 MB per launch, and 300 MB."""
    p = os.path.join(ROOT, "profiles", "r02_stream_bench.jsonl")
    if not os.path.exists(p):
        return {}
    best = {}
    for line in open(p):
        d = json.loads(line)
        k = "read_peak_59mb_gbs" if d["bytes"] < 100e6 and d["bytes"] > 50e6 else \
            "read_peak_300mb_gbs" if d["bytes"] > 200e6 else None
        if k:
            best[k] = max(best.get(k, 0.0), float(d["gbs"]))
    if "read_peak_59mb_gbs" in best:
        best["frac_of_read_peak_59mb"] = round(achieved / best["read_peak_59mb_gbs"], 4)
    best["read_peak_source"] = "profiles/r02_stream_bench.jsonl (tools/stream_bench.cu, B200)"
    return best


def make_layers(bits, sparsity, batch, world=1, rank=0, mask="uniform"):
    from paper_2412_17560_b200 import synth
    out = []
    for rows, cols, name in SHAPES:
        tag = f"llama3-8b/{rows}x{cols}/{bits}/{sparsity}/16/{mask}"
        seed = synth.seed_for(tag)
        bsr = synth.make_layer(seed, rows, cols, bits=bits, sparsity=sparsity, mask=mask)
        x = synth.make_x(seed + 1, batch, cols)
        lo, hi = synth.shard_rows(rows, world, rank)
        out.append(dict(name=name, rows=rows, cols=cols, bsr=bsr, x=x, lo=lo, hi=hi, tag=tag))
    return out


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, dev_index):
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML unavailable
            self.nv = None

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake_slowdown",
        }
        for bit, name in names.items():
            if r & bit:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- cpu baseline
def host_info():
    """nproc, the CPU model (lscpu "Model name" / /proc/cpuinfo) of the box."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


class pinned_core:
    """Pin this process to one host core while the oracle is timed (restores the mask)."""

    def __init__(self):
        self.core, self.prev = None, None

    def __enter__(self):
        try:
            self.prev = os.sched_getaffinity(0)
            self.core = min(self.prev)
            os.sched_setaffinity(0, {self.core})
        except (AttributeError, OSError):
            self.core = None
        return self

    def __exit__(self, *a):
        if self.prev is not None:
            os.sched_setaffinity(0, self.prev)


def cpu_oracle_baseline(layers, budget_s=12.0, max_reps=50, gpu_y=None):
    """The fp64 oracle as it stands, single process (numpy, 1 core: affinity
    pinned, BLAS/OpenMP threads 1), on whole layers of the workload, repeated
    until ~budget_s of CPU work.  Its first result per layer also checks the
    GPU output of the same layer (``gpu_y``: name -> [B][rows]) against the
    north-star gate G1 (max|dy| <= 1e-3 ||y||_2) and G3 (||dy||_2 <= 1e-4 ||y||_2)."""
    from oracle import gqsa_oracle as O
    done_bytes, t_total, reps = 0, 0.0, 0
    parity = {}
    pin = pinned_core()
    pin.__enter__()
    names = []
    while t_total < budget_s and reps < max_reps:
        for L in layers:
            bsr = L["bsr"]
            t0 = time.perf_counter()
            y_ref = O.gemv(bsr, L["x"])
            t_total += time.perf_counter() - t0
            if gpu_y is not None and L["name"] not in parity:
                d = np.abs(np.asarray(gpu_y[L["name"]], np.float64) - y_ref)
                nrm = float(np.linalg.norm(y_ref))
                g1, g3 = float(d.max()) / nrm, float(np.linalg.norm(d)) / nrm
                parity[L["name"]] = {"g1_maxabs_over_l2": g1, "g3_l2_rel": g3,
                                     "ok": bool(np.all(np.isfinite(d)) and g1 <= 1e-3 and g3 <= 1e-4)}
            done_bytes += counted_bytes(L["rows"], L["cols"], bsr["nnzg"], bsr["bits"], L["x"].shape[0])
            names.append(L["name"])
            if t_total >= budget_s:
                break
        reps += 1
    pin.__exit__()
    return {
        "value": done_bytes / t_total / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
        "pinned_core": pin.core, **host_info(),
        "sample": f"{len(names)} whole-layer oracle GEMVs ({', '.join(sorted(set(names)))}) of the "
                  f"same synthetic workload, {t_total:.1f} s of single-core numpy fp64",
        "seconds": round(t_total, 2),
        "gpu_parity": parity or None,
    }


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import gqsa_oracle as O
    layers = make_layers(args.bits, args.sparsity, args.batch)
    total_steps = args.steps + args.warmup
    budget = float(os.environ.get("GQSA_REF_BUDGET_S", "90"))
    per_step = budget / max(total_steps, 1)
    # a bounded row sample per layer, sized from a quick calibration
    t0 = time.perf_counter()
    O.gemv_rows(layers[0]["bsr"], layers[0]["x"], np.arange(64))
    per_row = (time.perf_counter() - t0) / 64
    rows_per_layer = int(max(1, min(4096, per_step / (per_row * 3 * 3.5))))
    rng = np.random.default_rng(0)
    samples = []
    for L in layers:
        ri = L["bsr"]["row_index"]
        rs = np.sort(rng.choice(L["rows"], size=min(rows_per_layer, L["rows"]), replace=False))
        nnz = int(np.sum(ri[rs + 1] - ri[rs]))
        b = nnz * (16 * args.bits // 8 + 6) + 4 * (len(rs) + 1) + 2 * args.batch * L["cols"] + 4 * args.batch * len(rs)
        samples.append((L, rs, b))
    for _ in range(args.warmup):
        for L, rs, _b in samples:
            O.gemv_rows(L["bsr"], L["x"], rs)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for L, rs, _b in samples:
            O.gemv_rows(L["bsr"], L["x"], rs)
    dt = time.perf_counter() - t0
    step_bytes = sum(b for _, _, b in samples)
    value = step_bytes * args.steps / dt / 1e9
    sample = (f"{rows_per_layer} random output rows of each of 4096x4096, 14336x4096, 4096x14336 "
              f"(W4S50, B={args.batch}) per step; bytes counted per sampled row")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; DESIGN.md §4 recipe)",
        "config": workload_config(args.batch, args.gpus, args.bits, args.sparsity),
        "method": {"host": "CPU fp64 oracle (oracle/gqsa_oracle.py), 1 core, rank 0"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
class StepTimer:
    """Times K steps replayed from CUDA graphs on `stream` with CUDA events.

    The graphs are exactly the ones the timed region replays -- one of `period`
    steps (a multiple of the weight-rotation period R) and one of the
    remainder -- and both are replayed during warm-up, so the timed region pays
    no first-replay upload.  A short device sleep precedes the start event so
    that the host has queued the replays before the GPU reaches them (no
    launch gaps inside the timed region)."""

    def __init__(self, torch, stream, step, R, steps, warmup, use_graph=True):
        self.torch, self.stream, self.step, self.steps = torch, stream, step, steps
        self.use_graph = use_graph
        self.period = R * max(1, -(-120 // R)) if steps > 120 else steps
        self.rem = steps % self.period
        if use_graph:
            self.g_full = self._capture(self.period, 0)
            self.g_rem = self._capture(self.rem, 0) if self.rem else None
        self.warm = max(warmup, 3)
        with torch.cuda.stream(stream):
            if use_graph:
                for _ in range(max(1, -(-self.warm // self.period))):
                    self.g_full.replay()
                if self.g_rem is not None:
                    self.g_rem.replay()
            else:
                for k in range(self.warm):
                    step(k)
        torch.cuda.synchronize()

    def _capture(self, n, start):
        g = self.torch.cuda.CUDAGraph()
        with self.torch.cuda.graph(g, stream=self.stream):
            for k in range(n):
                self.step(start + k)
        return g

    def run(self):
        """Returns milliseconds for `steps` steps (device time, CUDA events)."""
        torch = self.torch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(self.stream):
            torch.cuda._sleep(200_000)  # ~0.1 ms: the host queues the replays meanwhile
            e0.record(self.stream)
            if self.use_graph:
                for _ in range(self.steps // self.period):
                    self.g_full.replay()
                if self.g_rem is not None:
                    self.g_rem.replay()
            else:
                for k in range(self.steps):
                    self.step(k)
            e1.record(self.stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2412_17560_b200 import gqsa

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("GQSA_SHARE_DEVICE") == "1":  # test hook: several ranks on one GPU (gloo)
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    fused = args.allgather in ("fused", "nvls")
    nvls = args.allgather == "nvls"
    if os.environ.get("NCCL_DEBUG") and not os.environ.get("NCCL_DEBUG_FILE"):
        os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"  # NCCL's log to stderr: stdout carries the JSON line
    if world > 1 or fused:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        backend = os.environ.get("GQSA_DIST_BACKEND", "nccl")  # gloo: test hook for the plumbing
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
        else:
            dist.init_process_group(backend, rank=rank, world_size=world)
    nccl = dist.is_initialized() and dist.get_backend() == "nccl"

    bits, sp, B = args.bits, args.sparsity, args.batch
    layers = make_layers(bits, sp, B, world, rank)
    hbm_peak, peak_src = peaks()

    # pack this rank's row shard of every layer; R device copies for L2 rotation
    packed = []
    set_bytes = 0
    for L in layers:
        blob, desc = gqsa.pack(L["bsr"], L["lo"], L["hi"])
        packed.append((blob, desc))
        set_bytes += blob.size
    R = max(2, math.ceil(2.2 * L2_BYTES / max(set_bytes, 1)) + 1) if not args.no_rotate else 1
    copies = [[torch.from_numpy(blob).to(dev) for blob, _ in packed] for _ in range(R)]
    descs = [d for _, d in packed]
    ws = torch.zeros(gqsa.workspace_size(descs[0], B), dtype=torch.uint8, device=dev)
    xs = [torch.from_numpy(L["x"]).view(torch.float16).to(dev) for L in layers]
    ys = [torch.empty(B, d.rows, dtype=torch.float32, device=dev) for d in descs]
    yfull = [torch.empty(world * B * d.rows, dtype=torch.float32, device=dev) if world > 1 else None
             for d in descs]

    # fused all-gather: each rank's GEMV stores its rows
    # straight into every rank's full y (symmetric memory, NVLink P2P), then a
    # symmetric-memory barrier orders the step; no NCCL data movement
    if fused:
        import torch.distributed._symmetric_memory as symm_mem
        gname = dist.group.WORLD.group_name
        if hasattr(symm_mem, "enable_symm_mem_for_group"):
            symm_mem.enable_symm_mem_for_group(gname)
        yf = [symm_mem.empty((B, L["rows"]), dtype=torch.float32, device=dev) for L in layers]
        hdl = [symm_mem.rendezvous(t, gname) for t in yf]
        peers = [[h.get_buffer(p, (B, L["rows"]), torch.float32) for p in range(world)]
                 for h, L in zip(hdl, layers)]
        if nvls and not all(getattr(h, "multicast_ptr", 0) for h in hdl):
            raise SystemExit("--allgather nvls: symmetric memory has no multicast object on this system "
                             "(NVLS needs a multicast-capable NVSwitch domain of >= 2 GPUs)")

    path = "launches" if fused else args.path
    grouped = [gqsa.Grouped([(descs[i], copies[r][i], xs[i], ys[i], None) for i in range(len(layers))], ws,
                            x_ready=args.x_ready) for r in range(R)]

    def gemvs(r):
        """The step's sparse GEMVs (this rank's shards)."""
        if fused:
            for i in range(len(layers)):
                if nvls:  # one multimem.st per element; the NVSwitch replicates it to every rank
                    gqsa.gemm_allgather_multicast(descs[i], copies[r][i], xs[i], hdl[i].multicast_ptr,
                                                  ldy=layers[i]["rows"], row_offset=layers[i]["lo"], ws=ws)
                else:
                    gqsa.gemm_allgather(descs[i], copies[r][i], xs[i], peers[i], row_offset=layers[i]["lo"], ws=ws)
                hdl[i].barrier(channel=0)
        elif path == "grouped":
            grouped[r]()
        else:
            for i in range(len(layers)):
                gqsa.gemm_ex(descs[i], copies[r][i], xs[i], ys[i], ws=ws, x_ready=bool(args.x_ready))

    def gathers():
        """The step's exchange: all-gather of every layer's y shard over NCCL (N > 1)."""
        if world > 1 and not fused:
            for i in range(len(layers)):
                dist.all_gather_into_tensor(yfull[i], ys[i].view(-1))

    def step(k):
        gemvs(k % R)
        gathers()

    stream = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):  # eager first launches (attributes, module load, NCCL comms)
        for r in range(R):
            step(r)
    torch.cuda.synchronize()
    # NCCL collectives are graph-capturable; symmetric-memory barriers and the
    # gloo test hook stay eager
    use_graph = not fused and (world == 1 or nccl)
    timer = StepTimer(torch, stream, step, R, args.steps, args.warmup, use_graph)
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    with sampler:
        ms = timer.run()
    if world > 1:
        dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(ms)
    ms_step = ms / args.steps
    warm = timer.warm

    # counted bytes: every rank's shard (sum over ranks)
    step_bytes_rank = sum(counted_bytes(d.rows, d.cols, d.nnzg, bits, B) for d in descs)
    if world > 1:
        t = torch.tensor([step_bytes_rank], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        step_bytes = float(t.item())
    else:
        step_bytes = float(step_bytes_rank)
    value = step_bytes * args.steps / (ms * 1e-3) / 1e9

    # ---- multi-GPU split: kernels alone and the exchange alone,
    #      each timed like the step (graphs, max over ranks)
    split = None
    if world > 1 and not fused:
        ksteps = min(args.steps, 2000)
        kt = StepTimer(torch, stream, lambda k: gemvs(k % R), R, ksteps, args.warmup, use_graph)
        dist.barrier()
        k_ms = max_over_ranks(kt.run()) / ksteps
        gt = StepTimer(torch, stream, lambda k: gathers(), 1, ksteps, args.warmup, use_graph)
        dist.barrier()
        g_ms = max_over_ranks(gt.run()) / ksteps
        split = {"per_rank_kernel_us": round(k_ms * 1e3, 3), "allgather_us": round(g_ms * 1e3, 3),
                 "end_to_end_us": round(ms_step * 1e3, 3),
                 "kernel_only_aggregate_gbs": round(step_bytes / (k_ms * 1e-3) / 1e9, 1),
                 "allgather_bytes_per_rank": int(sum(B * d.rows * 4 for d in descs)),
                 "nccl": nccl}

    # ---- per-layer device time (one launch per layer), outside the timed region
    layer_rows = []
    if world == 1 and not args.no_layers:
        for i, L in enumerate(layers):
            d = descs[i]
            # this layer alone rotates over > 2.2x L2 of its own copies
            Rl = max(R, math.ceil(2.2 * L2_BYTES / int(d.blob_bytes)) + 1) if not args.no_rotate else 1
            lcop = [copies[r % R][i] if r < R else copies[0][i].clone() for r in range(Rl)]

            def one(k, i=i):  # dependent form: each launch may read the previous one's output
                if B == 1:
                    gqsa.gemv(d, lcop[k % Rl], xs[i][0], ys[i][0], None, ws)
                else:
                    gqsa.gemm_smallbatch(d, lcop[k % Rl], xs[i], ys[i], None, ws)

            def one_ready(k, i=i):  # independent form: x declared ready (pipelined launches at B <= 2)
                gqsa.gemm_ex(d, lcop[k % Rl], xs[i], ys[i], ws=ws, x_ready=True)
            reps = max(Rl, (2000 // Rl) * Rl)
            us = StepTimer(torch, stream, one, Rl, reps, 3 * Rl, True).run() * 1e3 / reps
            us_r = StepTimer(torch, stream, one_ready, Rl, reps, 3 * Rl, True).run() * 1e3 / reps
            del lcop
            cb = counted_bytes(d.rows, d.cols, d.nnzg, bits, B)
            layer_rows.append({"shape": f"{d.rows}x{d.cols}", "role": L["name"], "nnzg": d.nnzg,
                               "counted_bytes": cb, "blob_bytes": int(d.blob_bytes), "us": round(us, 3),
                               "gbs": round(cb / us / 1e3, 1),
                               "frac_of_8tbs": round(cb / us / 1e3 / NOMINAL_HBM_GBS, 4),
                               "frac_of_measured": round(cb / us / 1e3 / hbm_peak, 4),
                               "us_x_ready": round(us_r, 3), "gbs_x_ready": round(cb / us_r / 1e3, 1),
                               "frac_of_measured_x_ready": round(cb / us_r / 1e3 / hbm_peak, 4),
                               "rotation_copies": Rl})

    # ---- end to end through the public C ABI with host buffers (pinned):
    #      gqsa_gemm_multi_hostio = one H2D copy of the step's inputs, the
    #      step's GEMVs as one grouped launch, one D2H copy of its outputs; the
    #      caller synchronises and reads y every step
    e2e = None
    if world == 1:
        hX = torch.from_numpy(np.concatenate([L["x"].reshape(-1) for L in layers])).view(torch.float16).pin_memory()
        hY = torch.empty(sum(B * d.rows for d in descs), dtype=torch.float32).pin_memory()
        stage = torch.empty(gqsa.multi_hostio_stage_size(descs, B), dtype=torch.uint8, device=dev)
        ne = min(args.steps, args.e2e_steps)
        calls = [gqsa.MultiHostIO(descs, copies[r], hX, hY, stage, [ws], batch=B) for r in range(R)]

        def e2e_step(k):
            calls[k % R](stream)
            stream.synchronize()  # the caller reads y every step

        for k in range(3):
            e2e_step(k)
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(stream)
        for k in range(ne):
            e2e_step(k)
        b_.record(stream)
        stream.synchronize()
        wall = time.perf_counter() - t0
        e_ms = a.elapsed_time(b_)
        e2e = {"value": step_bytes * ne / (e_ms * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(hX.numel() * 2), "d2h_bytes_per_step": int(hY.numel() * 4),
               "steps": ne, "ms_per_step": e_ms / ne, "wall_ms_per_step": wall * 1e3 / ne,
               "api": "gqsa_gemm_multi_hostio (1 H2D + one grouped launch + 1 D2H, stream sync per step)"}

    # ---- outputs of the timed step, for the parity check in the cpu_baseline leg
    with torch.cuda.stream(stream):
        step(0)
    torch.cuda.synchronize()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        gpu_y = None if fused else {L["name"]: ys[i].cpu().numpy() for i, L in enumerate(layers)}
        cpu = cpu_oracle_baseline(layers, budget_s=args.cpu_budget, gpu_y=gpu_y)

    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    n_launch = (1 if path == "grouped" else len(layers)) * args.steps
    achieved = value if world == 1 else step_bytes / world / (ms_step * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": warm, "ms_per_step": ms_step,
        "us_per_step": round(ms_step * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u4xf16->f32",
        "data": "synthetic (seeded random W4 codes, fp16 s/z, uniform 50% group mask, N(0,1) fp16 x "
                "with 0.5% outlier channels; DESIGN.md §4)",
        "config": workload_config(B, world, bits, sp),
        "method": {"allgather": (args.allgather if (world > 1 or fused) else None),
                   "l2": f"inputs larger than L2: weights rotate over {R} device copies of the layer set "
                         f"({R * set_bytes / 2**20:.0f} MiB > 2x L2)",
                   "path": {"grouped": "one gqsa_gemm_grouped launch per step (the 3 independent GEMVs "
                                       "share one Stream-K partition)",
                            "launches": "one gqsa_gemm_ex launch per layer (PDL)"}[path],
                   "x_ready": bool(args.x_ready),
                   "timing": "CUDA graphs of the step (all graphs replayed in warm-up), CUDA events on the "
                             "launch stream, device sleep before the start event"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                     "peak_source": peak_src, "frac_of_nominal_8tbs": round(achieved / NOMINAL_HBM_GBS, 4),
                     **read_peak(achieved),
                     "kernel": f"gqsa::gqsa_stream_kernel<{bits},{B},16,{int(bool(args.x_ready) and B <= 2)}>",
                     "algorithmic_bytes_per_step": int(step_bytes),
                     "note": "achieved = algorithmic bytes of the step / device time of the step; the step is "
                             + ("ONE launch of the dominant kernel" if path == "grouped" else "3 launches")},
        "layers": layer_rows,
        "multi_gpu": split,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": n_launch,
        "clocks": sampler.summary(),
    }
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", default="gqsa", choices=["gqsa", "reference"])
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--bits", type=int, default=4, choices=[2, 4, 8],
                    help="secondary settings (W2S50, W4S30, ...); the metric's workload is W4S50")
    ap.add_argument("--sparsity", type=float, default=0.5)
    ap.add_argument("--e2e-steps", type=int, default=2000)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rotate", action="store_true")
    ap.add_argument("--no-layers", action="store_true", help="skip the per-layer timing loop (ncu launch lists)")
    ap.add_argument("--allgather", default="nccl", choices=["nccl", "fused", "nvls"],
                    help="row-shard output exchange: NCCL all_gather, the fused GEMV epilogue storing (nvls: "
                         "multicasting through NVLink SHARP) "
                         "into every rank's y over symmetric memory (gqsa_gemm_allgather)")
    ap.add_argument("--path", default="grouped", choices=["grouped", "launches"],
                    help="grouped: the step's GEMVs in one gqsa_gemm_grouped launch; launches: one gqsa_gemv "
                         "per layer")
    ap.add_argument("--x-ready", type=int, default=1, choices=[0, 1],
                    help="declare the step's x not produced by the previous kernel (true here: nothing in the "
                         "timed region writes x), so consecutive steps pipeline (DESIGN.md §6.2); 0 = every "
                         "launch waits for the previous one to complete before it reads x")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
