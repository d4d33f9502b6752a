"""The fused all-gather epilogue (gqsa_gemm_allgather) across PROCESSES: P
ranks (spawned processes, all on cuda:0 -- this box has one GPU) exchange
their full-length output buffers as CUDA IPC handles (torch.multiprocessing),
and each rank's kernel stores its row shard into every rank's buffer through
the IPC-mapped peer pointers (the same mechanism NVLink P2P / symmetric
memory gives across GPUs).  After a cross-process barrier every rank's y must
equal the oracle's full result bit-exactly (exact-integer mode)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
mp = pytest.importorskip("torch.multiprocessing")

ROWS, COLS, B = 2048, 4096, 2


@pytest.mark.parametrize("P", [2, 3])
def test_fused_allgather_across_processes(P):
    from oracle import gqsa_oracle as O
    from paper_2412_17560_b200 import synth
    ctx = mp.get_context("spawn")
    q_in = [ctx.Queue() for _ in range(P)]
    barrier = ctx.Barrier(P)
    result = ctx.Queue()
    procs = [ctx.Process(target=_worker_direct, args=(r, P, q_in, barrier, result)) for r in range(P)]
    for p in procs:
        p.start()
    got = dict(result.get(timeout=300) for _ in range(P))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    bsr = synth.make_layer(synth.seed_for("ipc-allgather"), ROWS, COLS, sparsity=0.5, mode="exact_int")
    x = synth.make_x(synth.seed_for("ipc-allgather-x"), B, COLS, mode="exact_int")
    ref = O.gemv(bsr, x)
    for r in range(P):
        assert np.array_equal(got[r].astype(np.float64), ref), r


def _worker_direct(rank, P, q_in, barrier, result):
    import torch
    from paper_2412_17560_b200 import gqsa, synth
    torch.cuda.set_device(0)
    bsr = synth.make_layer(synth.seed_for("ipc-allgather"), ROWS, COLS, sparsity=0.5, mode="exact_int")
    x = synth.make_x(synth.seed_for("ipc-allgather-x"), B, COLS, mode="exact_int")
    X = torch.from_numpy(x).view(torch.float16).cuda()
    Y = torch.full((B, ROWS), float("nan"), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    for d in range(P):                  # CUDA IPC: my output buffer to every other rank
        if d != rank:
            q_in[d].put((rank, Y))
    peers = {rank: Y}
    for _ in range(P - 1):
        r, t = q_in[rank].get(timeout=120)
        peers[r] = t
    barrier.wait()
    lo, hi = synth.shard_rows(ROWS, P, rank)
    blob, desc = gqsa.pack(bsr, lo, hi)
    ws = torch.zeros(gqsa.workspace_size(desc, B), dtype=torch.uint8, device="cuda")
    gqsa.gemm_allgather(desc, torch.from_numpy(blob).cuda(), X, [peers[r] for r in range(P)], row_offset=lo, ws=ws)
    torch.cuda.synchronize()
    barrier.wait()                      # every rank's peer stores have landed
    result.put((rank, Y.cpu().numpy()))
    barrier.wait()                      # keep the buffers alive until every rank has read its own
