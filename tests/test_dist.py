"""Multi-process (gloo, world size 2, CPU) test of the output-row sharding
plumbing used by bench.py under torchrun: each rank packs its row shard with
the C++ packer, the shard round-trips through gqsa_unpack, the per-shard
results (oracle, CPU) are all-gathered, and the assembled y equals the
unsharded result row for row."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import gqsa_oracle as O
        from paper_2412_17560_b200 import gqsa, synth
        N, K = 96, 512
        bsr = synth.make_layer(77, N, K, sparsity=0.5, mask="skewed", mode="exact_int")
        x = synth.make_x(78, 1, K, mode="exact_int")
        lo, hi = synth.shard_rows(N, world, rank)
        blob, d = gqsa.pack(bsr, lo, hi)
        assert (d.rows, d.row_begin, d.row_end) == (hi - lo, lo, hi)
        shard = gqsa.unpack(blob)
        y_shard = torch.from_numpy(O.gemv(shard, x)[0])
        out = torch.empty(N, dtype=torch.float64)
        dist.all_gather_into_tensor(out, y_shard)  # equal-size shards (N % world == 0)
        full = O.gemv(bsr, x)[0]
        q.put((rank, bool(np.array_equal(out.numpy(), full))))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_rowshard_allgather_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res
