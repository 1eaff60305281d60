"""CPU, world_size 2 over gloo: the host-side logic of the N>1 path —
heap-handle exchange in rank order, max-over-ranks timing, and the property the
device flag protocol relies on: every rank derives the identical segment plan
(same buckets, chunks, shard layout) from the same tensor list."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_05720_b200.collectives import TensorList
        from paper_2105_05720_b200.runtime import exchange_blobs, max_over_ranks
        from paper_2105_05720_b200.workloads import bert_large_counts

        mine = bytes([rank]) * 64  # a cudaIpcMemHandle_t is 64 bytes
        blob = exchange_blobs(mine, world)
        t = max_over_ranks(1.5 + rank)
        plans = {}
        for counts in ([10, 1500, 3, 700], bert_large_counts()):
            tl = TensorList(None, counts, world=world)
            h = hashlib.sha1()
            for r in list(range(world)) + [-1]:
                h.update(tl.segments(r).tobytes())
            h.update(np.array([tl.shard_elems, tl.state_elems, tl.total], np.int64).tobytes())
            plans[len(counts)] = h.hexdigest()
        allp = [None] * world
        dist.all_gather_object(allp, plans)
        q.put((rank, blob, t, allp))
    finally:
        dist.destroy_process_group()


def test_two_rank_bootstrap_and_plan_agreement():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, blob, t, allp in res:
        assert blob == bytes([0]) * 64 + bytes([1]) * 64  # rank order
        assert t == 2.5                                     # the slowest rank
        assert allp[0] == allp[1]                           # identical plans on every rank
