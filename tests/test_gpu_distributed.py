"""GPU, DISTRIBUTED mode with real processes: W processes share one B200, each
maps the others' heaps through CUDA IPC (coconet_heap_handle /
coconet_open_peers) — the same code path as one process per GPU over NVLink,
and the cross-process flag protocol (st.release.sys / ld.acquire.sys) runs
between contexts that the driver time-slices. Results must equal the
restated reference bit for bit (EXACT)."""
import os
import socket
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(W, counts):
    rng = np.random.default_rng(11)
    g = [rng.uniform(-1, 1, (W, n)).astype(np.float32) for n in counts]
    p = [rng.uniform(0.1, 0.9, n).astype(np.float32) for n in counts]
    m = [rng.uniform(-0.1, 0.1, n).astype(np.float32) for n in counts]
    v = [rng.uniform(0.01, 0.2, n).astype(np.float32) for n in counts]
    return g, p, m, v


def _worker(rank, world, port, counts, q, heap="cudamalloc"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import coconet_oracle as co
        from paper_2105_05720_b200 import _lib
        from paper_2105_05720_b200.collectives import AdamHParams, TensorList, allreduce, fused_rs_adam_ag
        from paper_2105_05720_b200.runtime import Context

        torch.cuda.set_device(0)
        ctx = Context(world, mode="distributed", rank=rank, device=0, heap_bytes=64 << 20, timeout_ms=60000,
                      heap=heap)
        assert ctx.heap_kind == heap
        tl = TensorList(ctx, counts)
        g, p, m, v = _inputs(world, counts)
        gb = [ctx.alloc([n]) for n in counts]
        pb = [ctx.alloc([n]) for n in counts]
        mb, vb = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
        tens, elem, sidx = tl.state_index_map(rank)
        ms = np.zeros(tl.shard_elems, np.float32)
        vs = np.zeros(tl.shard_elems, np.float32)
        for t in range(len(counts)):
            ctx.view(gb[t]).copy_(torch.from_numpy(g[t][rank]))
            ctx.view(pb[t]).copy_(torch.from_numpy(p[t]))
            sel = tens == t
            ms[sidx[sel]] = m[t][elem[sel]]
            vs[sidx[sel]] = v[t][elem[sel]]
        ctx.view(mb).copy_(torch.from_numpy(ms))
        ctx.view(vb).copy_(torch.from_numpy(vs))
        torch.cuda.synchronize()
        dist.barrier()
        hp = AdamHParams(0.01, 0.9, 0.999, 3.0, 0.0, True, _lib.MATH_EXACT, _lib.ALGO_TWO_SHOT)
        for _ in range(2):  # twice: epochs advance consistently across processes
            fused_rs_adam_ag(ctx, tl, gb, pb, mb, vb, hp)
            ctx.check()
        # the same two steps through the TMA ring (g pulled from the other
        # processes by the consumers, p pushed into them)
        pb_t = [ctx.alloc([n]) for n in counts]
        mb_t, vb_t = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
        for t in range(len(counts)):
            ctx.view(pb_t[t]).copy_(torch.from_numpy(p[t]))
        ctx.view(mb_t).copy_(torch.from_numpy(ms))
        ctx.view(vb_t).copy_(torch.from_numpy(vs))
        torch.cuda.synchronize()
        dist.barrier()
        os.environ["COCONET_ADAM_TMA"] = "1"
        try:
            for _ in range(2):
                fused_rs_adam_ag(ctx, tl, gb, pb_t, mb_t, vb_t, hp)
                ctx.check()
        finally:
            os.environ.pop("COCONET_ADAM_TMA")
        got_p_tma = [ctx.view(b).cpu().numpy() for b in pb_t]
        # AllReduce of the (original) gradients, out of place
        ob = [ctx.alloc([n]) for n in counts]
        for t in range(len(counts)):
            ctx.view(gb[t]).copy_(torch.from_numpy(g[t][rank]))
        torch.cuda.synchronize()
        dist.barrier()
        allreduce(ctx, tl, gb, ob)
        ctx.check()
        got_p = [ctx.view(b).cpu().numpy() for b in pb]
        got_ar = [ctx.view(b).cpu().numpy() for b in ob]
        # expected: two reference fused Adam steps on the same per-rank grads
        k = co.adam_consts(0.01, 0.9, 0.999, 3.0)
        m1, v1, p1 = co.fused_adam(g, m, v, p, k)
        _, _, p2 = co.fused_adam(g, m1, v1, p1, k)
        table = co.bucket_table(counts)
        flat = co.flatten_bucket_order(g, table)
        bounds = co.flat_chunks(flat.shape[1], world)
        owner = np.searchsorted(np.asarray(bounds[1:]), np.arange(flat.shape[1]), side="right")
        ar = co.unflatten_bucket_order(co.ring_reduce(flat, owner), counts, table)
        ok_p = all(np.array_equal(got_p[t], p2[t]) and np.array_equal(got_p_tma[t], p2[t]) for t in range(len(counts)))
        ok_ar = all(np.array_equal(got_ar[t], ar[t]) for t in range(len(counts)))
        dist.barrier()
        ctx.close()
        q.put((rank, ok_p, ok_ar, None))
    except Exception as e:  # report, don't hang the parent
        q.put((rank, False, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,heap", [(2, "cudamalloc"), (4, "cudamalloc"), (2, "cumem"), (4, "cumem")])
def test_distributed_processes_share_one_gpu(world, heap):
    """heap="cumem": the heaps are cuMemCreate allocations whose POSIX
    descriptors the processes pass over Unix sockets (heap_cumem.cu) instead
    of CUDA IPC handles; results must be the same bits."""
    counts = [3000, 1024, 77, 5000]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, counts, q, heap)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, ok_p, ok_ar, err in res:
        assert err is None, err
        assert ok_p, f"rank {rank}: fused Adam differs from the reference"
        assert ok_ar, f"rank {rank}: allreduce differs from the reference"


def _worker_lamb_rooted(rank, world, port, counts, q):
    """LAMB (GRID and STREAMED: cross-process per-tensor ready flags) and the
    rooted collectives, one process per rank."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import coconet_oracle as co
        from paper_2105_05720_b200 import _lib
        from paper_2105_05720_b200.collectives import LambHParams, TensorList, broadcast, fused_rs_lamb_ag, reduce
        from paper_2105_05720_b200.runtime import Context

        torch.cuda.set_device(0)
        ctx = Context(world, mode="distributed", rank=rank, device=0, heap_bytes=64 << 20, timeout_ms=60000)
        g, p, m, v = _inputs(world, counts)
        outs = {}
        for sched in (_lib.LAMB_GRID, _lib.LAMB_STREAMED, _lib.LAMB_TMA):
            tl = TensorList(ctx, counts, bucket_cap=512)
            gb = [ctx.alloc([n]) for n in counts]
            pb = [ctx.alloc([n]) for n in counts]
            mb, vb = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
            tens, elem, sidx = tl.state_index_map(rank)
            ms = np.zeros(tl.shard_elems, np.float32)
            vs = np.zeros(tl.shard_elems, np.float32)
            for t in range(len(counts)):
                ctx.view(gb[t]).copy_(torch.from_numpy(g[t][rank]))
                ctx.view(pb[t]).copy_(torch.from_numpy(p[t]))
                sel = tens == t
                ms[sidx[sel]] = m[t][elem[sel]]
                vs[sidx[sel]] = v[t][elem[sel]]
            ctx.view(mb).copy_(torch.from_numpy(ms))
            ctx.view(vb).copy_(torch.from_numpy(vs))
            torch.cuda.synchronize()
            dist.barrier()
            first = None
            for step in range(3):
                time.sleep(0.02 * ((rank + step) % world))  # skewed rank start times
                fused_rs_lamb_ag(ctx, tl, gb, pb, mb, vb,
                                 LambHParams(lr=0.01, beta1=0.9, beta2=0.999, t=float(step + 1), sched=sched,
                                             lag_elems=2000))
                ctx.check()
                if step == 0:
                    first = [ctx.view(b).cpu().numpy().copy() for b in pb]
            outs[sched] = ([ctx.view(b).cpu().numpy() for b in pb], first, ctx.view(mb).cpu().numpy(),
                           ctx.view(vb).cpu().numpy())
        same = all(np.array_equal(a, b) for a, b in zip(outs[_lib.LAMB_GRID][0], outs[_lib.LAMB_STREAMED][0]))
        # TMA (m, v, p through the bulk-copy ring, g pulled across processes):
        # m, v bitwise GRID's (they do not depend on p); p by its own segment
        # sums, so against the oracle below
        same = same and np.array_equal(outs[_lib.LAMB_TMA][2], outs[_lib.LAMB_GRID][2]) and np.array_equal(
            outs[_lib.LAMB_TMA][3], outs[_lib.LAMB_GRID][3])
        k = co.lamb_consts(0.01, 0.9, 0.999, 1.0, 1e-6, 0.01)
        table = co.bucket_table(counts)
        flat = co.flatten_bucket_order(g, table)
        bounds = co.flat_chunks(flat.shape[1], world)
        owner = np.searchsorted(np.asarray(bounds[1:]), np.arange(flat.shape[1]), side="right")
        gr = co.unflatten_bucket_order(co.ring_reduce(flat, owner), counts, table)
        dev = max(co.max_rel_deviation(outs[sc][1][t], co.lamb_oracle(gr[t], m[t], v[t], p[t], k)[2])
                  for t in range(len(counts)) for sc in (_lib.LAMB_STREAMED, _lib.LAMB_TMA))
        # a size-1 subgroup inside DISTRIBUTED mode (the bench's NCCL-baseline
        # leg): AUTO picks the TMA schedule; m, v equal GRID's bitwise
        g1 = ctx.group(rank, 1)
        local = {}
        for sched in (_lib.LAMB_AUTO, _lib.LAMB_GRID):
            tl1 = TensorList(ctx, counts, group=g1, bucket_cap=4096)
            gb = [ctx.alloc([n]) for n in counts]
            pb = [ctx.alloc([n]) for n in counts]
            mb, vb = ctx.alloc([tl1.shard_elems]), ctx.alloc([tl1.shard_elems])
            for t in range(len(counts)):
                ctx.view(gb[t]).copy_(torch.from_numpy(g[t][rank]))
                ctx.view(pb[t]).copy_(torch.from_numpy(p[t]))
            ctx.view(mb).zero_()
            ctx.view(vb).fill_(0.05)
            fused_rs_lamb_ag(ctx, tl1, gb, pb, mb, vb, LambHParams(lr=0.01, beta1=0.9, beta2=0.999, t=1.0, sched=sched))
            ctx.check()
            local[sched] = ([ctx.view(b).cpu().numpy() for b in pb], ctx.view(mb).cpu().numpy(), ctx.view(vb).cpu().numpy())
        pa, ma, va = local[_lib.LAMB_AUTO]
        pg, mg, vg = local[_lib.LAMB_GRID]
        same = same and np.array_equal(ma, mg) and np.array_equal(va, vg)
        dev = max(dev, max(co.max_rel_deviation(x, y) for x, y in zip(pa, pg)))
        # rooted collectives
        n = 4099
        x, o = ctx.alloc([n]), ctx.alloc([n])
        xs = np.random.default_rng(3).uniform(-1, 1, (world, n)).astype(np.float32)
        ctx.view(x).copy_(torch.from_numpy(xs[rank]))
        torch.cuda.synchronize()
        dist.barrier()
        reduce(ctx, x, o, root=world - 1)
        ctx.check()
        acc = xs[0].copy()
        for r in range(1, world):
            acc = (acc + xs[r]).astype(np.float32)
        got = ctx.view(o).cpu().numpy()
        ok_red = np.array_equal(got, acc if rank == world - 1 else np.zeros(n, np.float32))
        dist.barrier()
        broadcast(ctx, x, o, root=0)
        ctx.check()
        ok_bc = np.array_equal(ctx.view(o).cpu().numpy(), xs[0])
        dist.barrier()
        ctx.close()
        q.put((rank, same, dev, ok_red, ok_bc, None))
    except Exception as e:  # report, don't hang the parent
        q.put((rank, False, 1.0, False, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_lamb_schedules_and_rooted(world):
    counts = [3000, 1024, 77, 5000, 12_000]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_lamb_rooted, args=(r, world, port, counts, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, same, dev, ok_red, ok_bc, err in res:
        assert err is None, err
        assert same, f"rank {rank}: STREAMED differs from GRID across processes"
        assert dev <= 1e-5, f"rank {rank}: LAMB deviates {dev}"
        assert ok_red and ok_bc, f"rank {rank}: reduce {ok_red} broadcast {ok_bc}"


def _mp_pp_inputs(world, rows, H, r):
    g = torch.Generator().manual_seed(1000 + r)
    k = H // world
    x = torch.randn(rows, k, generator=g).to(torch.bfloat16)
    w = (torch.randn(k, H, generator=g) * k ** -0.5).to(torch.bfloat16)
    gs = torch.Generator().manual_seed(7)
    b = (torch.randn(H, generator=gs) * 0.1).to(torch.bfloat16)
    res = torch.randn(rows, H, generator=gs).to(torch.bfloat16)
    return x, w, b, res


def _run_mp(ctx, ranks, world, rows, H, fused):
    """MatMul + fused RS-bias-dropout-residual-AG on `ctx` for `ranks`:
    fused=False the two kernels, True the tile-flag one-kernel overlap,
    "auto" the AUTO schedule (the all-gather -> GEMM kernel)."""
    from paper_2105_05720_b200 import _lib
    from paper_2105_05720_b200.collectives import BdrHParams, fused_rs_bdr_ag, matmul, mm_overlap_fused_ar
    k = H // world
    xb, wb = ctx.alloc([rows, k], torch.bfloat16), ctx.alloc([k, H], torch.bfloat16)
    bb, rb = ctx.alloc([H], torch.bfloat16), ctx.alloc([rows, H], torch.bfloat16)
    part, out = ctx.alloc([rows, H], torch.bfloat16), ctx.alloc([rows, H], torch.bfloat16)
    for r in ranks:
        x, w, b, res = _mp_pp_inputs(world, rows, H, r)
        ctx.view(xb, r if ctx.mode == "virtual" else None).copy_(x)
        ctx.view(wb, r if ctx.mode == "virtual" else None).copy_(w)
        ctx.view(bb, r if ctx.mode == "virtual" else None).copy_(b)
        ctx.view(rb, r if ctx.mode == "virtual" else None).copy_(res)
    torch.cuda.synchronize()
    if ctx.mode == "distributed":
        dist.barrier()
    hp = BdrHParams(0.1, 1, 11617925594314093840, _lib.MATH_FAST)
    if fused == "auto":
        os.environ.pop("COCONET_MP_OVERLAP", None)
        mm_overlap_fused_ar(ctx, xb, wb, bb, rb, part, out, hp)
    elif fused:  # force the tile-flag one-kernel overlap
        os.environ["COCONET_MP_OVERLAP"] = "fused"
        try:
            mm_overlap_fused_ar(ctx, xb, wb, bb, rb, part, out, hp)
        finally:
            os.environ.pop("COCONET_MP_OVERLAP", None)
    else:
        matmul(ctx, xb, wb, part, math=_lib.MATH_FAST)
        fused_rs_bdr_ag(ctx, part, bb, rb, out, hp)
    ctx.check()
    return {r: ctx.view(out, r if ctx.mode == "virtual" else None).cpu().clone() for r in ranks}


def _worker_mp_pp(rank, world, port, q):
    """The MP epilogue (sequential and overlapped with the tcgen05 GEMM) and
    the PP RS -> send -> AG across processes must equal VIRTUAL mode bitwise."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_05720_b200 import _lib
        from paper_2105_05720_b200.collectives import BdrHParams, rs_fused_send_ag
        from paper_2105_05720_b200.runtime import Context

        torch.cuda.set_device(0)
        rows, H = 256, 128 * world
        dctx = Context(world, mode="distributed", rank=rank, device=0, heap_bytes=256 << 20, timeout_ms=60000)
        got_seq = _run_mp(dctx, [rank], world, rows, H, fused=False)[rank]
        got_ov = _run_mp(dctx, [rank], world, rows, H, fused=True)[rank]
        got_ag = _run_mp(dctx, [rank], world, rows, H, fused="auto")[rank]
        # PP: stages of world/2 ranks
        S = world // 2
        N = 4096 * S
        g0, g1 = dctx.group(0, S), dctx.group(S, S)
        xb, bb, rb, ob = (dctx.alloc([N]) for _ in range(4))
        gen = torch.Generator().manual_seed(50 + rank)
        dctx.view(xb).copy_(torch.randn(N, generator=gen))
        gs = torch.Generator().manual_seed(60)
        dctx.view(bb).copy_(torch.randn(N, generator=gs))
        dctx.view(rb).copy_(torch.randn(N, generator=gs))
        dctx.view(ob).zero_()
        torch.cuda.synchronize()
        dist.barrier()
        rs_fused_send_ag(dctx, g0, g1, xb, bb, rb, ob, BdrHParams(0.1, 1, 3251584743947114031, _lib.MATH_EXACT))
        dctx.check()
        got_pp = dctx.view(ob).cpu().clone()
        dist.barrier()
        dctx.close()
        # the same in VIRTUAL mode, all ranks in this process
        vctx = Context(world, mode="virtual", device=0, heap_bytes=256 << 20)
        want_seq = _run_mp(vctx, list(range(world)), world, rows, H, fused=False)[rank]
        want_ov = _run_mp(vctx, list(range(world)), world, rows, H, fused=True)[rank]
        want_ag = _run_mp(vctx, list(range(world)), world, rows, H, fused="auto")[rank]
        vg0, vg1 = vctx.group(0, S), vctx.group(S, S)
        vx, vb, vr, vo = (vctx.alloc([N]) for _ in range(4))
        gs = torch.Generator().manual_seed(60)
        bvals, rvals = torch.randn(N, generator=gs), torch.randn(N, generator=gs)
        for r in range(world):
            gen = torch.Generator().manual_seed(50 + r)
            vctx.view(vx, r).copy_(torch.randn(N, generator=gen))
            vctx.view(vb, r).copy_(bvals)
            vctx.view(vr, r).copy_(rvals)
            vctx.view(vo, r).zero_()
        rs_fused_send_ag(vctx, vg0, vg1, vx, vb, vr, vo, BdrHParams(0.1, 1, 3251584743947114031, _lib.MATH_EXACT))
        vctx.check()
        want_pp = vctx.view(vo, rank).cpu().clone()
        vctx.close()
        q.put((rank, torch.equal(got_seq, want_seq), torch.equal(got_ov, want_ov) and torch.equal(got_ag, want_ag),
               torch.equal(got_pp, want_pp), None))
    except Exception as e:  # report, don't hang the parent
        q.put((rank, False, False, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_mp_and_pp_match_virtual(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_mp_pp, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, ok_seq, ok_ov, ok_pp, err in res:
        assert err is None, err
        assert ok_seq, f"rank {rank}: MatMul + fused RS-BDR-AG differs from VIRTUAL mode"
        assert ok_ov, f"rank {rank}: overlapped MatMul+AR (tile flags or all-gather -> GEMM) differs from VIRTUAL mode"
        assert ok_pp, f"rank {rank}: PP RS->send->AG differs from VIRTUAL mode"


def _worker_missing_peer(rank, world, port, q):
    """Fault injection: rank 1 never joins the collective. Rank 0's kernel must
    give up on the flag barrier after its watchdog bound and report
    COCONET_ERR_TIMEOUT through check() - not hang - and the GPU must stay
    usable (a fresh context runs)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_05720_b200 import _lib
        from paper_2105_05720_b200.collectives import AdamHParams, TensorList, fused_rs_adam_ag
        from paper_2105_05720_b200.runtime import Context

        torch.cuda.set_device(0)
        ctx = Context(world, mode="distributed", rank=rank, device=0, heap_bytes=16 << 20, timeout_ms=300)
        counts = [4096, 77]
        tl = TensorList(ctx, counts)
        gb = [ctx.alloc([n]) for n in counts]
        pb = [ctx.alloc([n]) for n in counts]
        mb, vb = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
        dist.barrier()
        name, elapsed = None, 0.0
        if rank == 0:
            t0 = time.time()
            fused_rs_adam_ag(ctx, tl, gb, pb, mb, vb,
                             AdamHParams(0.01, 0.9, 0.999, 1.0, 0.0, True, _lib.MATH_FAST, _lib.ALGO_TWO_SHOT))
            try:
                ctx.check()
            except _lib.CoconetError as e:
                name = e.name
            elapsed = time.time() - t0
        dist.barrier()
        ctx.close()
        usable = True
        if rank == 0:
            c2 = Context(1, heap_bytes=16 << 20)
            x = c2.alloc([16])
            c2.view(x, 0).fill_(3.0)
            usable = bool(torch.all(c2.view(x, 0) == 3.0))
            c2.close()
        q.put((rank, name, elapsed, usable, None))
    except Exception as e:
        q.put((rank, "exception", 0.0, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_watchdog_reports_a_missing_peer():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_missing_peer, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    rank0 = res[0]
    assert rank0[4] is None, rank0[4]
    assert rank0[1] == "Timeout", rank0
    assert rank0[2] < 30, f"gave up after {rank0[2]:.1f} s"
    assert rank0[3], "GPU unusable after the watchdog fired"
