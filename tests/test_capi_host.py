"""CPU: the C-ABI library loads, exports every entry point include/*.h
declares, and its host-side logic (bucket tables, chunking, shard layout,
error codes) matches the reference's definitions — no device needed."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import coconet_oracle as co
from paper_2105_05720_b200 import _lib
from paper_2105_05720_b200.collectives import TensorList

ROOT = Path(__file__).resolve().parent.parent


def declared(header: Path):
    text = re.sub(r"/\*.*?\*/", "", header.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(coconet_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared(ROOT / "include" / "coconet_cuda.h")
    assert len(names) > 30
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (coconet_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert getattr(lib, n)
    # and the binding table covers the header
    assert set(_lib.exported_symbols()) >= set(names)


def test_status_names_mirror_errcode():
    lib = _lib.load()
    # ErrCode order (types.hpp:102-124): status = index + 1
    for status, name in [(1, "LayoutMismatch"), (3, "InvalidInput"), (14, "NoSuchRank"),
                         (16, "DivisibilityError"), (17, "ReplicationViolation"), (101, "Timeout")]:
        assert lib.coconet_status_name(status).decode() == name
        assert _lib.CoconetError(status, "x").name == name


def test_init_without_device_fails_loudly():
    # no GPU in this container: init must return a CUDA error, never crash or fall back
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    lib = _lib.load()
    h = C.c_void_p()
    rc = lib.coconet_init(C.byref(h), _lib.MODE_VIRTUAL, 0, 2, 0, 1 << 20)
    assert rc == 100 and not h.value
    assert lib.coconet_last_error()


def test_plan_rejects_like_the_reference():
    with pytest.raises(_lib.CoconetError) as e:
        TensorList(None, [5, 0, 3], world=2)          # build_bucket_table: no elements
    assert e.value.name == "InvalidInput"
    with pytest.raises(_lib.CoconetError) as e:
        TensorList(None, [1, 2], world=4)             # fewer elements than ranks
    assert e.value.name == "DivisibilityError"
    with pytest.raises(_lib.CoconetError) as e:
        TensorList(None, [8], world=9)
    assert e.value.name == "NoSuchRank"


@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("counts", [[10, 1500, 3, 700], [1024] * 5, [1, 1, 1, 1, 1, 1, 1, 1, 5000],
                                    [336_232 + 2, 4096, 31]])
def test_segment_tables_cover_flat_chunks(W, counts):
    """Every element is owned by exactly one rank; rank r's elements are the
    flat chunk [total*r/W, total*(r+1)/W) of the round-robin bucket order
    (runtime.hpp:63-66, 592-614); shard indices are unique, in range, and
    quad-aligned with the tensor offsets."""
    if sum(counts) < W:
        pytest.skip()
    tl = TensorList(None, counts, world=W)
    table = co.bucket_table(counts)
    assert tl.n_buckets == len(table)
    total = sum(counts)
    assert tl.total == total
    # bucket-order flat position of each (tensor, element)
    flatpos = [np.zeros(n, np.int64) for n in counts]
    for t, o, e, f in table:
        flatpos[t][o:o + e] = np.arange(f, f + e)
    seen = np.zeros(total, np.int32)
    for r in range(W):
        lo, hi = tl.chunk(r)
        assert (lo, hi) == (total * r // W, total * (r + 1) // W)
        tens, elem, sidx = tl.state_index_map(r)
        fp = np.array([flatpos[t][e] for t, e in zip(tens, elem)], dtype=np.int64)
        assert np.all((fp >= lo) & (fp < hi))
        assert np.all(np.diff(fp) > 0)
        seen[fp] += 1
        assert len(np.unique(sidx)) == len(sidx)
        assert sidx.max(initial=0) < tl.shard_elems
        assert np.all((sidx % 4) == (elem % 4))
    assert np.all(seen == 1)
    # one-shot table: every element once, each segment has one owner
    tens, elem, sidx = tl.state_index_map(-1)
    assert len(tens) == total and len(np.unique(sidx)) == total and sidx.max() < tl.state_elems
    assert np.all((sidx % 4) == (elem % 4))


def test_bert_large_list_plan():
    from paper_2105_05720_b200.workloads import BERT_LARGE_PARAMS, bert_large_counts
    counts = bert_large_counts()
    assert len(counts) == 398 and sum(counts) == BERT_LARGE_PARAMS
    tl = TensorList(None, counts, world=8)
    assert tl.n_buckets == sum(-(-n // 1024) for n in counts)
    # shard storage overhead of the alignment padding is tiny
    assert tl.shard_elems < BERT_LARGE_PARAMS / 8 * 1.01


def _global_groups(counts_per_rank, lag):
    """Restatement of tlist_stream_plan's global (pass, tensor) sequence."""
    size = np.max(counts_per_rank, axis=0)
    groups, pending, pos = [], [], 0
    for t in range(len(size)):
        groups.append((0, t))
        pos += int(size[t])
        pending.append((t, pos))
        while pending and pending[0][1] + lag <= pos:
            groups.append((1, pending.pop(0)[0]))
    groups += [(1, t) for t, _ in pending]
    return groups


@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("counts,cap,lag", [([10, 1500, 3, 700], 1024, 512),
                                             ([1024] * 5, 256, 1024),
                                             ([1, 1, 1, 1, 1, 1, 1, 1, 5000], 1024, 64),
                                             ([336_232 + 2, 4096, 31, 9000, 70_000], 4096, 20_000)])
def test_stream_plan_is_complete_and_deadlock_free(W, counts, cap, lag):
    """STREAMED-LAMB work lists: every segment of rank r appears once per pass;
    each tensor's pass-1 items are contiguous and in toff order; every rank's
    (pass, tensor) group order is a subsequence of ONE global sequence in which
    P2(t) follows P1(t) and P2(t) starts only after `lag` more elements of
    pass 1 (or at the end) - which is what makes the persistent grid
    deadlock-free across ranks."""
    if sum(counts) < W:
        pytest.skip()
    tl = TensorList(None, counts, world=W, bucket_cap=cap)
    elems = np.zeros((W, len(counts)), np.int64)
    for r in range(W):
        segs = tl.segments(r)
        np.add.at(elems[r], segs[:, 0], segs[:, 2])
    glob = _global_groups(elems, lag)
    gpos = {g: i for i, g in enumerate(glob)}
    for t in range(len(counts)):
        assert gpos[(1, t)] > gpos[(0, t)]
    for r in range(W):
        items = tl.stream_items(lag, r)
        segs = tl.segments(r)
        key = lambda a: sorted(map(tuple, a[:, :3].tolist()))
        assert key(items[items[:, 3] == 0]) == key(segs[:, :3]) == key(items[items[:, 3] == 1])
        order = [gpos[(int(p), int(t))] for t, p in zip(items[:, 0], items[:, 3])]
        assert np.all(np.diff(order) >= 0), "rank list must follow the global group sequence"
        for t in np.unique(items[:, 0]):
            idx1 = np.nonzero((items[:, 0] == t) & (items[:, 3] == 0))[0]
            assert np.all(np.diff(idx1) == 1)
            assert np.all(np.diff(items[idx1, 1]) > 0)


def test_stream_plan_bert_large_lag():
    """BERT-336M at W=1, default lag 2^21: between a tensor's last pass-1 item
    and its first pass-2 item there are at least `lag` elements of pass-1 work
    (except the tail), so the grid's in-flight window (~1.2M elements) never
    reaches a tensor whose pass 1 is still running."""
    from paper_2105_05720_b200.workloads import bert_large_counts
    counts = bert_large_counts()
    lag = 1 << 21
    tl = TensorList(None, counts, world=1, bucket_cap=4096)
    items = tl.stream_items(lag, 0)
    assert len(items) == 2 * len(tl.segments(0))
    p1_elems = np.cumsum(np.where(items[:, 3] == 0, items[:, 2], 0))
    total = p1_elems[-1]
    for t in range(len(counts)):
        i1 = np.nonzero((items[:, 0] == t) & (items[:, 3] == 0))[0][-1]
        i2 = np.nonzero((items[:, 0] == t) & (items[:, 3] == 1))[0][0]
        assert p1_elems[i2] - p1_elems[i1] >= lag or p1_elems[i2] == total
