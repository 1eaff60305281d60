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
