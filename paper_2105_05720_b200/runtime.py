"""Context and symmetric memory (Python side of include/coconet_cuda.h).

A `Context` owns one symmetric heap per rank. `SymmBuffer` is an allocation
with the same offset on every rank; `ctx.view(buf, r)` is rank r's copy as a
torch tensor (zero-copy, via __cuda_array_interface__).

VIRTUAL mode keeps all W ranks on one device in this process — the
reference's own in-process rank model (state.hpp:17-20) — and one call runs
every rank. DISTRIBUTED mode is one process per GPU: heap handles are
exchanged through torch.distributed (any backend; NCCL is only bootstrap) and
peers are mapped over NVLink.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check, load

_DTYPES = {torch.float32: _lib.F32, torch.float16: _lib.F16, torch.bfloat16: _lib.BF16}


def elem_of(dtype: torch.dtype) -> int:
    try:
        return _DTYPES[dtype]
    except KeyError:
        raise _lib.CoconetError(3, f"unsupported dtype {dtype}") from None


def exchange_blobs(mine: bytes, world: int, pg=None) -> bytes:
    """All-gathers one fixed-size blob per rank (heap handles) over any
    torch.distributed backend and returns them concatenated in rank order —
    the layout coconet_open_peers expects."""
    import torch.distributed as dist

    allb = [None] * world
    dist.all_gather_object(allb, mine, group=pg)
    if any(b is None or len(b) != len(mine) for b in allb):
        raise _lib.CoconetError(3, "heap handles of different sizes across ranks")
    return b"".join(allb)


def max_over_ranks(value: float, pg=None) -> float:
    """Timing reduction used by bench.py: the job's time is the slowest rank's."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(pg) == 1:
        return float(value)
    dev = "cuda" if dist.get_backend(pg) == "nccl" else "cpu"
    t = torch.tensor([float(value)], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=pg)
    return float(t.item())


class _CAI:
    """Minimal __cuda_array_interface__ exporter for a raw device range."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
            "strides": None,
        }


@dataclass(frozen=True)
class SymmBuffer:
    offset: int
    shape: tuple
    dtype: torch.dtype

    @property
    def numel(self) -> int:
        n = 1
        for s in self.shape:
            n *= int(s)
        return n

    @property
    def nbytes(self) -> int:
        return self.numel * torch.empty((), dtype=self.dtype).element_size()


class Context:
    def __init__(self, world: int, mode: str = "virtual", rank: int = 0, device: int = 0,
                 heap_bytes: int = 1 << 30, process_group=None, timeout_ms: int | None = None,
                 heap: str = "default"):
        self.lib = load()
        self.world = int(world)
        self.mode = mode
        self.rank = int(rank) if mode == "distributed" else 0
        self.device = int(device)
        m = _lib.MODE_VIRTUAL if mode == "virtual" else _lib.MODE_DISTRIBUTED
        h = C.c_void_p()
        torch.cuda.set_device(self.device)
        torch.cuda.init()
        if heap not in _lib.HEAP_KINDS:
            raise ValueError(f"heap must be one of {sorted(_lib.HEAP_KINDS)}")
        check(self.lib.coconet_init_ex(C.byref(h), m, self.rank, self.world, self.device, heap_bytes,
                                       _lib.HEAP_KINDS[heap]))
        self.handle = h
        self.heap_kind = {v: k for k, v in _lib.HEAP_KINDS.items()}[int(self.lib.coconet_heap_kind(h))]
        if timeout_ms is not None:
            check(self.lib.coconet_set_timeout_ms(h, int(timeout_ms)))
        if mode == "distributed":
            self._open_peers(process_group)
            if self.heap_kind == "nvls":
                self._nvls_setup(process_group)
        self._heap_bytes = None
        self._heaps: dict[int, torch.Tensor] = {}
        self._bases: dict[int, int] = {}
        self.groups = {0: (0, self.world)}

    # -- bootstrap -------------------------------------------------------------
    def _open_peers(self, pg):
        import torch.distributed as dist

        n = C.c_size_t(0)
        check(self.lib.coconet_heap_handle(self.handle, None, C.byref(n)))
        buf = (C.c_char * n.value)()
        check(self.lib.coconet_heap_handle(self.handle, buf, C.byref(n)))
        blob = exchange_blobs(bytes(buf), self.world, pg)
        check(self.lib.coconet_open_peers(self.handle, C.c_char_p(blob), n.value))
        dist.barrier(group=pg)

    def _nvls_setup(self, pg):
        """coconet_nvls_setup's three collective stages. After each, the ranks
        agree on success (a MAX all-reduce of the status instead of a bare
        barrier), so a stage that fails on one rank raises on every rank and
        no rank is left waiting in a later collective."""
        import torch.distributed as dist

        dev = "cuda" if dist.get_backend(pg) == "nccl" else "cpu"
        for stage in range(3):
            rc = int(self.lib.coconet_nvls_setup(self.handle, stage))
            msg = _lib.last_error() if rc else ""
            flag = torch.tensor([rc], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=pg)
            if int(flag.item()):
                raise _lib.CoconetError(rc or int(flag.item()),
                                        f"NVLS setup stage {stage}: " + (msg or "failed on another rank"))

    @property
    def nvls(self) -> bool:
        """True when the world group's heaps are mapped through an NVSwitch multicast object."""
        return bool(self.lib.coconet_nvls_mapped(self.handle))

    def close(self):
        if self.handle:
            torch.cuda.synchronize(self.device)
            self._heaps.clear()
            self.lib.coconet_finalize(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- memory ------------------------------------------------------------------
    def local_ranks(self):
        return list(range(self.world)) if self.mode == "virtual" else [self.rank]

    def _heap(self, rank: int) -> torch.Tensor:
        t = self._heaps.get(rank)
        if t is None:
            base = self.lib.coconet_symm_ptr(self.handle, rank, 0)
            if not base:
                raise _lib.CoconetError(14, f"rank {rank}'s heap is not addressable here")
            size = int(self.lib.coconet_heap_bytes(self.handle))
            t = torch.as_tensor(_CAI(base, size), device=f"cuda:{self.device}")
            self._heaps[rank] = t
        return t

    def alloc(self, shape, dtype=torch.float32) -> SymmBuffer:
        shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        buf = SymmBuffer(0, shape, dtype)
        off = C.c_size_t(0)
        check(self.lib.coconet_symm_alloc(self.handle, max(1, buf.nbytes), C.byref(off)))
        return SymmBuffer(off.value, shape, dtype)

    def free(self, buf: SymmBuffer):
        """Returns `buf` to the symmetric heap (collective, like alloc)."""
        check(self.lib.coconet_symm_free(self.handle, buf.offset))

    def reset(self):
        check(self.lib.coconet_symm_reset(self.handle))

    def high_water(self) -> int:
        return int(self.lib.coconet_symm_high_water(self.handle))

    def view(self, buf: SymmBuffer, rank: int | None = None) -> torch.Tensor:
        r = self.rank if rank is None else rank
        h = self._heap(r)
        return h[buf.offset:buf.offset + buf.nbytes].view(buf.dtype).view(buf.shape)

    def ptr(self, buf: SymmBuffer, rank: int | None = None) -> int:
        r = (0 if self.mode == "virtual" else self.rank) if rank is None else rank
        base = self._bases.get(r)
        if base is None:  # heap bases are fixed for the context's lifetime
            base = self._bases[r] = int(self.lib.coconet_symm_ptr(self.handle, r, 0) or 0)
        return base + buf.offset if base else int(self.lib.coconet_symm_ptr(self.handle, r, buf.offset) or 0)

    # -- groups / sync -------------------------------------------------------------
    def group(self, first_rank: int, size: int) -> int:
        g = C.c_int(0)
        check(self.lib.coconet_group_create(self.handle, first_rank, size, C.byref(g)))
        self.groups[g.value] = (first_rank, size)
        return g.value

    @staticmethod
    def stream_ptr(stream=None) -> int:
        if stream is None:  # the raw handle without building a Stream object
            return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())
        return int(stream.cuda_stream)

    def check(self, stream=None):
        check(self.lib.coconet_check(self.handle, C.c_void_p(self.stream_ptr(stream))))

    def launch_count(self) -> int:
        return int(self.lib.coconet_launch_count(self.handle))


def nvls_supported(device: int = 0, world: int = 8) -> tuple[bool, str]:
    """(supported, reason) for an NVSwitch multicast object over `world` GPUs."""
    lib = load()
    why = C.create_string_buffer(256)
    ok = bool(lib.coconet_nvls_supported(int(device), int(world), why, 256))
    return ok, why.value.decode()
