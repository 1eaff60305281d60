"""Python binding of GpuEngine (include/coconet/gpu_engine.hpp), the drop-in
for ccopt::Engine: load a program (+ schedule) in the reference's JSON
formats, generate inputs with the reference's gen_decl_values, run every plan
step on the GPU, read back the RunReport (results, counters, digest)."""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np

from . import _lib

LIB = Path(__file__).resolve().parent / "libcoconet_engine.so"
_elib = None

SCHEDULED, BASE = 0, 1

# void (*)(const void* in, size_t bytes, void* out, void* user)
ALLGATHER_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


def torch_allgather(process_group=None):
    """A world all-gather over torch.distributed (any backend; gloo in the
    tests) in the engine's callback form: raw bytes in, world x bytes out."""
    import torch
    import torch.distributed as dist

    def fn(src, nbytes, dst, _user):
        world = dist.get_world_size(process_group)
        buf = torch.frombuffer(C.string_at(src, nbytes), dtype=torch.uint8) if nbytes else torch.empty(0, dtype=torch.uint8)
        out = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(out, buf.clone(), group=process_group)
        flat = torch.cat(out).numpy() if nbytes else np.empty(0, np.uint8)
        C.memmove(dst, flat.ctypes.data, flat.nbytes)
    return fn


def load():
    global _elib
    if _elib is None:
        _lib.load()  # libcoconet_cuda first (the engine links it)
        if not LIB.exists():
            raise ImportError(f"{LIB} missing: it is built by __graft_entry__.build() where the DSL headers exist")
        lib = C.CDLL(str(LIB))
        P, I, I64, U64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64
        FP = C.POINTER(C.c_float)
        for name, res, args in [
            ("coconet_engine_last_error", C.c_char_p, []),
            ("coconet_engine_open", P, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p]),
            ("coconet_engine_close", None, [P]),
            ("coconet_engine_gen", I, [P, U64]),
            ("coconet_engine_set", I, [P, C.c_char_p, I, FP, I64]),
            ("coconet_engine_run", I, [P, U64, I, I, I, I]),
            ("coconet_engine_run_dist", I, [P, U64, I, I, I, I, I, I, ALLGATHER_FN, P]),
            ("coconet_engine_digest", U64, [P]),
            ("coconet_engine_report", I, [P, C.c_char_p, I64]),
            ("coconet_engine_result", I, [P, C.c_char_p, I, FP, I64]),
            ("coconet_engine_tune", I, [C.c_char_p, C.c_char_p, U64, C.c_double, I, I, I, C.c_char_p, I64]),
        ]:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _elib = lib
    return _elib


class EngineError(RuntimeError):
    pass


def _check(rc):
    if rc < 0:
        raise EngineError(load().coconet_engine_last_error().decode())
    return rc


class GpuEngineSession:
    def __init__(self, program, schedule=None, dims=None, sched_program=None):
        lib = load()
        enc = lambda x: b"" if x is None else (x if isinstance(x, str) else json.dumps(x)).encode()
        self.h = lib.coconet_engine_open(enc(program), enc(schedule), enc(sched_program),
                                         json.dumps(dims or {}).encode())
        if not self.h:
            raise EngineError(lib.coconet_engine_last_error().decode())
        self.lib = lib

    def close(self):
        if self.h:
            self.lib.coconet_engine_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def gen(self, seed: int):
        _check(self.lib.coconet_engine_gen(self.h, seed))

    def set(self, name: str, rank: int, data: np.ndarray):
        a = np.ascontiguousarray(data, dtype=np.float32).ravel()
        _check(self.lib.coconet_engine_set(self.h, name.encode(), rank,
                                           a.ctypes.data_as(C.POINTER(C.c_float)), a.size))

    def run(self, seed: int, which: int = SCHEDULED, device: int = 0, math: int = _lib.MATH_EXACT,
            fused: bool = True, rank: int | None = None, world: int = 0, allgather=None):
        """VIRTUAL (rank None): every rank in this process. DISTRIBUTED: this
        process is world rank `rank`; `allgather(src, nbytes, dst, user)` is a
        collective world all-gather (engine.torch_allgather() for
        torch.distributed)."""
        if rank is None:
            _check(self.lib.coconet_engine_run(self.h, seed, which, device, math, int(fused)))
            return
        cb = ALLGATHER_FN(allgather)
        self._cb = cb  # keep the trampoline alive for the call
        _check(self.lib.coconet_engine_run_dist(self.h, seed, which, device, math, int(fused), rank, world, cb, None))

    def digest(self) -> int:
        return int(self.lib.coconet_engine_digest(self.h))

    def report(self) -> dict:
        buf = C.create_string_buffer(1 << 20)
        _check(self.lib.coconet_engine_report(self.h, buf, len(buf)))
        return json.loads(buf.value.decode())

    def result(self, key: str, idx: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.float32)
        _check(self.lib.coconet_engine_result(self.h, key.encode(), idx,
                                              out.ctypes.data_as(C.POINTER(C.c_float)), n))
        return out


def gpu_tune(program, dims=None, seed: int = 1, tol: float = 1e-5, device: int = 0,
             math: int = _lib.MATH_EXACT, reps: int = 3) -> dict:
    """ccopt tune (autotune.hpp:285-315) over the reference's own candidate
    schedules, each verified against the oracle and ranked by MEASURED device
    time on the GPU (include/coconet/gpu_tune.hpp). Returns the tune report
    (reference fields + device_ms per candidate, winner by device_ms, and the
    reference's simulated_winner)."""
    lib = load()
    prog = program if isinstance(program, str) else json.dumps(program)
    n = 1 << 20
    while True:
        buf = C.create_string_buffer(n)
        rc = lib.coconet_engine_tune(prog.encode(), json.dumps(dims or {}).encode(), seed, tol, device, math,
                                     reps, buf, n)
        if rc == -1000 or rc >= 0 or -rc <= 30:
            _check(rc)
            return json.loads(buf.value.decode())
        n = -rc
