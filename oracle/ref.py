"""ctypes wrapper of oracle/_ref/libccopt_ref.so — the UNMODIFIED reference
(ccopt headers compiled in place, oracle/Makefile) behind oracle/ref_capi.cpp.

TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, as the checker and the CPU
baseline. The product never imports this module.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libccopt_ref.so"

ORACLE, ENGINE_SCHED, ENGINE_BASE = 0, 1, 2

_lib = None


def available() -> bool:
    return LIB.exists()


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise FileNotFoundError(f"{LIB} not built (make -C oracle ref; needs /root/reference)")
        lib = C.CDLL(str(LIB))
        P, I, I64, U64, D = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
        FP = C.POINTER(C.c_float)
        sig = {
            "ccref_last_error": (C.c_char_p, []),
            "ccref_open": (P, [C.c_char_p, C.c_char_p, C.c_char_p]),
            "ccref_open_pair": (P, [C.c_char_p, C.c_char_p, C.c_char_p]),
            "ccref_close": (None, [P]),
            "ccref_gen": (I, [P, U64]),
            "ccref_set": (I, [P, C.c_char_p, I, FP, I64]),
            "ccref_get_input": (I, [P, C.c_char_p, I, FP, I64]),
            "ccref_run": (I, [P, U64, I, I, C.POINTER(D)]),
            "ccref_time_engine": (D, [P, U64, I, I]),
            "ccref_result_keys": (I, [P, I, C.c_char_p, I64]),
            "ccref_result": (I, [P, I, C.c_char_p, I, FP, I64]),
            "ccref_value": (I, [P, C.c_char_p, I, FP, I64]),
            "ccref_digest": (U64, [P, I]),
            "ccref_compare": (D, [P, I, I]),
            "ccref_report": (I, [P, I, C.c_char_p, I64]),
            "ccref_program_json": (I, [P, I, C.c_char_p, I64]),
            "ccref_fnv1a": (U64, [P, I64, U64]),
            "ccref_counter_uniform": (D, [U64, U64, U64]),
            "ccref_bucket_table": (I64, [I, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64),
                                         C.POINTER(I64), I64]),
            "ccref_bucket_metadata_bytes": (I64, [I, C.POINTER(I64)]),
            "ccref_scattered_allreduce": (I, [I, C.POINTER(I64), I, C.POINTER(FP), C.POINTER(FP)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class RefError(RuntimeError):
    pass


def _check(rc):
    if rc < 0:
        raise RefError(load().ccref_last_error().decode())
    return rc


def _fp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


class RefSession:
    """One reference program (+ schedule) at concrete sizes.

    mirrors `ccopt run` (tools/ccopt.cpp:184-193): program_from_json ->
    apply_schedule -> gen_decl_values -> oracle / Engine -> compare / digest.
    """

    def __init__(self, program: str | dict, schedule: str | dict | None = None,
                 dims: dict | None = None, sched_program: str | dict | None = None):
        lib = load()
        prog = program if isinstance(program, str) else json.dumps(program)
        d = json.dumps(dims or {}).encode()
        if sched_program is not None:
            sp = sched_program if isinstance(sched_program, str) else json.dumps(sched_program)
            self.h = lib.ccref_open_pair(prog.encode(), sp.encode(), d)
        else:
            sch = b"" if schedule is None else (schedule if isinstance(schedule, str)
                                                 else json.dumps(schedule)).encode()
            self.h = lib.ccref_open(prog.encode(), sch, d)
        if not self.h:
            raise RefError(lib.ccref_last_error().decode())
        self.lib = lib

    def close(self):
        if self.h:
            self.lib.ccref_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def gen(self, seed: int):
        _check(self.lib.ccref_gen(self.h, seed))

    def set(self, name: str, rank: int, data: np.ndarray):
        a = np.ascontiguousarray(data, dtype=np.float32).ravel()
        _check(self.lib.ccref_set(self.h, name.encode(), rank, _fp(a), a.size))

    def get_input(self, name: str, rank: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.float32)
        _check(self.lib.ccref_get_input(self.h, name.encode(), rank, _fp(out), n))
        return out

    def run(self, seed: int, which: int, threaded: bool = False) -> float:
        t = C.c_double()
        _check(self.lib.ccref_run(self.h, seed, which, int(threaded), C.byref(t)))
        return t.value

    def time_engine(self, seed: int, which: int = ENGINE_SCHED, threaded: bool = False) -> float:
        t = self.lib.ccref_time_engine(self.h, seed, which, int(threaded))
        if t < 0:
            raise RefError(self.lib.ccref_last_error().decode())
        return t

    def result_keys(self, which: int) -> list[tuple[str, int, int]]:
        buf = C.create_string_buffer(1 << 16)
        _check(self.lib.ccref_result_keys(self.h, which, buf, len(buf)))
        out = []
        for line in buf.value.decode().splitlines():
            k, n, e = line.split("\t")
            out.append((k, int(n), int(e)))
        return out

    def result(self, which: int, key: str, idx: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.float32)
        _check(self.lib.ccref_result(self.h, which, key.encode(), idx, _fp(out), n))
        return out

    def results(self, which: int) -> dict[str, list[np.ndarray]]:
        return {k: [self.result(which, k, i, e) for i in range(n)] for k, n, e in self.result_keys(which)}

    def value(self, node: str, rank: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.float32)
        _check(self.lib.ccref_value(self.h, node.encode(), rank, _fp(out), n))
        return out

    def digest(self, which: int) -> int:
        return int(self.lib.ccref_digest(self.h, which))

    def compare(self, a: int, b: int) -> float:
        d = self.lib.ccref_compare(self.h, a, b)
        if d < 0:
            raise RefError(self.lib.ccref_last_error().decode())
        return d

    def report(self, which: int) -> dict:
        buf = C.create_string_buffer(1 << 20)
        _check(self.lib.ccref_report(self.h, which, buf, len(buf)))
        return json.loads(buf.value.decode())

    def program_json(self, which: int) -> dict:
        n = 1 << 20
        while True:
            buf = C.create_string_buffer(n)
            rc = self.lib.ccref_program_json(self.h, which, buf, n)
            if rc >= 0:
                return json.loads(buf.value.decode())
            n = -rc + 16


def counter_uniform(seed: int, key: int, idx: int) -> float:
    return load().ccref_counter_uniform(seed, key, idx)


def bucket_table(counts) -> list[tuple[int, int, int]]:
    lib = load()
    n = len(counts)
    c = (C.c_int64 * n)(*counts)
    cap = sum((x + 1023) // 1024 for x in counts) + 1
    t = (C.c_int64 * cap)()
    o = (C.c_int64 * cap)()
    e = (C.c_int64 * cap)()
    nb = _check(lib.ccref_bucket_table(n, c, t, o, e, cap))
    return [(t[i], o[i], e[i]) for i in range(nb)]


def bucket_metadata_bytes(counts) -> int:
    n = len(counts)
    return int(load().ccref_bucket_metadata_bytes(n, (C.c_int64 * n)(*counts)))


def scattered_allreduce(tensors: list[np.ndarray]) -> list[np.ndarray]:
    """tensors[i]: [world, count_i] float32 -> same shape results."""
    lib = load()
    n = len(tensors)
    world = tensors[0].shape[0]
    counts = (C.c_int64 * n)(*[t.shape[1] for t in tensors])
    ins = [np.ascontiguousarray(t, np.float32) for t in tensors]
    outs = [np.zeros_like(t) for t in ins]
    FP = C.POINTER(C.c_float)
    _check(lib.ccref_scattered_allreduce(n, counts, world, (FP * n)(*[_fp(a) for a in ins]),
                                         (FP * n)(*[_fp(a) for a in outs])))
    return outs
