"""CPU restatement of the reference's hot-path arithmetic (numpy + oracle_c.c).

TEST INFRASTRUCTURE ONLY — the checker for the CUDA path. Imported only by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg; never by the
product package.

Pinned: tests/test_oracle_pinned.py checks every function here against the
compiled reference (oracle/_ref, when present) and against the committed golden
digests in tests/golden/ (generated from the reference by oracle/make_golden.py).

Each function cites the reference routine it restates (paths relative to
/root/reference/proj/include/ccopt/). numpy float64 ufuncs are IEEE
correctly-rounded with no contraction, like the reference's g++ -O2 x86-64
build, so the double-precision element math reproduces eval_expr bit for bit.
"""
from __future__ import annotations

import ctypes as C
import math
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_CLIB = HERE / "_build" / "liboracle_c.so"
_c = None

PHI = np.uint64(0x9E3779B97F4A7C15)
FNV_OFFSET = 0xCBF29CE484222325


def _clib():
    global _c
    if _c is None and _CLIB.exists():
        lib = C.CDLL(str(_CLIB))
        lib.co_fnv1a.restype = C.c_uint64
        lib.co_fnv1a.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
        _c = lib
    return _c


# ---------------------------------------------------------------------------
# FNV-1a (types.hpp:161-170)

def fnv1a(data: bytes | str | np.ndarray, h: int = FNV_OFFSET) -> int:
    if isinstance(data, str):
        data = data.encode()
    if isinstance(data, np.ndarray):
        data = np.ascontiguousarray(data)
        lib = _clib()
        if lib is not None:
            return int(lib.co_fnv1a(data.ctypes.data, data.nbytes, h))
        data = data.tobytes()
    lib = _clib()
    if lib is not None and len(data) > 64:
        buf = C.create_string_buffer(data, len(data))
        return int(lib.co_fnv1a(buf, len(data), h))
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


# ---------------------------------------------------------------------------
# Counter PRNG (expr.hpp:15-27)

def prng_bits(seed: int, key: int, idx) -> np.ndarray:
    """53-bit numerator of counter_uniform; idx: uint64 array-like."""
    with np.errstate(over="ignore"):
        i = np.asarray(idx, dtype=np.uint64)
        x = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(key & 0xFFFFFFFFFFFFFFFF) * PHI) ^ (
            i + np.uint64(0x632BE59BD9B4E019))
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
        return x >> np.uint64(11)


def counter_uniform(seed: int, key: int, idx) -> np.ndarray:
    return prng_bits(seed, key, idx).astype(np.float64) * (1.0 / 9007199254740992.0)


def dropout_keep(seed: int, key: int, idx, rate: float) -> np.ndarray:
    return counter_uniform(seed, key, idx) >= rate


# ---------------------------------------------------------------------------
# DistView / local_shape (view.hpp:17-71) and gen_decl_values (state.hpp:55-74)

def slice_global_index(shape, sliced_dim: int, world: int, rank: int) -> np.ndarray:
    """DistView::to_global(rank, li) for every local index li."""
    shape = [int(s) for s in shape]
    if shape[sliced_dim] % world:
        raise ValueError("DivisibilityError")
    stride = int(np.prod(shape[sliced_dim + 1:])) if sliced_dim + 1 < len(shape) else 1
    per = shape[sliced_dim] // world
    n_local = int(np.prod(shape)) // world
    li = np.arange(n_local, dtype=np.int64)
    before = li // (stride * per)
    lc = (li // stride) % per
    after = li % stride
    return (before * shape[sliced_dim] + rank * per + lc) * stride + after


def decl_key(name: str, layout: str, rank: int) -> int:
    key = fnv1a(name)
    if layout == "local":
        key ^= ((rank + 1) * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    return key


def gen_decl(seed: int, name: str, shape, layout: str, rank: int, world: int,
             sliced_dim: int = -1) -> np.ndarray:
    """Rank-local storage of a decl, as gen_decl_values writes it."""
    n = int(np.prod(shape)) if len(shape) else 1
    gi = (slice_global_index(shape, sliced_dim, world, rank) if layout == "sliced"
          else np.arange(n, dtype=np.int64))
    u = counter_uniform(seed, decl_key(name, layout, rank), gi)
    return (0.1 + 0.8 * u).astype(np.float32)


# ---------------------------------------------------------------------------
# Chunks and the ring reduce-scatter (runtime.hpp:57-92, 302-327)

def flat_chunks(total: int, world: int) -> list[int]:
    return [total * c // world for c in range(world + 1)]


def ring_reduce(xs: np.ndarray, owner, red: str = "sum") -> np.ndarray:
    """xs: [W, n] float32 per-rank values; owner: chunk owner per element
    (scalar or [n]). Chunk c accumulates x[c+1], x[c+2], ..., x[c] in fp32."""
    xs = np.asarray(xs, dtype=np.float32)
    W, n = xs.shape
    owner = np.broadcast_to(np.asarray(owner, dtype=np.int64), (n,))
    cols = np.arange(n)
    acc = xs[(owner + 1) % W, cols].copy()
    for j in range(2, W + 1):
        x = xs[(owner + j) % W, cols]
        if red == "sum":
            acc = (acc + x).astype(np.float32)
        elif red == "max":
            acc = np.where(acc > x, acc, x)
        else:
            acc = np.where(acc < x, acc, x)
    return acc


def rank_order_reduce(xs: np.ndarray) -> np.ndarray:
    """oracle_reduce (oracle.hpp:14-28): double, rank order, rounded once."""
    acc = xs[0].astype(np.float64)
    for r in range(1, xs.shape[0]):
        acc = acc + xs[r].astype(np.float64)
    return acc.astype(np.float32)


# ---------------------------------------------------------------------------
# BucketTable (runtime.hpp:575-614)

def bucket_table(counts, cap: int = 1024):
    """[(tensor, offset, extent, flat_start)] in round-robin order."""
    per = []
    for t, n in enumerate(counts):
        if n <= 0:
            raise ValueError("InvalidInput: tensor has no elements")
        per.append([(t, o, min(cap, n - o)) for o in range(0, n, cap)])
    out = []
    cursor = [0] * len(per)
    remaining = sum(len(b) for b in per)
    flat = 0
    while remaining:
        for i, bs in enumerate(per):
            if cursor[i] < len(bs):
                t, o, e = bs[cursor[i]]
                out.append((t, o, e, flat))
                flat += e
                cursor[i] += 1
                remaining -= 1
    return out


def flatten_bucket_order(arrays, table) -> np.ndarray:
    """Concatenates per-tensor arrays (last axis) in bucket order."""
    return np.concatenate([arrays[t][..., o:o + e] for t, o, e, _ in table], axis=-1)


def unflatten_bucket_order(flat: np.ndarray, counts, table):
    out = [np.zeros(flat.shape[:-1] + (n,), dtype=flat.dtype) for n in counts]
    for t, o, e, f in table:
        out[t][..., o:o + e] = flat[..., f:f + e]
    return out


# ---------------------------------------------------------------------------
# Fused expressions (the three fused patterns)

def adam_consts(lr, beta1, beta2, t, eps=0.0, cv_beta1=True):
    """double constants exactly as eval_expr forms them from the f32 decls."""
    b1, b2 = float(np.float32(beta1)), float(np.float32(beta2))
    tt = float(np.float32(t))
    return dict(b1=b1, b2=b2, cm=1.0 - b1, cv=(1.0 - b1) if cv_beta1 else (1.0 - b2),
                bc1=1.0 - math.pow(b1, tt), bc2=1.0 - math.pow(b2, tt),
                lr=float(np.float32(lr)), eps=float(np.float32(eps)))


def adam_exact(g, m, v, p, k):
    """update(p, p - lr*(update(m, m*beta1 + c*g)/(1-pow(beta1,t))) /
    sqrt(update(v, v*beta2 + c*g*g)/(1-pow(beta2,t)))) in double, the parser's
    association (json_io.hpp:166-183); Update stores float and feeds the
    unrounded double on (expr.hpp:207-211). Returns float32 (m', v', p')."""
    g = np.asarray(g, np.float32).astype(np.float64)
    mn = np.asarray(m, np.float32).astype(np.float64) * k["b1"] + k["cm"] * g
    vn = np.asarray(v, np.float32).astype(np.float64) * k["b2"] + (k["cv"] * g) * g
    m1 = mn / k["bc1"]
    v1 = vn / k["bc2"]
    pn = np.asarray(p, np.float32).astype(np.float64) - (k["lr"] * m1) / (np.sqrt(v1) + k["eps"])
    return mn.astype(np.float32), vn.astype(np.float32), pn.astype(np.float32)


def fused_adam(grads_by_rank, m, v, p, k, counts=None, cap=1024):
    """Tensor-list FusedAllReduce(Adam) with sliced state, as the reference
    Engine computes it on the bucket-order flattening (runtime.hpp:471-516):
    grads_by_rank[t]: [W, n_t]; m, v, p: per-tensor arrays (global views).
    Returns per-tensor (m', v', p')."""
    counts = counts or [g.shape[1] for g in grads_by_rank]
    W = grads_by_rank[0].shape[0]
    table = bucket_table(counts, cap)
    G = flatten_bucket_order(grads_by_rank, table)
    total = G.shape[1]
    bounds = flat_chunks(total, W)
    owner = np.searchsorted(np.asarray(bounds[1:]), np.arange(total), side="right")
    g = ring_reduce(G, owner)
    mf, vf, pf = (flatten_bucket_order(a, table) for a in (m, v, p))
    mn, vn, pn = adam_exact(g, mf, vf, pf, k)
    return tuple(unflatten_bucket_order(a, counts, table) for a in (mn, vn, pn))


def seq_sum(x: np.ndarray) -> float:
    """Sequential double accumulation (eval_pointwise's ReduceTensor loop,
    state.hpp:141-160)."""
    x = np.asarray(x, np.float64)
    return float(np.cumsum(x)[-1]) if x.size else 0.0


def lamb_consts(lr, beta1, beta2, t, eps, wd):
    b1, b2, tt = float(np.float32(beta1)), float(np.float32(beta2)), float(np.float32(t))
    return dict(b1=b1, b2=b2, c1=1.0 - b1, c2=1.0 - b2, bc1=1.0 - math.pow(b1, tt),
                bc2=1.0 - math.pow(b2, tt), lr=float(np.float32(lr)),
                eps=float(np.float32(eps)), wd=float(np.float32(wd)))


def lamb_oracle(g_reduced, m, v, p, k):
    """LAMB golden (tests/golden/lamb_*.json) on one tensor by definition, in
    double:  m' = m*b1 + (1-b1)*g ; v' = v*b2 + (1-b2)*g*g ;
    u = m'/bc1/(sqrt(v'/bc2) + eps) + wd*p ;
    p' = p - lr*sqrt(sum(p*p))/sqrt(sum(u*u))*u."""
    g = np.asarray(g_reduced, np.float32).astype(np.float64)
    p64 = np.asarray(p, np.float32).astype(np.float64)
    mn = np.asarray(m, np.float32).astype(np.float64) * k["b1"] + k["c1"] * g
    vn = np.asarray(v, np.float32).astype(np.float64) * k["b2"] + (k["c2"] * g) * g
    u = (mn / k["bc1"]) / (np.sqrt(vn / k["bc2"]) + k["eps"]) + k["wd"] * p64
    P = seq_sum(p64 * p64)
    U = seq_sum(u * u)
    pn = p64 - ((k["lr"] * math.sqrt(P)) / math.sqrt(U)) * u
    return mn.astype(np.float32), vn.astype(np.float32), pn.astype(np.float32)


def dropout_threshold(rate: float) -> int:
    """smallest integer k with k * 2^-53 >= rate (exact: power-of-two scale)."""
    return int(math.ceil(float(rate) * 9007199254740992.0))


def bdr_exact(x, b, r, rate, seed, key, gidx):
    """dropout(x + b, rate, key) + r (goldens/model_parallel.json,
    pipeline.json) in double with the global flat index as the PRNG counter."""
    s = np.asarray(x, np.float32).astype(np.float64) + np.asarray(b, np.float32).astype(np.float64)
    keep = prng_bits(seed, key, gidx) >= np.uint64(dropout_threshold(rate))
    d = np.where(keep, s / (1.0 - float(rate)), 0.0)
    return (d + np.asarray(r, np.float32).astype(np.float64)).astype(np.float32)


def matmul_exact(x, w):
    """eval_matmul (state.hpp:94-121): double accumulation in k order."""
    x = np.asarray(x, np.float32).astype(np.float64)
    w = np.asarray(w, np.float32).astype(np.float64)
    acc = np.zeros((x.shape[0], w.shape[1]), np.float64)
    for k in range(x.shape[1]):
        acc = acc + x[:, k:k + 1] * w[k:k + 1, :]
    return acc.astype(np.float32)


# ---------------------------------------------------------------------------
# Results (state.hpp:227-274)

def max_rel_deviation(a, b) -> float:
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    if a.shape != b.shape:
        raise ValueError("ShapeMismatch: result sizes differ")
    if a.size == 0:
        return 0.0
    diff = float(np.max(np.abs(a - b)))
    scale = max(1e-12, float(np.max(np.abs(a))), float(np.max(np.abs(b))))
    return diff / scale


def compare_results(a: dict, b: dict) -> float:
    worst = 0.0
    for key, arrs in a.items():
        if key not in b:
            raise KeyError(f"missing result {key}")
        for x, y in zip(arrs, b[key]):
            worst = max(worst, max_rel_deviation(x, y))
    return worst


def digest_results(res: dict) -> int:
    """FNV-1a over keys (std::map order) and raw fp32 bytes."""
    h = FNV_OFFSET
    for key in sorted(res):
        h = fnv1a(key.encode(), h)
        for arr in res[key]:
            h = fnv1a(np.ascontiguousarray(arr, dtype=np.float32), h)
    return h
