"""Per-tensor LAMB golden over a TENSOR LIST, evaluated by the UNMODIFIED
reference (oracle/_ref). TEST INFRASTRUCTURE ONLY.

Run here (where /root/reference exists):  python -m oracle.make_lamb_golden

The reference ships no LAMB program; tests/golden/lamb_*.json
author a single-tensor one. LAMB's trust ratio is per tensor, so a tensor
list is one fused node per tensor ("per-tensor trust ratio
means one node per tensor"). This script authors those programs in the
reference JSON format for a list of T tensors:

  base  : per tensor i  avg_i = allreduce(g_i); m_i', v_i', u_i pointwise;
          p_i' = update(p_i, p_i - lr*sqrt(reduce_sum(p_i*p_i))/sqrt(reduce_sum(u_i*u_i))*u_i)
  fused : per tensor i  one fused_allreduce (RS -> LAMB on the slice with the
          nested ReduceTensor cross-rank sums, state.hpp:139-174 /
          runtime.hpp:489-495 -> AG of p_i), m_i / v_i sliced

and records, for W = 1, 2, 4, 8 at seed 1: the oracle (base program) and
Engine (fused program) digests, their deviation, and the Engine's result
arrays (tensor:p_i, tensor:m_i, tensor:v_i), written to
tests/golden/lamb_list_cases.json + lamb_list_results.npz. The GPU box has no
reference: its tests compare the CUDA tensor-list kernel with these arrays.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

from oracle import coconet_oracle as co
from oracle import ref

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden"

COUNTS = [1000, 2048, 8, 504, 3072]  # every count divisible by 8 (Sliced(0) m, v: view.hpp:20-22)
WORLDS = [1, 2, 4, 8]
SCALARS = ("lr", "beta1", "beta2", "t", "eps", "wd")

U_EXPR = ("update(m{i}, m{i}*beta1 + (1-beta1)*{g})/(1 - pow(beta1, t)) / "
          "(sqrt(update(v{i}, v{i}*beta2 + (1-beta2)*{g}*{g})/(1 - pow(beta2, t))) + eps) + wd*p{i}")


def _decls(counts, sliced_state: bool, g_elem: str):
    ts = []
    for i, n in enumerate(counts):
        ts.append({"name": f"g{i}", "elem": g_elem, "shape": [n], "layout": {"kind": "local"}, "group": 0})
        ts.append({"name": f"p{i}", "elem": "f32", "shape": [n], "layout": {"kind": "replicated"}, "group": 0})
        for s in ("m", "v"):
            lay = {"kind": "sliced", "dim": 0} if sliced_state else {"kind": "replicated"}
            ts.append({"name": f"{s}{i}", "elem": "f32", "shape": [n], "layout": lay, "group": 0})
    for s in SCALARS:
        ts.append({"name": s, "elem": "f32", "shape": [], "layout": {"kind": "replicated"}, "group": 0})
    return ts


def base_program(counts, g_elem="f32") -> dict:
    nodes, outs = [], []
    for i in range(len(counts)):
        nodes += [
            {"id": f"avg{i}", "kind": "allreduce", "inputs": [f"g{i}"]},
            {"id": f"m{i}_", "kind": "pointwise", "inputs": [f"m{i}", "beta1", f"avg{i}"],
             "attrs": {"expr": f"update(m{i}, m{i}*beta1 + (1-beta1)*avg{i})"}},
            {"id": f"v{i}_", "kind": "pointwise", "inputs": [f"v{i}", "beta2", f"avg{i}"],
             "attrs": {"expr": f"update(v{i}, v{i}*beta2 + (1-beta2)*avg{i}*avg{i})"}},
            {"id": f"u{i}", "kind": "pointwise",
             "inputs": [f"m{i}_", f"v{i}_", "beta1", "beta2", "t", "eps", "wd", f"p{i}"],
             "attrs": {"expr": f"m{i}_/(1 - pow(beta1, t)) / (sqrt(v{i}_/(1 - pow(beta2, t))) + eps) + wd*p{i}"}},
            {"id": f"p{i}_", "kind": "pointwise", "inputs": [f"p{i}", "lr", f"u{i}"],
             "attrs": {"expr": f"update(p{i}, p{i} - lr*sqrt(reduce_sum(p{i}*p{i}))/sqrt(reduce_sum(u{i}*u{i}))*u{i})"}},
        ]
        outs.append(f"p{i}_")
    return {"name": "lamb_list", "groups": [{"id": 0, "size": "W"}], "tensors": _decls(counts, False, g_elem),
            "nodes": nodes, "outputs": outs}


def fused_program(counts, g_elem="f32") -> dict:
    nodes, outs = [], []
    for i in range(len(counts)):
        u = U_EXPR.format(i=i, g=f"g{i}")
        expr = f"update(p{i}, p{i} - lr*sqrt(reduce_sum(p{i}*p{i}))/sqrt(reduce_sum(({u})*({u})))*({u}))"
        nodes.append({"id": f"f{i}", "kind": "fused_allreduce",
                      "inputs": [f"g{i}", f"m{i}", "beta1", f"v{i}", "beta2", "t", "eps", "wd", f"p{i}", "lr"],
                      "attrs": {"axis": 0, "gather": f"p{i}", "stages": 4, "expr": expr}})
        outs.append(f"f{i}")
    return {"name": "lamb_list_fused", "groups": [{"id": 0, "size": "W"}], "tensors": _decls(counts, True, g_elem),
            "nodes": nodes, "outputs": outs}


def restated(counts, W, seed=1):
    """co.lamb_oracle per tensor on the restated inputs: the reference's
    per-tensor RS (ring order of each tensor's own chunk owner) then the LAMB
    definition in double."""
    sc = {s: float(co.gen_decl(seed, s, [], "replicated", 0, W)[0]) for s in SCALARS}
    k = co.lamb_consts(*(sc[s] for s in SCALARS))
    out = {}
    for i, n in enumerate(counts):
        g = np.stack([co.gen_decl(seed, f"g{i}", [n], "local", r, W) for r in range(W)])
        p, m, v = (co.gen_decl(seed, f"{s}{i}", [n], "replicated", 0, W) for s in ("p", "m", "v"))
        gr = g[0]
        if W > 1:  # Sliced(0): rank c owns [c*n/W, (c+1)*n/W) of this tensor
            owner = np.searchsorted(np.asarray(co.flat_chunks(n, W)[1:]), np.arange(n), side="right")
            gr = co.ring_reduce(g, owner)
        mo, vo, po = co.lamb_oracle(gr, m, v, p, k)
        out[i] = (po, mo, vo)
    return out


def main():
    if not ref.available():
        sys.exit("oracle/_ref/libccopt_ref.so missing: make -C oracle ref")
    base, fused = base_program(COUNTS), fused_program(COUNTS)
    (OUT / "lamb_list_program.json").write_text(json.dumps(base, indent=1))
    (OUT / "lamb_list_fused_program.json").write_text(json.dumps(fused, indent=1))
    recs, arrays = [], {}
    for W in WORLDS:
        s = ref.RefSession(base, None, {"W": W}, sched_program=fused)
        s.gen(1)
        s.run(1, ref.ORACLE)
        s.run(1, ref.ENGINE_SCHED)
        res = s.results(ref.ENGINE_SCHED)
        rec = {"name": f"lamb_list_W{W}", "W": W, "counts": COUNTS, "seed": 1,
               "engine_sched_digest": "%016x" % s.digest(ref.ENGINE_SCHED),
               "oracle_digest": "%016x" % s.digest(ref.ORACLE),
               "deviation_sched_vs_oracle": s.compare(ref.ORACLE, ref.ENGINE_SCHED),
               "scalars": {n: float(s.get_input(n, 0, 1)[0]) for n in SCALARS}}
        rest = restated(COUNTS, W)
        dev = 0.0
        for i in range(len(COUNTS)):
            for name, j in (("p", 0), ("m", 1), ("v", 2)):
                a = res[f"tensor:{name}{i}"][0]
                arrays[f"W{W}_{name}{i}"] = a
                dev = max(dev, co.max_rel_deviation(rest[i][j], a))
        rec["restated_vs_engine"] = dev
        recs.append(rec)
        print(rec["name"], rec["engine_sched_digest"], "oracle dev", rec["deviation_sched_vs_oracle"],
              "restated dev", dev)
    (OUT / "lamb_list_cases.json").write_text(json.dumps(recs, indent=1))
    np.savez_compressed(OUT / "lamb_list_results.npz", **arrays)


if __name__ == "__main__":
    main()
