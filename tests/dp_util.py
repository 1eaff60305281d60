"""Shared set-up for the data-parallel parity tests: builds the adam / LAMB
workloads on a virtual-rank context exactly as the reference's
gen_decl_values would (state.hpp:55-74), runs the CUDA path, and collects the
results in the reference's result-key form (state.hpp:227-236)."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import torch

from oracle import coconet_oracle as co
from paper_2105_05720_b200 import _lib
from paper_2105_05720_b200.collectives import (AdamHParams, LambHParams, TensorList, fused_rs_adam_ag,
                                               fused_rs_lamb_ag, gen_values)
from paper_2105_05720_b200.runtime import Context

GOLD = Path(__file__).resolve().parent / "golden"


GOLD_DIR = GOLD


def golden_lamb_list(W: int) -> dict:
    """tests/golden/lamb_list_cases.json (oracle/make_lamb_golden.py)."""
    return next(r for r in json.loads((GOLD / "lamb_list_cases.json").read_text()) if r["W"] == W)


def golden(name: str) -> dict:
    for f in GOLD.glob("*_cases.json"):
        for rec in json.loads(f.read_text()):
            if rec["name"] == name:
                return rec
    raise KeyError(name)


class DPWorkload:
    """A tensor list with per-rank gradients, replicated params and sliced
    (or, for one-shot, replicated) optimizer state on a virtual context."""

    def __init__(self, ctx: Context, counts, g_dtype=torch.float32, one_shot=False, names=None,
                 seed=1, bucket_cap=1024):
        self.ctx, self.counts, self.seed = ctx, list(counts), seed
        W = ctx.world
        self.W = W
        self.tl = TensorList(ctx, counts, bucket_cap=bucket_cap)
        self.one_shot = one_shot
        self.grads = [ctx.alloc([n], g_dtype) for n in counts]
        self.params = [ctx.alloc([n], torch.float32) for n in counts]
        st = self.tl.state_elems if one_shot else self.tl.shard_elems
        self.m = ctx.alloc([st], torch.float32)
        self.v = ctx.alloc([st], torch.float32)
        self.names = names or [f"t{i}" for i in range(len(counts))]
        self.maps = [self.tl.state_index_map(-1 if one_shot else r) for r in range(W)]

    # -- inputs ---------------------------------------------------------------
    def gen_dsl(self, g_name="g", p_name="p", m_name="m", v_name="v"):
        """Single-tensor DSL names (goldens/adam.json): g Local, p/m/v by value."""
        assert len(self.counts) == 1
        n = self.counts[0]
        full_m = torch.empty(n, dtype=torch.float32, device="cuda")
        full_v = torch.empty_like(full_m)
        for r in range(self.W):
            gen_values(self.ctx, self.ctx.view(self.grads[0], r), self.seed, g_name, "local", r, [n],
                       group_size=self.W)
            gen_values(self.ctx, self.ctx.view(self.params[0], r), self.seed, p_name, "replicated", r,
                       [n], group_size=self.W)
        gen_values(self.ctx, full_m, self.seed, m_name, "replicated", 0, [n], group_size=self.W)
        gen_values(self.ctx, full_v, self.seed, v_name, "replicated", 0, [n], group_size=self.W)
        self.set_state([full_m], [full_v])

    def set_host(self, grads_by_rank, params, m, v):
        """grads_by_rank[t]: [W, n] ; params/m/v[t]: [n] (global views)."""
        for t in range(len(self.counts)):
            for r in range(self.W):
                self.ctx.view(self.grads[t], r).copy_(torch.from_numpy(grads_by_rank[t][r]))
                self.ctx.view(self.params[t], r).copy_(torch.from_numpy(params[t]))
        self.set_state([torch.from_numpy(x).cuda() for x in m], [torch.from_numpy(x).cuda() for x in v])

    def set_state(self, m_full, v_full):
        for r in range(self.W):
            tens, elem, sidx = self.maps[r]
            for buf, full in ((self.m, m_full), (self.v, v_full)):
                dst = self.ctx.view(buf, r)
                for t in range(len(self.counts)):
                    sel = tens == t
                    if sel.any():
                        dst[torch.from_numpy(sidx[sel]).cuda()] = full[t][torch.from_numpy(elem[sel]).cuda()]

    # -- results --------------------------------------------------------------
    def params_host(self, r=0):
        return [self.ctx.view(p, r).cpu().numpy().copy() for p in self.params]

    def state_host(self):
        """Global views of m and v assembled from every rank's shard."""
        outs = []
        for buf in (self.m, self.v):
            arrs = [np.zeros(n, np.float32) for n in self.counts]
            for r in range(self.W):
                tens, elem, sidx = self.maps[r]
                src = self.ctx.view(buf, r).cpu().numpy()
                for t in range(len(self.counts)):
                    sel = tens == t
                    arrs[t][elem[sel]] = src[sidx[sel]]
            outs.append(arrs)
        return outs

    def dsl_results(self):
        p = self.params_host(0)[0]
        (m,), (v,) = self.state_host()
        return {"out0": [p], "tensor:m": [m], "tensor:p": [p], "tensor:v": [v]}

    def adam(self, hp: AdamHParams):
        fused_rs_adam_ag(self.ctx, self.tl, self.grads, self.params, self.m, self.v, hp)

    def lamb(self, hp: LambHParams):
        fused_rs_lamb_ag(self.ctx, self.tl, self.grads, self.params, self.m, self.v, hp)


def dsl_scalars(seed=1, W=4):
    """Replicated scalar decls of goldens/adam.json as gen_decl_values makes them."""
    return {n: float(co.gen_decl(seed, n, [], "replicated", 0, W)[0])
            for n in ("lr", "beta1", "beta2", "t")}


def new_ctx(W, heap_mb=64):
    return Context(W, mode="virtual", heap_bytes=heap_mb << 20, timeout_ms=5000)
