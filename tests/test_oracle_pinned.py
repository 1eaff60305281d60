"""CPU: the restated oracle (oracle/coconet_oracle.py) pinned against the
reference itself (oracle/_ref, compiled in place from /root/reference when
present) and against the committed golden fixtures the reference generated
(tests/golden, oracle/make_golden.py)."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import coconet_oracle as co
from oracle import ref

GOLD = Path(__file__).resolve().parent / "golden"
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (no /root/reference)")


def cases(kind):
    return json.loads((GOLD / f"{kind}_cases.json").read_text())


def test_prng_known_values():
    # counter_uniform(seed, key, idx) (expr.hpp:15-23): values pinned from the reference
    assert co.fnv1a("dropout") == 11617925594314093840  # mp dropout key
    assert co.fnv1a("send") == 3251584743947114031       # pp dropout key
    u = co.counter_uniform(1, 2, [3, 4, 1 << 40])
    assert np.all((u >= 0) & (u < 1))
    assert len(set(u.tolist())) == 3


@needs_ref
def test_prng_matches_reference():
    rng = np.random.default_rng(0)
    for _ in range(200):
        s, k, i = (int(x) for x in rng.integers(0, 2**63, 3, dtype=np.int64))
        assert float(co.counter_uniform(s, k, [i])[0]) == ref.counter_uniform(s, k, i)


def test_dropout_rate_statistics():
    # Dropout.RateAndScaling (test_expr.cpp:23-30)
    keep = co.dropout_keep(5, 11, np.arange(20000), 0.25)
    assert abs(keep.mean() - 0.75) < 0.02
    # the integer threshold form is exact
    for rate in (0.1, 0.25, 0.5, 1e-9, 0.999):
        bits = co.prng_bits(5, 11, np.arange(5000))
        assert np.array_equal(bits >= np.uint64(co.dropout_threshold(rate)),
                              co.counter_uniform(5, 11, np.arange(5000)) >= rate)


@pytest.mark.parametrize("rec", cases("adam"), ids=lambda r: r["name"])
def test_restated_fused_adam_reproduces_reference_engine_digest(rec):
    """The numpy restatement of FusedAllReduce(Adam) is bit-exact with the
    reference Engine on the scheduled program (golden digest)."""
    W, N = rec["dims"]["W"], rec["dims"]["N"]
    g = np.stack([co.gen_decl(1, "g", [N], "local", r, W) for r in range(W)])
    p, m, v = (co.gen_decl(1, n, [N], "replicated", 0, W) for n in "pmv")
    sc = {n: float(co.gen_decl(1, n, [], "replicated", 0, W)[0]) for n in ("lr", "beta1", "beta2", "t")}
    mo, vo, po = co.fused_adam([g], [m], [v], [p], co.adam_consts(**sc))
    res = {"out0": [po[0]], "tensor:m": [mo[0]], "tensor:p": [po[0]], "tensor:v": [vo[0]]}
    assert "%016x" % co.digest_results(res) == rec["engine_sched_digest"]
    assert rec["report_sched"]["comm_bytes"] == [2 * (W - 1) * (N // W) * 4] * W
    assert rec["report_sched"]["kernel_steps"] == 1
    assert rec["report_sched"]["memory_elems"]["m"] == N // W


def test_adam_kat_restated():
    """AdamScalarChainFrozenValues (test_oracle.cpp:24-48) via the restatement."""
    kat = json.loads((GOLD / "adam_kat.json").read_text())
    k = co.adam_consts(0.01, 0.9, 0.999, 1.0)
    g = co.ring_reduce(np.ones((4, 4), np.float32), 0)
    assert g.tolist() == [4.0] * 4
    mo, vo, po = co.adam_exact(g, np.zeros(4), np.zeros(4), np.ones(4), k)
    assert po.tolist() == kat["engine_sched"]["tensor:p"]
    assert mo.tolist() == kat["engine_sched"]["tensor:m"]
    assert vo.tolist() == kat["engine_sched"]["tensor:v"]
    assert abs(kat["oracle"]["v1"] - 1600.0) < 0.05


@needs_ref
@pytest.mark.parametrize("name", ["adam_W4_N1024", "adam_W8_N4096"])
def test_gen_decl_matches_reference(name):
    """gen_decl_values (state.hpp:55-74): Local decls keyed per rank."""
    rec = [c for c in cases("adam") if c["name"] == name][0]
    W, N = rec["dims"]["W"], rec["dims"]["N"]
    s = ref.RefSession(json.dumps(rec["base_program"]), None, {})
    s.gen(7)
    for r in range(W):
        assert np.array_equal(s.get_input("g", r, N), co.gen_decl(7, "g", [N], "local", r, W))
    assert np.array_equal(s.get_input("p", 0, N), co.gen_decl(7, "p", [N], "replicated", 0, W))
    assert np.array_equal(s.get_input("lr", 0, 1), co.gen_decl(7, "lr", [], "replicated", 0, W))


@needs_ref
def test_gen_decl_sliced_matches_reference():
    rec = cases("mp")[2]  # W=4, in: Sliced(2) [B,S,H]
    W = rec["dims"]["W"]
    s = ref.RefSession(json.dumps(rec["sched_program"]), None, {})
    s.gen(5)
    shape = [rec["dims"]["B"], rec["dims"]["S"], rec["dims"]["H"]]
    n = int(np.prod(shape))
    for r in range(W):
        full = s.get_input("in", r, n)
        gi = co.slice_global_index(shape, 2, W, r)
        assert np.array_equal(full[gi], co.gen_decl(5, "in", shape, "sliced", r, W, sliced_dim=2))


def test_sliced_index_map():
    # DistView::to_global for Sliced(2) (view.hpp:62-70): rank c owns column block c
    gi = co.slice_global_index([2, 3, 8], 2, 4, 1)
    assert gi.tolist()[:4] == [2, 3, 10, 11]
    with pytest.raises(ValueError):
        co.slice_global_index([6], 0, 4, 0)


@needs_ref
def test_bucket_table_matches_reference():
    rng = np.random.default_rng(2)
    for _ in range(20):
        counts = [int(x) for x in rng.integers(1, 5000, rng.integers(1, 12))]
        mine = [(t, o, e) for t, o, e, _ in co.bucket_table(counts)]
        assert mine == ref.bucket_table(counts)
        assert ref.bucket_metadata_bytes(counts) == 12 * ((sum(counts) + 1023) // 1024)


def test_bucket_metadata_overhead_formula():
    # acceptance criterion 4 (acceptance.cpp:203-208): ~0.59% at 334M f16
    N = 334_000_000
    over = 12 * -(-N // 1024) / (2 * N)
    assert 0.0058 < over < 0.0060


@needs_ref
def test_scattered_equals_contiguous_exactly():
    """Scattered.EqualsContiguousExactly (test_runtime.cpp:199-238): the
    restated ring AllReduce on the bucket-order flattening equals the
    reference's scattered_collective bit for bit."""
    rng = np.random.default_rng(17)
    for _ in range(10):
        W = int(rng.choice([2, 4, 8]))
        counts = [int(x) for x in rng.integers(1, 3000, rng.integers(1, 8))]
        if sum(counts) < W:
            continue
        ts = [rng.uniform(-1, 1, (W, n)).astype(np.float32) for n in counts]
        want = ref.scattered_allreduce(ts)
        table = co.bucket_table(counts)
        flat = co.flatten_bucket_order(ts, table)
        bounds = co.flat_chunks(flat.shape[1], W)
        owner = np.searchsorted(np.asarray(bounds[1:]), np.arange(flat.shape[1]), side="right")
        got = co.unflatten_bucket_order(co.ring_reduce(flat, owner), counts, table)
        for t in range(len(counts)):
            for r in range(W):
                assert np.array_equal(got[t], want[t][r])


@needs_ref
@pytest.mark.parametrize("W,N", [(1, 1024), (2, 2048), (4, 4096)])
def test_lamb_programs_and_restated_oracle(W, N):
    """The authored LAMB programs (reference JSON format) evaluate in the
    reference; the fused program matches the oracle on the base within 1e-5;
    the restated co.lamb_oracle matches the reference oracle within 1e-6."""
    base = (GOLD / "lamb_program.json").read_text()
    fused = (GOLD / "lamb_fused_program.json").read_text()
    s = ref.RefSession(base, None, {"N": N, "W": W}, sched_program=fused)
    s.gen(3)
    s.run(3, ref.ORACLE)
    s.run(3, ref.ENGINE_SCHED)
    assert s.compare(ref.ORACLE, ref.ENGINE_SCHED) <= 1e-5
    gl = np.stack([s.get_input("g", r, N) for r in range(W)])
    sc = {n: float(s.get_input(n, 0, 1)[0]) for n in ("lr", "beta1", "beta2", "t", "eps", "wd")}
    k = co.lamb_consts(sc["lr"], sc["beta1"], sc["beta2"], sc["t"], sc["eps"], sc["wd"])
    avg = co.rank_order_reduce(gl)
    mo, vo, po = co.lamb_oracle(avg, s.get_input("m", 0, N), s.get_input("v", 0, N),
                                s.get_input("p", 0, N), k)
    res = s.results(ref.ORACLE)
    assert co.max_rel_deviation(res["tensor:p"][0], po) <= 1e-6
    assert co.max_rel_deviation(res["tensor:m"][0], mo) <= 1e-6


@pytest.mark.parametrize("rec", cases("pp"), ids=lambda r: r["name"])
def test_pipeline_golden_counters(rec):
    """Pipeline.IntergroupBytesPerRank (test_runtime.cpp:240-252): N*bw per
    sender before the schedule, N/(W/2)*bw after."""
    W, N = rec["dims"]["W"], rec["dims"]["N"]
    half = W // 2
    assert rec["report_base"]["intergroup_bytes"][:half] == [N * 4] * half
    assert rec["report_sched"]["intergroup_bytes"][:half] == [N // half * 4] * half
    assert rec["deviation_sched_vs_oracle"] <= 1e-5


def test_digest_is_fnv_over_sorted_keys():
    res = {"b": [np.array([1.0], np.float32)], "a": [np.array([2.0, 3.0], np.float32)]}
    h = co.FNV_OFFSET
    for k in ("a", "b"):
        h = co.fnv1a(k, h)
        h = co.fnv1a(res[k][0].tobytes(), h)
    assert co.digest_results(res) == h


# ---- per-tensor LAMB over a tensor list (oracle/make_lamb_golden.py) -------

def _lamb_list_cases():
    return json.loads((GOLD / "lamb_list_cases.json").read_text())


@pytest.mark.parametrize("rec", _lamb_list_cases(), ids=lambda r: r["name"])
def test_lamb_list_restated_equals_reference_engine(rec):
    """The restated LAMB (co.lamb_oracle per tensor, on each tensor's own
    ring-order RS) reproduces the reference Engine's per-tensor fused LAMB
    programs bit for bit on every tensor of the list (p, m, v), W = 1..8; the
    Engine itself is within 1e-6 of the reference oracle on the base program."""
    from oracle.make_lamb_golden import restated
    arrs = np.load(GOLD / "lamb_list_results.npz")
    W = rec["W"]
    assert rec["deviation_sched_vs_oracle"] <= 1e-6
    rest = restated(rec["counts"], W, rec["seed"])
    for i in range(len(rec["counts"])):
        for name, j in (("p", 0), ("m", 1), ("v", 2)):
            assert np.array_equal(rest[i][j], arrs[f"W{W}_{name}{i}"]), (name, i)


@needs_ref
def test_lamb_list_golden_regenerates():
    """The committed per-tensor LAMB fixture is what the reference computes."""
    from oracle.make_lamb_golden import COUNTS, base_program, fused_program
    rec = next(r for r in _lamb_list_cases() if r["W"] == 4)
    s = ref.RefSession(base_program(COUNTS), None, {"W": 4}, sched_program=fused_program(COUNTS))
    s.gen(1)
    s.run(1, ref.ENGINE_SCHED)
    assert "%016x" % s.digest(ref.ENGINE_SCHED) == rec["engine_sched_digest"]
