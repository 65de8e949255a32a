"""Query parity: the fixed-plan executor (sx_tpch_q*, through the C ABI) vs the CPU oracle on the
same seeded TPC-H-shaped data.  Integer/decimal outputs bit-exact, avg within 1e-9 relative
(north_star).  Small SF: oracle computed live; larger SF: oracle answers committed under
tests/golden/ by oracle/make_answers.py.
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle
from tests.helpers import GOLDEN, diff_rows, golden_tables, load_golden, rows_equal

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2508_04701_b200 as sx  # noqa: E402
from paper_2508_04701_b200 import tpch  # noqa: E402

QUERIES = ["q1", "q6", "q3", "q9", "q18"]


@pytest.fixture(scope="module")
def ctx():
    return sx.Ctx(0)


def to_dev(t):
    return {tn: {cn: torch.from_numpy(np.ascontiguousarray(a)).cuda() for cn, a in cols.items()}
            for tn, cols in t.items()}


@pytest.mark.parametrize("name", ["q1", "q6", "q6_empty", "q3", "q9", "q18"])
def test_hand_tables(ctx, name):
    case = load_golden("hand_queries.json")[name]
    q = name.split("_")[0]
    host = golden_tables(case["tables"], key_dtype=np.int32)
    got = tpch.Tpch(ctx, to_dev(host)).run(q)
    want = [tuple(r) for r in case["answer"]]
    assert rows_equal(got, want), diff_rows(got, want)


@pytest.fixture(scope="module", params=[10, 100])
def small(request, ctx):
    host = gen.cpu_tables(request.param, seed=42)
    return request.param, host, tpch.Tpch(ctx, to_dev(host))


@pytest.mark.parametrize("q", QUERIES)
def test_query_vs_live_oracle(small, q):
    sfm, host, T = small
    want = oracle.run_query(q, host)
    got = T.run(q)
    assert rows_equal(got, want), diff_rows(got, want)


def test_query_params_vs_oracle(small):
    sfm, host, T = small
    for over in (dict(q18_qty_gt=25000), dict(q18_qty_gt=20000)):
        got = T.run("q18", tpch.default_params(**over))
        want = oracle.run_query("q18", host, oracle.default_params(**over))
        assert rows_equal(got, want), diff_rows(got, want)
    got = T.run("q3", tpch.default_params(q3_limit=500, q3_date=9500, q3_segment=3))
    want = oracle.run_query("q3", host, oracle.default_params(q3_date=9500, q3_segment=3), limit=500)
    assert rows_equal(got, want), diff_rows(got, want)
    got = T.run("q9", tpch.default_params(q9_color="blue"))
    want = oracle.run_query("q9", host, oracle.default_params(q9_color="blue"))
    assert rows_equal(got, want), diff_rows(got, want)


@pytest.mark.parametrize("mode", ["0", "2"])
def test_q18_group_strategies(small, monkeypatch, mode):
    """Q18's subquery group-by through the hash table (SX_GB_SORTED=0) and through the
    sorted-run strategy forced at any table size (=2; by default it engages only when the
    hash table would exceed half the L2, i.e. at the bench scale)."""
    sfm, host, T = small
    monkeypatch.setenv("SX_GB_SORTED", mode)
    for over in ({}, dict(q18_qty_gt=20000)):
        got = T.run("q18", tpch.default_params(**over))
        want = oracle.run_query("q18", host, oracle.default_params(**over))
        assert rows_equal(got, want), diff_rows(got, want)


@pytest.mark.parametrize("case", ["tails", "run20", "run60", "run200", "big", "unsorted", "lean-off"])
def test_q18_owned_runs(ctx, monkeypatch, case):
    """Q18's owned-run aggregation (K10l lean kernel, else K10r; forced with SX_GB_SORTED=2 at SF 0.1):
    a ragged tail, runs of 20 / 60 rows crossing lanes and warps (lead hand-off, scalar
    continuation), a 200-row run (past kRunAhead: K10r, then hashing), a quantity >= 2^40 (K10l
    refuses: K10r), an unsorted key column (hashing), and SX_RUNS_LEAN=0 (K10r) on the same data."""
    monkeypatch.setenv("SX_GB_SORTED", "2")
    if case == "lean-off":
        monkeypatch.setenv("SX_RUNS_LEAN", "0")
    host = gen.cpu_tables(100, seed=13)
    li = {k: v.copy() for k, v in host["lineitem"].items()}
    n = len(li["l_orderkey"]) - (1111 if case == "tails" else 0)
    li = {k: v[:n].copy() for k, v in li.items()}
    ok = li["l_orderkey"]
    if case in ("run20", "run60", "run200"):
        L = {"run20": 20, "run60": 60, "run200": 200}[case]
        for start in (4096 * 7 + 100, 2048 * 40 - 30, 256 * 100 - 3, n - L):  # inside, across tiles/warps, at the end
            ok[start:start + L] = ok[start]
    if case == "big":
        li["l_quantity"][[5, 70_000, n - 1]] = 1 << 41
    if case == "unsorted":
        ok[[1000, 1001]] = ok[[1001, 1000]] if ok[1000] != ok[1001] else (ok[1000], ok[1000] - 1)
        ok[300_000], ok[300_001] = ok[300_001], ok[300_000]
    host = dict(host)
    host["lineitem"] = li
    T = tpch.Tpch(ctx, to_dev(host))
    for over in ({}, dict(q18_qty_gt=15000)):
        got = T.run("q18", tpch.default_params(**over))
        want = oracle.run_query("q18", host, oracle.default_params(**over))
        assert rows_equal(got, want), diff_rows(got, want)



@pytest.mark.parametrize("case", ["fused", "ops", "tails", "run30", "unsorted", "wide"])
def test_q3_plans(ctx, monkeypatch, case):
    """Q3 through the fused lineitem pass (K10q, the default: warp-range owned orderkey groups,
    interpolated carries) and the operator-at-a-time plan (SX_Q3_PLAN=ops), at SF 0.1: a ragged
    tail, 30-row orderkey runs crossing warp ranges, an unsorted l_orderkey (the fused pass steps
    aside), and an extendedprice of 2^40 (revenue terms beyond 32 bits) — against the oracle."""
    monkeypatch.setenv("SX_Q3_PLAN", "ops" if case == "ops" else "fused")
    host = gen.cpu_tables(100, seed=17)
    li = {k: v.copy() for k, v in host["lineitem"].items()}
    n = len(li["l_orderkey"]) - (777 if case == "tails" else 0)
    li = {k: v[:n].copy() for k, v in li.items()}
    ok = li["l_orderkey"]
    if case == "run30":
        for start in (4096 * 5 + 11, 256 * 77 - 5, n - 30):
            ok[start:start + 30] = ok[start]
            li["l_shipdate"][start:start + 30] = 9300  # after the Q3 date: every row of the run joins if its order does
    if case == "unsorted":
        ok[[2000, 2001]] = ok[[2001, 2000]] if ok[2000] != ok[2001] else (ok[2000], ok[2000] - 1)
    if case == "wide":
        li["l_extendedprice"][[3, n // 2]] = 1 << 40
    host = dict(host)
    host["lineitem"] = li
    T = tpch.Tpch(ctx, to_dev(host))
    for lim in (10, 1000):
        got = T.run("q3", tpch.default_params(q3_limit=lim))
        want = oracle.run_query("q3", host, limit=lim)
        assert rows_equal(got, want), diff_rows(got, want)



def test_orders_not_in_key_order(ctx, monkeypatch):
    """Orders rows shuffled: Q9's single-pass date fill detects keys that are not strictly
    increasing and reruns the scatter fill; Q3 and Q18 do not depend on the orders' row order."""
    host = gen.cpu_tables(100, seed=19)
    o = host["orders"]
    perm = np.random.default_rng(4).permutation(len(o["o_orderkey"]))
    host = dict(host)
    host["orders"] = {k: v[perm].copy() for k, v in o.items()}
    T = tpch.Tpch(ctx, to_dev(host))
    for q in ("q9", "q3", "q18", "q3-fused"):
        if q == "q3-fused":  # the fused plan's binary-search carries find no order: operator steps
            monkeypatch.setenv("SX_Q3_PLAN", "fused")
        got = T.run(q[:2])
        want = oracle.run_query(q[:2], host)
        assert rows_equal(got, want), f"{q}: " + diff_rows(got, want)



@pytest.mark.parametrize("lazy3", ["0", "1"])
def test_q6_lazy_levels(ctx, monkeypatch, lazy3):
    """Q6's dense program with two lazy levels (shipdate, then discount/quantity/price) and three
    (SX_Q6_LAZY3=1: discount gates quantity/price), with boundary values of every predicate."""
    monkeypatch.setenv("SX_Q6_LAZY3", lazy3)
    host = gen.cpu_tables(100, seed=23)
    li = {k: v.copy() for k, v in host["lineitem"].items()}
    n = len(li["l_shipdate"]) - 5
    li = {k: v[:n].copy() for k, v in li.items()}
    rng = np.random.default_rng(2)
    for col, vals in (("l_shipdate", [8765, 8766, 9130, 9131]), ("l_discount", [4, 5, 7, 8]), ("l_quantity", [2399, 2400])):
        li[col][rng.choice(n, 2000, replace=False)] = rng.choice(vals, 2000)
    host = dict(host)
    host["lineitem"] = li
    got = tpch.Tpch(ctx, to_dev(host)).run("q6")
    want = oracle.run_query("q6", host)
    assert rows_equal(got, want), diff_rows(got, want)



@pytest.mark.parametrize("case", ["sorted", "lookup", "hash", "customer-shuffled", "customer-missing"])
def test_q18_join_modes(ctx, monkeypatch, case):
    """Q18's orders/customer joins by the fused sorted-PK lookup kernel (default), by separate
    lookups + gathers (SX_Q18_JOIN=lookup), by hash joins (SX_Q18_JOIN=hash), with the customer
    rows shuffled (lookups fail: hash joins), and with qualifying orders whose customer is missing
    (inner-join semantics: those orders drop out)."""
    if case in ("hash", "lookup"):
        monkeypatch.setenv("SX_Q18_JOIN", case)
    host = gen.cpu_tables(100, seed=29)
    host = dict(host)
    c = host["customer"]
    if case == "customer-shuffled":
        perm = np.random.default_rng(6).permutation(len(c["c_custkey"]))
        host["customer"] = {k: v[perm].copy() for k, v in c.items()}
    if case == "customer-missing":
        keep = np.ones(len(c["c_custkey"]), bool)
        keep[::3] = False
        host["customer"] = {k: v[keep].copy() for k, v in c.items()}
    T = tpch.Tpch(ctx, to_dev(host))
    for over in ({}, dict(q18_qty_gt=15000)):
        got = T.run("q18", tpch.default_params(**over))
        want = oracle.run_query("q18", host, oracle.default_params(**over))
        assert rows_equal(got, want), diff_rows(got, want)



@pytest.mark.parametrize("ring", ["1", "0"])
@pytest.mark.parametrize("trim", [0, 777])
def test_q9_ring(ctx, monkeypatch, ring, trim):
    """Q9's lineitem pass fed by the tile ring (K10wr, SX_Q9_RING=1, >= 1024 rows per SM) and by
    per-lane loads (K10w, the default), with whole tiles only and with a ragged tail (global-load
    path in the last CTA) — against the oracle, also for another colour."""
    monkeypatch.setenv("SX_Q9_RING", ring)  # (K10wr is opt-in: measured slower than K10w)
    host = gen.cpu_tables(200, seed=31)
    li = host["lineitem"]
    n = len(li["l_orderkey"])
    n = n - n % 1024 - trim if trim == 0 else n - trim
    host = dict(host)
    host["lineitem"] = {k: v[:n].copy() for k, v in li.items()}
    T = tpch.Tpch(ctx, to_dev(host))
    for color in ("green", "blue"):
        got = T.run("q9", tpch.default_params(q9_color=color))
        want = oracle.run_query("q9", host, oracle.default_params(q9_color=color))
        assert rows_equal(got, want), diff_rows(got, want)



def test_q9_repeated_partsupp_pair_fails(ctx):
    """A repeated (ps_partkey, ps_suppkey) pair — the fused plan relies on it being a key — fails
    loudly (DESIGN §3 reading) instead of picking one cost."""
    host = dict(gen.cpu_tables(200, seed=37))
    ps = {k: v.copy() for k, v in host["partsupp"].items()}
    ps["ps_suppkey"][1::4] = ps["ps_suppkey"][0::4]
    host["partsupp"] = ps
    with pytest.raises(Exception, match="repeated"):
        tpch.Tpch(ctx, to_dev(host)).run("q9")



def test_gpu_generator_matches_cpu_generator():
    cpu = gen.cpu_tables(10, seed=42)
    g = gen.gpu_tables(10, seed=42)
    for t in cpu:
        for cname in cpu[t]:
            assert np.array_equal(g[t][cname].cpu().numpy(), cpu[t][cname]), (t, cname)


@pytest.mark.parametrize("sfm", [1000, 10000])
def test_query_vs_committed_answers(ctx, sfm):
    path = os.path.join(GOLDEN, f"answers_sf{sfm}_seed42.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    ans = json.load(open(path))
    T = tpch.Tpch(ctx, gen.gpu_tables(sfm, seed=42))
    for q in QUERIES:
        if q not in ans["answers"]:
            continue
        want = [tuple(r) for r in ans["answers"][q]]
        if q == "q9":
            want = [(oracle.NATIONS[r[0]], r[1], r[2]) for r in want]
        if q == "q18":
            want = [(oracle.c_name(r[0]),) + tuple(r) for r in want]
        got = T.run(q)
        assert rows_equal(got, want), f"{q}: " + diff_rows(got, want)


@pytest.mark.parametrize("trunc", [0, 3, 5])
def test_q1_q6_dense_guard_and_tails(ctx, trunc):
    """The dense small-G kernel (k_gb_dense) vs the oracle where its fast-path guard fails
    (ext >= 2^26, negative discount, tax >= 2^7: exact slow path), where a 5th/6th group key
    appears (more keys than register slots: global path), and for row counts that are not a
    multiple of the 4/8-row vector groups (scalar tail)."""
    host = gen.cpu_tables(10, seed=7)
    li = {k: v.copy() for k, v in host["lineitem"].items()}
    n = len(li["l_shipdate"]) - trunc
    li = {k: v[:n].copy() for k, v in li.items()}
    rng = np.random.default_rng(3)
    for col, val in (("l_extendedprice", 1 << 40), ("l_discount", -5), ("l_tax", 200), ("l_quantity", 1 << 30)):
        idx = rng.choice(n, 7, replace=False)
        li[col][idx] = val
    li["l_returnflag"][rng.choice(n, 5, replace=False)] = ord("Z")
    li["l_linestatus"][rng.choice(n, 5, replace=False)] = ord("Q")
    # Q6 rows that pass the date/discount/quantity ranges but carry a huge extendedprice
    ok = np.nonzero((li["l_shipdate"] >= 8766) & (li["l_shipdate"] < 9131) & (li["l_discount"] >= 5) &
                    (li["l_discount"] <= 7) & (li["l_quantity"] < 2400))[0]
    li["l_extendedprice"][ok[:3]] = (1 << 27) + 11
    host = dict(host)
    host["lineitem"] = li
    T = tpch.Tpch(ctx, to_dev(host))
    for q in ("q1", "q6"):
        want = oracle.run_query(q, host)
        got = T.run(q)
        assert rows_equal(got, want), f"{q}: " + diff_rows(got, want)


@pytest.mark.parametrize("case", ["tails", "guard", "overflow", "ring-off"])
def test_q1_ring(ctx, monkeypatch, case):
    """Q1 through K9r (producer warp + cp.async.bulk tile ring, >= 1024 rows per SM: SF 0.1): a
    ragged last tile (global-load tail), rows failing the register fast path (exact per-CTA slow
    list), a slow list that overflows (the host reruns K9d), and SX_RING=0 (K9d) on the same data."""
    host = gen.cpu_tables(100, seed=11)
    li = {k: v.copy() for k, v in host["lineitem"].items()}
    n = len(li["l_shipdate"]) - (777 if case == "tails" else 0)
    li = {k: v[:n].copy() for k, v in li.items()}
    rng = np.random.default_rng(5)
    if case == "guard":
        for col, val in (("l_extendedprice", 1 << 40), ("l_discount", -5), ("l_tax", 17), ("l_quantity", 8192),
                         ("l_discount", 16), ("l_extendedprice", 1 << 24)):
            li[col][rng.choice(n, 9, replace=False)] = val
        li["l_returnflag"][rng.choice(n, 9, replace=False)] = ord("Z")
        li["l_linestatus"][rng.choice(n, 9, replace=False)] = ord("Q")
    if case == "overflow":
        li["l_returnflag"][rng.choice(n, n // 3, replace=False)] = ord("B")
    if case == "ring-off":
        monkeypatch.setenv("SX_RING", "0")
    host = dict(host)
    host["lineitem"] = li
    want = oracle.run_query("q1", host)
    got = tpch.Tpch(ctx, to_dev(host)).run("q1")
    assert rows_equal(got, want), diff_rows(got, want)


@pytest.mark.parametrize("plan", ["fused", "fused-mat", "fused-dense", "fused-wscan", "fused-wscan-partitioned",
                                  "fused-partitioned", "ops"])
def test_q9_plans(small, monkeypatch, plan):
    """Q9 through the fused probe-chain group-by (default: gathering the semi-join's rows; or a dense
    scan; or with radix-partitioned PK tables) and the operator-at-a-time plan."""
    sfm, host, T = small
    if plan == "ops":
        monkeypatch.setenv("SX_Q9_PLAN", "ops")
    else:
        monkeypatch.setenv("SX_Q9_PLAN", "fused")
        monkeypatch.setenv("SX_Q9_SCAN", {"fused-dense": "dense", "fused-mat": "mat", "fused-wscan": "wscan",
                                          "fused-wscan-partitioned": "wscan"}.get(plan, "gather"))
        # PK payload tables built radix-partitioned region by region (forced at any size)
        monkeypatch.setenv("SX_PT_PARTITION", "2" if plan.endswith("partitioned") else "1")
    for over in ({}, dict(q9_color="blue")):
        got = T.run("q9", tpch.default_params(**over))
        want = oracle.run_query("q9", host, oracle.default_params(**over))
        assert rows_equal(got, want), diff_rows(got, want)


def test_q1_bulk_staged(ctx, monkeypatch):
    """Q1 through the bulk-staged (cp.async.bulk + mbarrier) dense aggregation, SX_BULK=1: needs
    >= 1024 rows per SM, so SF 0.1 (~600k rows, a ragged last tile)."""
    monkeypatch.setenv("SX_BULK", "1")
    host = gen.cpu_tables(100, seed=5)
    T = tpch.Tpch(ctx, to_dev(host))
    for q in ("q1", "q6"):
        want = oracle.run_query(q, host)
        got = T.run(q)
        assert rows_equal(got, want), f"{q}: " + diff_rows(got, want)


def test_q9_q3_wide_orderkeys(ctx):
    """int64 orderkeys spread over more than 2^30 (no exact bitmaps: Q9's fused plan falls back to the
    operator-at-a-time plan, Q3's orders build keeps its hash table) still match the oracle."""
    host = gen.cpu_tables(10, seed=3)
    host = {t: dict(c) for t, c in host.items()}
    for t, col in (("orders", "o_orderkey"), ("lineitem", "l_orderkey")):
        host[t][col] = host[t][col].astype(np.int64) * (1 << 24) + 5
    T = tpch.Tpch(ctx, to_dev(host))
    for q in ("q9", "q3", "q18"):
        want = oracle.run_query(q, host)
        got = T.run(q)
        assert rows_equal(got, want), f"{q}: " + diff_rows(got, want)


@pytest.mark.parametrize("empty", ["lineitem", "orders_lineitem", "part", "customer"])
def test_queries_on_empty_tables(ctx, empty):
    """Degenerate inputs: empty lineitem (and orders), no part, no customer — every plan returns
    what the oracle returns (empty results, a NULL Q6, no groups)."""
    host = gen.cpu_tables(10, seed=9)
    host = {t: {c: a.copy() for c, a in cols.items()} for t, cols in host.items()}

    def clear(t):
        for c in list(host[t]):
            if c == "p_name_offsets":
                host[t][c] = host[t][c][:1].copy()
                host[t][c][:] = 0
            elif c == "p_name_chars":
                host[t][c] = host[t][c][:0]
            else:
                host[t][c] = host[t][c][:0]

    for t in {"lineitem": ["lineitem"], "orders_lineitem": ["orders", "lineitem"], "part": ["part"],
              "customer": ["customer"]}[empty]:
        clear(t)
    T = tpch.Tpch(ctx, to_dev(host))
    for q in QUERIES:
        want = oracle.run_query(q, host)
        got = T.run(q)
        assert rows_equal(got, want), f"{q}: " + diff_rows(got, want)


def test_upload_from_host_tables(ctx):
    """sx_tpch_upload: tables in (pinned) host memory copied by the library, then the five plans."""
    host = gen.cpu_tables(10, seed=4)
    pinned = {t: {c: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for c, a in cols.items()}
              for t, cols in host.items()}
    T = tpch.Tpch.upload(ctx, pinned)
    try:
        for q in QUERIES:
            want = oracle.run_query(q, host)
            got = T.run(q)
            assert rows_equal(got, want), f"{q}: " + diff_rows(got, want)
    finally:
        T.free()


@pytest.mark.parametrize("scan", ["wscan", "gather"])
def test_q9_wide_orderdates_fall_back(ctx, monkeypatch, scan):
    """The fused Q9 keeps year(o_orderdate) as one byte (1900..2027): an order dated outside that
    range (here 2100 and 1850, then 2030 just past the byte's range) makes it step aside to the
    operator-at-a-time plan, still exact; 1901 and 2027 stay inside."""
    monkeypatch.setenv("SX_Q9_SCAN", scan)
    host = gen.cpu_tables(10, seed=5)
    od = host["orders"]["o_orderdate"].copy()
    od[::97] += 47000   # ~2100
    od[1::97] -= 44000  # ~1850
    host["orders"]["o_orderdate"] = od
    T = tpch.Tpch(ctx, to_dev(host))
    want = oracle.run_query("q9", host)
    got = T.run("q9")
    assert rows_equal(got, want), diff_rows(got, want)
    od = gen.cpu_tables(10, seed=5)["orders"]["o_orderdate"].copy()
    od[::53] = 22066   # 2030-06-01
    host["orders"]["o_orderdate"] = od
    T = tpch.Tpch(ctx, to_dev(host))
    assert rows_equal(T.run("q9"), oracle.run_query("q9", host))
    od[::53] = -25000  # 1901-07-28
    od[1::53] = 20800  # 2026-12-13
    host["orders"]["o_orderdate"] = od
    T = tpch.Tpch(ctx, to_dev(host))
    want = oracle.run_query("q9", host)
    got = T.run("q9")
    assert rows_equal(got, want), diff_rows(got, want)


@pytest.mark.parametrize("nl", [1, 7, 511, 512, 513, 1025, 4099])
def test_q9_wscan_window_edges(ctx, monkeypatch, nl):
    """K10w (the default Q9 lineitem pass) on lineitem prefixes around its 512-row warp window and
    the 8-row lane chunk: a single row, a partial chunk, one window +- 1, several windows + tail.
    SF 0.01 tables (at SF 0.001 the generator's partsupp (partkey, suppkey) pairs can repeat,
    SURVEY App. A, and the PK payload table refuses them)."""
    monkeypatch.setenv("SX_Q9_SCAN", "wscan")
    host = gen.cpu_tables(10, seed=3)
    host["lineitem"] = {c: np.ascontiguousarray(a[:nl]) for c, a in host["lineitem"].items()}
    T = tpch.Tpch(ctx, to_dev(host))
    for over in ({}, dict(q9_color="blue")):
        want = oracle.run_query("q9", host, oracle.default_params(**over))
        got = T.run("q9", tpch.default_params(**over))
        assert rows_equal(got, want), diff_rows(got, want)
