"""Operator parity: libsx CUDA kernels (through the C ABI) vs the CPU oracle, element by element.

Sizes span several tiles (2048 rows per compaction tile) with ragged tails; edge cases:
empty input, all/none selected, duplicate keys, negative and extreme keys, key 0 (the
aggregation table's EMPTY value), one group, every row its own group.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2508_04701_b200 as sx  # noqa: E402
from paper_2508_04701_b200 import _abi as A  # noqa: E402

SIZES = [0, 1, 2047, 2048, 2049, 100_003]


@pytest.fixture(scope="module")
def ctx():
    return sx.Ctx(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def c(t, typ=None):
    return sx.col(t, typ)


def i128_rows(t):
    a = t.cpu().numpy()
    return [(int(lo) & ((1 << 64) - 1)) | (int(hi) << 64) for lo, hi in a]


# ------------------------------------------------------------------------------------- filter
@pytest.mark.parametrize("n", SIZES)
def test_filter_conjunction(ctx, n):
    rng = np.random.default_rng(n + 1)
    a = rng.integers(-100, 100, n).astype(np.int32)
    b = rng.integers(0, 256, n).astype(np.uint8)
    d = rng.integers(-(2**62), 2**62, n).astype(np.int64)
    ta, tb, td = dev(a), dev(b), dev(d)
    cols = [c(ta), c(tb), c(td)]
    for conj in ([(0, "ge", -10), (1, "ne", 7), (2, "gt", 0)], [(0, "between", -5, 5)], [(1, "eq", 3)],
                 [(2, "le", -(2**61)), (0, "lt", 50)], []):
        sel, gathered = ctx.filter(cols, conj, gather=[0, 2])
        want = oracle.filter([a, b, d], conj) if conj else np.arange(n, dtype=np.int32)
        assert np.array_equal(sel.cpu().numpy(), want)
        assert np.array_equal(gathered[0].cpu().numpy(), a[want])
        assert np.array_equal(gathered[1].cpu().numpy(), d[want])


def test_filter_in_sel(ctx):
    rng = np.random.default_rng(5)
    n = 50_000
    a = rng.integers(0, 1000, n).astype(np.int64)
    base = np.sort(rng.choice(n, 20_000, replace=False)).astype(np.int32)
    sel, _ = ctx.filter([c(dev(a))], [(0, "lt", 300)], in_sel=dev(base))
    assert np.array_equal(sel.cpu().numpy(), base[a[base] < 300])


@pytest.mark.parametrize("pattern", [b"green", b"g", b"zz", b"een ap"])
def test_filter_contains(ctx, pattern):
    import gen

    p = gen.cpu_tables(20, seed=3, tables=("part",))["part"]
    offs, chars = p["p_name_offsets"], p["p_name_chars"]
    sel, _ = ctx.filter([sx.col(dev(chars), A.SX_STR, offsets=dev(offs))], [(0, "contains", pattern)])
    assert np.array_equal(sel.cpu().numpy(), oracle.contains(offs, chars, pattern))


# ------------------------------------------------------------------------------------- group-by
def canon(keys, aggs, ops):
    """GPU outputs -> rows sorted by key (canonical ORDER BY)."""
    cols = [k.cpu().numpy().astype(np.int64).tolist() for k in keys]
    vals = []
    for t, op in zip(aggs, ops):
        if op == "sum":
            vals.append(i128_rows(t))
        elif op == "avg":
            vals.append(t.cpu().numpy().tolist())
        else:
            vals.append(t.cpu().numpy().tolist())
    rows = list(zip(*cols, *vals)) if (cols or vals) else []
    return sorted(rows, key=lambda r: r[: len(keys)])


def check_gb(got, want):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        for x, y in zip(g, w):
            if isinstance(y, float):
                assert abs(x - y) <= 1e-9 * max(1.0, abs(y)), (g, w)
            else:
                assert x == y, (g, w)


AGGS = [("sum", [(1, [(2, 1, 0), (3, -1, 100)])]), ("count", []), ("min", [(1, [(2, 1, 0)])]),
        ("max", [(1, [(2, 1, 0)])]), ("avg", [(1, [(3, 1, 0)])], 2), ("sum", [(1, [(2, 1, 0)]), (-3, [(3, 1, 7)])])]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("ng,hint", [(3, 4), (4, 4), (300, 512), (175, 256), (3000, 100), (5000, 0), (None, 0)])
def test_groupby_one_key(ctx, n, ng, hint):
    rng = np.random.default_rng(n + (ng or 0))
    dom = ng if ng else max(n, 1)
    k = rng.integers(-(dom // 2), dom - dom // 2, n).astype(np.int32)  # includes key 0 (EMPTY) and negatives
    v = rng.integers(-(10**12), 10**12, n).astype(np.int64)
    w = rng.integers(0, 100, n).astype(np.int64)
    cols = [c(dev(k)), c(dev(k)), c(dev(v)), c(dev(w))]
    keys, aggs, g = ctx.groupby(cols, [(0, "id")], AGGS, groups_hint=hint)
    got = canon(keys, aggs, [a[0] for a in AGGS])
    want = oracle.groupby([k, k, v, w], [0], AGGS)
    check_gb(got, want)
    assert g == len(want)


SIMPLE_AGGS = [("sum", [(1, [(1, 1, 0)])]), ("count", []), ("min", [(1, [(1, 1, 0)])]), ("max", [(1, [(1, 1, 0)])]),
               ("avg", [(1, [(1, 1, 0)])], 2), ("max", [(1, [(2, 1, 0)])])]


@pytest.mark.parametrize("G,hint,wide", [(4, 4, False), (100, 128, False), (1000, 1024, True), (5000, 5000, False),
                                         (200_000, 200_000, False), (3000, 1500, False), (300, 0, False),
                                         (3_000_000, 3_000_000, False)])
def test_groupby_plain_shape(ctx, G, hint, wide):
    """K18 (the plain shape: one int64 key, plain-column aggregates; >= 2^20 rows): shared replicas
    (hint <= 1024), partitioned shared tables (hint > 1024; two partition levels above 2^21),
    an under-hinted G (falls back), the
    key INT64_MIN (the shared tables' EMPTY marker: side slot), values >= 2^40 (exact global
    path in K18s), an int32 value column — against the oracle."""
    rng = np.random.default_rng(G)
    n = (1 << 20) + 12_345
    keys = np.unique(rng.integers(-(2**63), 2**63 - 1, G * 2, dtype=np.int64))[:G]
    keys[0] = -(2**63)
    k = keys[rng.integers(0, G, n)]
    v = rng.integers(-(10**9), 10**9, n).astype(np.int64)
    if wide:
        v[rng.integers(0, n, 50)] = 2**61
    w = rng.integers(-(2**31), 2**31 - 1, n).astype(np.int32)
    cols = [sx.col(dev(k)), sx.col(dev(v), A.SX_DEC64, 2), sx.col(dev(w), A.SX_I32)]
    keys_o, aggs_o, g = ctx.groupby(cols, [(0, "id")], SIMPLE_AGGS, groups_hint=hint)
    got = canon(keys_o, aggs_o, [a[0] for a in SIMPLE_AGGS])
    want = oracle.groupby([k, v, w], [0], SIMPLE_AGGS)
    check_gb(got, want)
    assert g == len(want)


FIXED_AGGS = [("sum", [(1, [(1, 1, 0)])]), ("count", []), ("min", [(1, [(1, 1, 0)])]), ("max", [(1, [(1, 1, 0)])]),
              ("avg", [(1, [(1, 1, 0)])], 2)]


@pytest.mark.parametrize("G,hint,wide,v32", [(4, 4, False, False), (13, 16, True, False), (40, 16, False, False),
                                             (100, 128, False, True), (256, 256, True, False),
                                             (1000, 1024, False, False), (5000, 5000, False, False),
                                             (200_000, 200_000, False, False), (3000, 300, False, False),
                                             (262_144, 262_144, False, True), (6000, 6000, True, False),
                                             (100_000, 8192, False, False), (1_500_000, 2_000_000, False, False)])
def test_groupby_fixed_signature(ctx, G, hint, wide, v32):
    """The fixed signature (one value column: count + sum/min/max/avg, >= 2^20 rows): K19t
    lane-private cells (hint <= 48 direct, <= 16384 behind a radix partition), K18 above;
    under-hinted G (a warp dictionary or a hinted table overflows: K18 or the generic path takes
    over), the key INT64_MIN (side slot), values >= 2^40 (K19's exact global path), an int32 value
    column — against the oracle."""
    rng = np.random.default_rng(G + hint)
    n = (1 << 20) + 4_321
    keys = np.unique(rng.integers(-(2**63), 2**63 - 1, G * 2, dtype=np.int64))[:G]
    keys[0] = -(2**63)
    k = keys[rng.integers(0, G, n)]
    if v32:
        v = rng.integers(-(2**31), 2**31 - 1, n).astype(np.int32)
        vc = sx.col(dev(v), A.SX_I32)
    else:
        v = rng.integers(-(10**9), 10**9, n).astype(np.int64)
        if wide:
            v[rng.integers(0, n, 50)] = -(2**61)
        vc = sx.col(dev(v), A.SX_DEC64, 2)
    keys_o, aggs_o, g = ctx.groupby([sx.col(dev(k)), vc], [(0, "id")], FIXED_AGGS, groups_hint=hint)
    got = canon(keys_o, aggs_o, [a[0] for a in FIXED_AGGS])
    want = oracle.groupby([k, v], [0], FIXED_AGGS)
    check_gb(got, want)
    assert g == len(want)


@pytest.mark.parametrize("n,G,hint,keytype", [((1 << 20) + 1, 1, 1, np.int64), ((1 << 21) - 7, 3, 4, np.int32),
                                              ((1 << 20) + 255, 60, 48, np.int64), ((1 << 20) + 33, 2000, 2048, np.int32)])
def test_groupby_k19_edges(ctx, n, G, hint, keytype):
    """K19t edge cases: one group, a ragged tail (n not a multiple of the 256-row warp batch),
    int32 keys, more groups than a warp's 48 cells (rows of the groups past them take the exact
    global path), partitioned with int32 keys; values straddling 2^32 (the split sums)."""
    rng = np.random.default_rng(n + G)
    keys = np.unique(rng.integers(-(2**31), 2**31 - 1, G * 4))[:G].astype(keytype)
    k = keys[rng.integers(0, G, n)]
    v = rng.integers(-(2**39), 2**39, n).astype(np.int64)
    v[::7] = (2**32) - 1
    v[1::7] = -(2**32)
    kc = sx.col(dev(k), A.SX_I32 if keytype == np.int32 else A.SX_I64)
    keys_o, aggs_o, g = ctx.groupby([kc, sx.col(dev(v), A.SX_DEC64, 2)], [(0, "id")], FIXED_AGGS, groups_hint=hint)
    got = canon(keys_o, aggs_o, [a[0] for a in FIXED_AGGS])
    want = oracle.groupby([k.astype(np.int64), v], [0], FIXED_AGGS)
    check_gb(got, want)
    assert g == len(want)


@pytest.mark.parametrize("hint", [4, 64])
def test_groupby_two_u8_keys_where(ctx, hint):
    rng = np.random.default_rng(11)
    n = 70_001
    a = rng.choice(np.array([ord("A"), ord("N"), ord("R")], np.uint8), n)
    b = rng.choice(np.array([ord("F"), ord("O")], np.uint8), n)
    s = rng.integers(0, 100, n).astype(np.int32)
    v = rng.integers(0, 10**9, n).astype(np.int64)
    cols = [c(dev(a)), c(dev(b)), c(dev(s)), c(dev(v))]
    aggs = [("sum", [(1, [(3, 1, 0), (2, -1, 100)])]), ("avg", [(1, [(3, 1, 0)])], 2), ("count", [])]
    keys, outs, g = ctx.groupby(cols, [(0, "id"), (1, "id")], aggs, where=[(2, "le", 80)], groups_hint=hint)
    got = canon(keys, outs, [x[0] for x in aggs])
    m = s <= 80
    want = oracle.groupby([a[m], b[m], s[m], v[m]], [0, 1], aggs)
    check_gb(got, want)


def test_groupby_year_key_and_i64_key(ctx):
    rng = np.random.default_rng(12)
    n = 40_000
    d = rng.integers(-1000, 20000, n).astype(np.int32)
    k64 = rng.integers(-(2**62), 2**62, n).astype(np.int64) // 1000 * 1000
    k64[::7] = 0
    v = rng.integers(-1000, 1000, n).astype(np.int64)
    cols = [sx.col(dev(d), A.SX_DATE32), c(dev(v)), c(dev(k64))]
    keys, outs, g = ctx.groupby(cols, [(0, "year")], [("sum", [(1, [(1, 1, 0)])])], groups_hint=64)
    years = np.array([oracle.civil_year(int(x)) for x in d], np.int64)
    want = oracle.groupby([years, v], [0], [("sum", [(1, [(1, 1, 0)])])])
    check_gb(canon(keys, outs, ["sum"]), want)
    keys, outs, g = ctx.groupby(cols, [(2, "id")], [("count", []), ("max", [(1, [(1, 1, 0)])])], groups_hint=n)
    want = oracle.groupby([k64, v], [0], [("count", []), ("max", [(1, [(1, 1, 0)])])])
    check_gb(canon(keys, outs, ["count", "max"]), want)


@pytest.mark.parametrize("n", [0, 1, 5000, 100_003])
def test_groupby_keyless_reduce(ctx, n):
    rng = np.random.default_rng(n)
    a = rng.integers(0, 100, n).astype(np.int32)
    v = rng.integers(-(10**15), 10**15, n).astype(np.int64)
    cols = [c(dev(a)), c(dev(v))]
    aggs = [("sum", [(1, [(1, 1, 0)])]), ("count", []), ("min", [(1, [(1, 1, 0)])])]
    keys, outs, g = ctx.groupby(cols, [], aggs, where=[(0, "lt", 40)])
    assert g == 1
    m = a < 40
    cnt = int(outs[1].cpu().item())
    assert cnt == int(m.sum())
    if cnt:
        assert i128_rows(outs[0])[0] == sum(int(x) for x in v[m])
        assert int(outs[2].cpu().item()) == int(v[m].min())


def test_groupby_having_and_sel(ctx):
    rng = np.random.default_rng(21)
    n = 200_000
    k = np.sort(rng.integers(1, 40_000, n)).astype(np.int32)  # clustered keys (run pre-reduction)
    q = rng.integers(1, 51, n).astype(np.int64) * 100
    base = np.sort(rng.choice(n, n // 2, replace=False)).astype(np.int32)
    cols = [c(dev(k)), c(dev(q))]
    keys, outs, g = ctx.groupby(cols, [(0, "id")], [("sum", [(1, [(1, 1, 0)])])], in_sel=dev(base),
                                having=(0, "gt", 1200), groups_hint=40_000)
    want = [r for r in oracle.groupby([k[base], q[base]], [0], [("sum", [(1, [(1, 1, 0)])])]) if r[1] > 1200]
    check_gb(canon(keys, outs, ["sum"]), want)


@pytest.mark.parametrize("n", [1, 1023, 1024, 1025, 100_003])
@pytest.mark.parametrize("order", ["sorted", "unsorted", "one_run"])
def test_groupby_sorted_runs(ctx, monkeypatch, n, order):
    """Sorted-input strategy (forced with SX_GB_SORTED=2): non-decreasing keys aggregate by runs
    into a dense array; a decrease anywhere falls back to hashing.  Runs cross tile (1024 rows)
    and warp boundaries; keys include 0 and negatives; HAVING applies at extraction."""
    monkeypatch.setenv("SX_GB_SORTED", "2")
    rng = np.random.default_rng(n + len(order))
    if order == "one_run":
        k = np.full(n, 7, np.int32)
    else:
        k = np.sort(rng.integers(-50, max(n // 3, 2), n)).astype(np.int32)
        if order == "unsorted" and n > 1:
            j = int(rng.integers(1, n))
            k[j - 1], k[j] = k[j] + 1, k[j - 1]  # one descent (the last step, if j = n - 1)
    v = rng.integers(-(10**12), 10**12, n).astype(np.int64)
    w = rng.integers(0, 100, n).astype(np.int64)
    cols = [c(dev(k)), c(dev(k)), c(dev(v)), c(dev(w))]
    keys, aggs, g = ctx.groupby(cols, [(0, "id")], AGGS, groups_hint=n + 10)
    want = oracle.groupby([k, k, v, w], [0], AGGS)
    check_gb(canon(keys, aggs, [a[0] for a in AGGS]), want)
    assert g == len(want)
    keys, outs, g = ctx.groupby(cols, [(0, "id")], [("count", [])], having=(0, "ge", 3), groups_hint=n + 10)
    want = [r for r in oracle.groupby([k, k, v, w], [0], [("count", [])]) if r[1] >= 3]
    check_gb(canon(keys, outs, ["count"]), want)


def test_groupby_expression_overflow_is_an_error(ctx):
    v = np.array([2**62, 3], np.int64)
    with pytest.raises(sx.SxError) as e:
        ctx.groupby([c(dev(v))], [], [("sum", [(4, [(0, 1, 0)])])])
    assert e.value.status == A.SX_EOVERFLOW


# ------------------------------------------------------------------------------------- joins
@pytest.mark.parametrize("nb,np_,dom", [(0, 100, 10), (1, 1, 1), (3000, 5000, 1000), (20_000, 100_003, 40_000),
                                        (5000, 70_000, 2**40), (2000, 3000, 5)])
def test_join_types(ctx, nb, np_, dom):
    rng = np.random.default_rng(nb + np_)
    dt = np.int64 if dom > 2**31 else np.int32
    bk = rng.integers(-dom, dom, nb).astype(dt)
    pk = rng.integers(-dom, dom, np_).astype(dt)
    bpay = rng.integers(0, 10**9, nb).astype(np.int64)
    ppay = rng.integers(0, 255, np_).astype(np.uint8)
    tb, tp = dev(bk), dev(pk)
    ht = ctx.hash_build([c(tb), c(dev(bpay))], [0])
    assert ht.rows == nb
    p, b, pay = ctx.hash_probe(ht, [c(tp), c(dev(ppay))], [0], "inner", build_cols=[c(tb), c(dev(bpay))], bp=[1], pp=[1])
    wp, wb = oracle.join(bk, pk, "inner")
    got = sorted(zip(p.cpu().numpy().tolist(), b.cpu().numpy().tolist()))
    assert got == sorted(zip(wp.tolist(), wb.tolist()))
    pr, br = p.cpu().numpy(), b.cpu().numpy()
    assert np.array_equal(pay[0].cpu().numpy(), bpay[br]) and np.array_equal(pay[1].cpu().numpy(), ppay[pr])
    assert np.all(np.diff(pr) >= 0)  # typed keys: count/scan/expand emits in probe order
    s, _, _ = ctx.hash_probe(ht, [c(tp)], [0], "semi")
    assert np.array_equal(s.cpu().numpy(), oracle.join(bk, pk, "semi"))
    a, _, _ = ctx.hash_probe(ht, [c(tp)], [0], "anti")
    assert np.array_equal(a.cpu().numpy(), oracle.join(bk, pk, "anti"))


@pytest.mark.parametrize("kind", ["two_i32", "u8"])
def test_join_non_unique_other_keys(ctx, kind):
    """Non-unique INNER joins on packed two-column keys (typed expand path) and on u8 keys
    (generic path): the multiset of (probe, build) pairs and the gathered payloads."""
    rng = np.random.default_rng(17)
    nb, n = 4000, 20_000
    if kind == "two_i32":
        b1, b2 = rng.integers(0, 30, nb).astype(np.int32), rng.integers(0, 20, nb).astype(np.int32)
        p1, p2 = rng.integers(0, 35, n).astype(np.int32), rng.integers(0, 20, n).astype(np.int32)
        bcols, pcols, keys = [c(dev(b1)), c(dev(b2))], [c(dev(p1)), c(dev(p2))], [0, 1]
        bk = (b1.astype(np.int64) << 32) | b2
        pk = (p1.astype(np.int64) << 32) | p2
    else:
        b1 = rng.integers(0, 200, nb).astype(np.uint8)
        p1 = rng.integers(0, 256, n).astype(np.uint8)
        bcols, pcols, keys = [c(dev(b1))], [c(dev(p1))], [0]
        bk, pk = b1.astype(np.int64), p1.astype(np.int64)
    bpay = rng.integers(0, 10**9, nb).astype(np.int64)
    ht = ctx.hash_build(bcols + [c(dev(bpay))], keys)
    p, b, pay = ctx.hash_probe(ht, pcols, keys, "inner", build_cols=bcols + [c(dev(bpay))], bp=[len(keys)])
    wp, wb = oracle.join(bk, pk, "inner")
    got = sorted(zip(p.cpu().numpy().tolist(), b.cpu().numpy().tolist()))
    assert got == sorted(zip(wp.tolist(), wb.tolist()))
    assert np.array_equal(pay[0].cpu().numpy(), bpay[b.cpu().numpy()])


def test_join_unique_build_two_keys_where(ctx):
    rng = np.random.default_rng(3)
    nb = 30_000
    k1 = rng.integers(1, 5000, nb).astype(np.int32)
    k2 = rng.integers(1, 1000, nb).astype(np.int32)
    packed = (k1.astype(np.int64) << 32) | k2.astype(np.int64)
    _, first = np.unique(packed, return_index=True)
    k1, k2 = k1[np.sort(first)], k2[np.sort(first)]
    nb = len(k1)
    cost = rng.integers(100, 100000, nb).astype(np.int64)
    n = 150_000
    idx = rng.integers(0, nb, n)
    p1, p2 = k1[idx].copy(), k2[idx].copy()
    p2[::5] += 1000  # misses
    f = rng.integers(0, 10, n).astype(np.int32)
    ht = ctx.hash_build([c(dev(k1)), c(dev(k2)), c(dev(cost))], [0, 1], unique=True)
    p, b, pay = ctx.hash_probe(ht, [c(dev(p1)), c(dev(p2)), c(dev(f))], [0, 1], "inner", where=[(2, "lt", 7)],
                               build_cols=[c(dev(k1)), c(dev(k2)), c(dev(cost))], bp=[2], pp=[2])
    bpk = (k1.astype(np.int64) << 32) | k2.astype(np.int64)
    ppk = (p1.astype(np.int64) << 32) | p2.astype(np.int64)
    wp, wb = oracle.join(bpk, np.where(f < 7, ppk, np.int64(-1)), "inner")
    # unique build: output is ordered by probe row
    assert np.array_equal(p.cpu().numpy(), wp) and np.array_equal(b.cpu().numpy(), wb)
    assert np.array_equal(pay[0].cpu().numpy(), cost[wb])
    assert np.array_equal(pay[1].cpu().numpy(), f[wp])


# ------------------------------------------------------------------------------------- sort / top-k
def as_i128_tensor(vals):
    arr = np.array([[v & ((1 << 64) - 1), v >> 64] for v in vals], dtype=object)
    lo = np.array([int(x) if x < 2**63 else int(x) - 2**64 for x in arr[:, 0]], np.int64) if len(vals) else np.zeros(0, np.int64)
    hi = np.array([int(x) for x in arr[:, 1]], np.int64) if len(vals) else np.zeros(0, np.int64)
    return torch.from_numpy(np.stack([lo, hi], axis=1) if len(vals) else np.zeros((0, 2), np.int64)).cuda()


@pytest.mark.parametrize("n", [1, 2, 1000, 2048, 2049, 50_000, 300_001])
@pytest.mark.parametrize("k", [-1, 1, 10, 100, 1024])
def test_sort_topk(ctx, n, k):
    rng = np.random.default_rng(n * 7 + k)
    a = rng.integers(0, 5, n).astype(np.int32)  # many ties -> stability matters
    b = [int(x) for x in rng.integers(-(2**40), 2**40, n)]
    b = [x * (2**50) + 3 for x in b]  # beyond int64: exercise I128 words
    d = rng.integers(8000, 10500, n).astype(np.int32)
    u = rng.integers(0, 256, n).astype(np.uint8)
    cols = [sx.col(dev(a), A.SX_I32), sx.col(as_i128_tensor(b), A.SX_I128), sx.col(dev(d), A.SX_DATE32), c(dev(u))]
    for keys in ([(0, 0), (1, 1)], [(1, 1), (2, 0)], [(3, 1)], [(2, 0), (0, 1), (3, 0)]):
        perm = ctx.sort_topk(cols, keys, k)
        src = [a.tolist(), b, d.tolist(), u.tolist()]
        want = oracle.sort([src[i] for i, _ in keys], [1 if dd else 0 for _, dd in keys], k)
        assert np.array_equal(perm.cpu().numpy(), want), keys


@pytest.mark.parametrize("mode", ["tournament", "select", "warp"])
def test_topk_paths(ctx, monkeypatch, mode):
    """Top-k (k <= 1024) through the tournament rounds, the radix select (SX_TOPK=select) and the
    warp lists (K14w, SX_TOPK=warp, k <= 32), several rounds deep (n = 3e5, k = 1024 -> 150 chunks
    -> ... -> one CTA)."""
    monkeypatch.setenv("SX_TOPK", mode)
    rng = np.random.default_rng(11)
    n = 300_000
    v = rng.integers(-50, 50, n).astype(np.int64)  # heavy ties: the position word decides
    w = rng.integers(0, 3, n).astype(np.int32)
    for k in (1, 7, 32, 1000, 1024):
        perm = ctx.sort_topk([c(dev(v)), sx.col(dev(w), A.SX_I32)], [(0, 1), (1, 0)], k)
        want = oracle.sort([v.tolist(), w.tolist()], [1, 0], k)
        assert np.array_equal(perm.cpu().numpy(), want), k


@pytest.mark.parametrize("mode", ["onesweep", "onesweep-match", "lsd"])
def test_sort_many_tiles(ctx, monkeypatch, mode):
    """Full sorts spanning ~500 onesweep tiles (decoupled look-back chains across many CTAs):
    full-range int64 keys (all 8 digits vary), and heavy ties resolved by stability."""
    if mode == "lsd":
        monkeypatch.setenv("SX_SORT", "lsd")
    if mode == "onesweep-match":
        monkeypatch.setenv("SX_SORT_RANK", "match")
    rng = np.random.default_rng(21)
    n = 2_000_003
    v = rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64)
    perm = ctx.sort_topk([c(dev(v))], [(0, 0)], -1)
    assert np.array_equal(perm.cpu().numpy(), oracle.sort([v.tolist()], [0], -1))
    t = rng.integers(0, 3, n).astype(np.int32)
    perm = ctx.sort_topk([sx.col(dev(t), A.SX_I32)], [(0, 1)], -1)
    assert np.array_equal(perm.cpu().numpy(), oracle.sort([t.tolist()], [1], -1))


def test_sort_with_sel(ctx):
    rng = np.random.default_rng(8)
    n = 20_000
    v = rng.integers(-1000, 1000, n).astype(np.int64)
    base = np.sort(rng.choice(n, 7000, replace=False)).astype(np.int32)
    perm = ctx.sort_topk([c(dev(v))], [(0, 1)], 50, in_sel=dev(base))
    want = base[oracle.sort([v[base].tolist()], [1], 50)]
    assert np.array_equal(perm.cpu().numpy(), want)


def test_gather(ctx):
    rng = np.random.default_rng(1)
    v = rng.integers(-5, 5, 10_000).astype(np.int64)
    s = rng.integers(0, 10_000, 777).astype(np.int32)
    assert np.array_equal(ctx.gather(c(dev(v)), dev(s)).cpu().numpy(), v[s])


@pytest.mark.parametrize("span", [1000, 1 << 31])
def test_membership_only_build(ctx, span):
    """SX_BUILD_MEMBERSHIP: semi/anti probes equal those of a full build (bitmap when the key range
    allows, else the table is built after all); INNER probes are refused when no table exists."""
    rng = np.random.default_rng(9)
    bk = rng.integers(-span // 2, span // 2, 5000, dtype=np.int64)
    pk = rng.integers(-span // 2, span // 2, 20_011, dtype=np.int64)
    bk[:100] = pk[:100]  # guaranteed matches
    b, p = dev(bk), dev(pk)
    ht = ctx.hash_build([c(b)], [0], membership=True)
    for jt in ("semi", "anti"):
        got, _, _ = ctx.hash_probe(ht, [c(p)], [0], jt)
        want = oracle.join(bk, pk, jt)
        assert np.array_equal(got.cpu().numpy(), want), jt
    if span <= (1 << 30):
        with pytest.raises(sx.SxError):
            ctx.hash_probe(ht, [c(p)], [0], "inner")
    else:
        op, ob, _ = ctx.hash_probe(ht, [c(p)], [0], "inner")
        wp, wb = oracle.join(bk, pk, "inner")
        assert sorted(zip(op.cpu().numpy().tolist(), ob.cpu().numpy().tolist())) == sorted(zip(wp.tolist(), wb.tolist()))


@pytest.mark.parametrize("ng,hint,nkeys", [(50_000, 50_000, 1), (300_000, 400_000, 2), (9_000, 8_192, 1)])
def test_groupby_partitioned_ranges(ctx, ng, hint, nkeys):
    """K10p (mid G, >= 2^22 rows): radix partition on the group key + per-range shared tables,
    with a where-predicate, keys 0/negative, two packed keys, and against the global-table path."""
    rng = np.random.default_rng(ng)
    n = (1 << 22) + 37
    k = rng.integers(-(ng // 2), ng - ng // 2, n).astype(np.int32)
    k2 = (rng.integers(0, 3, n)).astype(np.int32)
    v = rng.integers(-(10**12), 10**12, n).astype(np.int64)
    w = rng.integers(0, 100, n).astype(np.int64)
    cols = [c(dev(k)), c(dev(k2)), c(dev(v)), c(dev(w))]
    keys = [(0, "id")] + ([(1, "id")] if nkeys == 2 else [])
    aggs = AGGS[:5]
    got_keys, got_aggs, g = ctx.groupby(cols, keys, aggs, where=[(3, "lt", 90)], groups_hint=hint)
    got = canon(got_keys, got_aggs, [a[0] for a in aggs])
    m = w < 90
    want = oracle.groupby([k[m], k2[m], v[m], w[m]], list(range(nkeys)), aggs)
    check_gb(got, want)
    assert g == len(want)


@pytest.mark.parametrize("direct", ["1", "0"])
def test_unique_build_direct_address(ctx, monkeypatch, direct):
    """Unique single-key builds whose table would exceed 8 MB over a small key range become a
    bitmap + direct row array (no hash table); SX_DIRECT=0 keeps the table.  INNER (with payload
    gather and a probe predicate), SEMI and ANTI equal the oracle's either way."""
    monkeypatch.setenv("SX_DIRECT", direct)
    rng = np.random.default_rng(21)
    nb = 700_001
    bk = (rng.permutation(nb * 3)[:nb] - nb).astype(np.int32)  # unique, negatives included
    bp = rng.integers(-10**9, 10**9, nb).astype(np.int64)
    npr = 2_000_003
    pk = rng.integers(-nb - 5, 2 * nb + 5, npr).astype(np.int32)
    pw = rng.integers(0, 10, npr).astype(np.int32)
    b, p = dev(bk), dev(pk)
    ht = ctx.hash_build([c(b)], [0], unique=True)
    op, ob, (pay,) = ctx.hash_probe(ht, [c(p), c(dev(pw))], [0], "inner", where=[(1, "lt", 7)],
                                    build_cols=[c(b), c(dev(bp))], bp=[1])
    m = pw < 7
    wp, wb = oracle.join(bk, pk[m], "inner")
    idx = np.nonzero(m)[0]
    got = sorted(zip(op.cpu().numpy().tolist(), ob.cpu().numpy().tolist()))
    assert got == sorted(zip(idx[wp].tolist(), wb.tolist()))
    assert np.array_equal(pay.cpu().numpy(), bp[ob.cpu().numpy()])
    for jt in ("semi", "anti"):
        got, _, _ = ctx.hash_probe(ht, [c(p)], [0], jt)
        assert np.array_equal(got.cpu().numpy(), oracle.join(bk, pk, jt)), jt


@pytest.mark.parametrize("op", ["lt", "le", "gt", "ge", "eq", "ne", "between"])
def test_filter_int32_constants_beyond_int32(ctx, op):
    """32-bit dense predicate path: constants outside the int32 range (uniformly true / false) and
    at its edges, vs the oracle's int64 comparisons; a ragged tail."""
    rng = np.random.default_rng(17)
    n = 50_021
    x = rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    x[:4] = [-2**31, 2**31 - 1, 0, -1]
    t = dev(x)
    for lo, hi in ((2**40, 2**41), (-2**40, 2**40), (-2**40, -2**39), (2**31 - 1, 2**31), (-2**31, -2**31),
                   (5, 3), (-7, 2**35)):
        pr = (0, op, lo, hi) if op == "between" else (0, op, lo)
        sel, _ = ctx.filter([c(t)], [pr])
        want = oracle.filter([x.astype(np.int64)], [pr])
        assert np.array_equal(sel.cpu().numpy(), want), (op, lo, hi)


LONG = b"greenish-goldenrod-x"  # 20 bytes: verification reaches past one 16-byte chunk


@pytest.mark.parametrize("maxlen", [40, 300])
def test_filter_contains_edges(ctx, maxlen):
    """Warp-cooperative CONTAINS: empty strings, matches at the first / last byte, a pattern split
    across two neighbouring strings (must not match), warps whose byte span exceeds the shared
    stage (maxlen 300), a ragged last warp, the empty pattern, a 20-byte pattern, and a chars buffer
    that starts off a 16-byte boundary."""
    rng = np.random.default_rng(maxlen)
    n = 10_007
    strs = []
    for i in range(n):
        L = int(rng.integers(0, maxlen))
        s = bytes(rng.integers(97, 123, L, dtype=np.uint8))
        r = i % 7
        if r == 0 and L >= 5:
            s = b"green" + s[5:]
        elif r == 1 and L >= 5:
            s = s[:-5] + b"green"
        elif r == 2:
            s = s + b"gre"          # and the next string starts with "en": no match across the boundary
        elif r == 3:
            s = b"en" + s
        elif r == 4 and L >= 30:
            s = s[:3] + LONG + s[3 + len(LONG):]
        strs.append(s)
    offs = np.zeros(n + 1, np.int64)
    offs[1:] = np.cumsum([len(x) for x in strs])
    chars = np.frombuffer(b"".join(strs), np.uint8).copy()
    for pat in (b"green", b"gre", b"gr", b"gree", b"", b"q", LONG):
        sel, _ = ctx.filter([sx.col(dev(chars), A.SX_STR, offsets=dev(offs))], [(0, "contains", pat)])
        assert np.array_equal(sel.cpu().numpy(), oracle.contains(offs, chars, pat)), pat
    # a chars buffer that does not start on a 16-byte boundary
    pad = torch.zeros(chars.size + 3, dtype=torch.uint8, device="cuda")
    pad[3:] = dev(chars)
    for pat in (b"green", LONG):
        sel, _ = ctx.filter([sx.col(pad[3:], A.SX_STR, offsets=dev(offs))], [(0, "contains", pat)])
        assert np.array_equal(sel.cpu().numpy(), oracle.contains(offs, chars, pat)), pat


@pytest.mark.parametrize("pat", [b"a", b"ab", b"aba", b"abab", b"aabab", b"babbaabab"])
def test_filter_contains_dense_alphabet(ctx, pat):
    """Two-letter alphabet: overlapping occurrences, candidates in every 4-byte window, matches that
    straddle lane (16-byte) and warp-step (512-byte) boundaries, patterns of 1..9 bytes."""
    rng = np.random.default_rng(len(pat))
    n = 20_011
    lens = rng.integers(0, 24, n)
    offs = np.zeros(n + 1, np.int64)
    offs[1:] = np.cumsum(lens)
    chars = rng.choice(np.frombuffer(b"ab", np.uint8), int(offs[-1]), p=[0.6, 0.4]).astype(np.uint8)
    sel, _ = ctx.filter([sx.col(dev(chars), A.SX_STR, offsets=dev(offs))], [(0, "contains", pat)])
    assert np.array_equal(sel.cpu().numpy(), oracle.contains(offs, chars, pat))


def test_misaligned_and_strided_columns_rejected(ctx):
    """sx.h alignment rule: an offset or strided view is rejected by the binding, and a
    misaligned pointer passed straight through the C ABI returns SX_EINVAL instead of faulting."""
    import ctypes as C

    x = torch.arange(1000, dtype=torch.int64, device="cuda")
    with pytest.raises(sx.SxError):
        sx.col(x[1:])
    with pytest.raises(sx.SxError):
        sx.col(x[::2])
    raw = (A.Col * 1)(A.Col(A.SX_I64, 0, 999, x.data_ptr() + 8, None, None))
    pred = (A.Pred * 1)(A.Pred(0, A.SX_LT, 5, 0, None, 0, 0))
    out = A.Sel()
    st = ctx.L.sx_filter(ctx.h, raw, 1, pred, 1, None, None, 0, C.byref(out), None)
    assert st == A.SX_EINVAL
    # the context is still healthy (no sticky fault): an aligned call succeeds
    sel, _ = ctx.filter([sx.col(x)], [(0, "lt", 5)])
    assert sel.cpu().tolist() == [0, 1, 2, 3, 4]
