"""Oracle query pins on generated TPC-H-shaped data (SURVEY §8(c) "What pins each part"):
an independent implementation of each query through a library relational engine
(pandas merge/groupby/sort_values) at small SF, plus invariants and closed forms.
"""
import math

import numpy as np
import pandas as pd
import pytest

import gen
import oracle

NAT = oracle.NATIONS


@pytest.fixture(scope="module", params=[10, 50])
def data(request):
    return request.param, gen.cpu_tables(request.param, seed=42, key_bytes=8)


def df(t):
    return pd.DataFrame({k: v for k, v in t.items() if k not in ("p_name_offsets", "p_name_chars")})


def test_q1_vs_pandas(data):
    sfm, t = data
    li = df(t["lineitem"])
    f = li[li.l_shipdate <= 10471].copy()
    f["dp"] = f.l_extendedprice * (100 - f.l_discount)
    f["ch"] = f.dp * (100 + f.l_tax)
    g = f.groupby(["l_returnflag", "l_linestatus"]).agg(
        q=("l_quantity", "sum"), b=("l_extendedprice", "sum"), dp=("dp", "sum"), ch=("ch", "sum"),
        d=("l_discount", "sum"), n=("l_quantity", "size")).reset_index().sort_values(["l_returnflag", "l_linestatus"])
    want = [(chr(r.l_returnflag), chr(r.l_linestatus), int(r.q), int(r.b), int(r.dp), int(r.ch), int(r.n))
            for r in g.itertuples()]
    got = oracle.run_query("q1", t)
    assert [(r[0], r[1], r[2], r[3], r[4], r[5], r[9]) for r in got] == want
    for r, w in zip(got, g.itertuples()):
        assert math.isclose(r[6], w.q / w.n / 100, rel_tol=1e-12)
        assert math.isclose(r[8], w.d / w.n / 100, rel_tol=1e-12)
    # invariants: exactly 4 groups; sum of counts = filtered rows
    assert len(got) == 4 and sum(r[9] for r in got) == int(np.sum(t["lineitem"]["l_shipdate"] <= 10471))


def test_q6_vs_numpy(data):
    sfm, t = data
    li = t["lineitem"]
    s, d, q, e = li["l_shipdate"], li["l_discount"], li["l_quantity"], li["l_extendedprice"]
    m = (s >= 8766) & (s < 9131) & (d >= 5) & (d <= 7) & (q < 2400)
    assert oracle.run_query("q6", t) == [(int(np.sum(e[m] * d[m])),)]


def _q3_pandas(t, limit):
    c, o, li = df(t["customer"]), df(t["orders"]), df(t["lineitem"])
    j = c[c.c_mktsegment == 1].merge(o[o.o_orderdate < 9204], left_on="c_custkey", right_on="o_custkey")
    j = j.merge(li[li.l_shipdate > 9204], left_on="o_orderkey", right_on="l_orderkey")
    j["rev"] = j.l_extendedprice * (100 - j.l_discount)
    g = j.groupby(["l_orderkey", "o_orderdate", "o_shippriority"]).rev.sum().reset_index()
    g = g.sort_values(["rev", "o_orderdate", "l_orderkey"], ascending=[False, True, True])
    rows = [(int(r.l_orderkey), int(r.rev), int(r.o_orderdate), int(r.o_shippriority)) for r in g.itertuples()]
    return rows if limit < 0 else rows[:limit], len(j)


def test_q3_vs_pandas(data):
    sfm, t = data
    want_all, joined = _q3_pandas(t, -1)
    assert oracle.run_query("q3", t, limit=-1) == want_all
    assert oracle.run_query("q3", t) == want_all[:10]
    # closed forms (App. C): joined rows ~ 29,925*SF, groups ~ 11,322*SF (loose: +-6 sigma Poisson)
    sf = sfm / 1000
    assert abs(joined - 29925 * sf) < 6 * math.sqrt(29925 * sf) + 0.05 * 29925 * sf
    revs = [r[1] for r in want_all]
    assert revs == sorted(revs, reverse=True)


def _q9_pandas(t, color="green"):
    p = t["part"]
    names = [p["p_name_chars"][p["p_name_offsets"][i]:p["p_name_offsets"][i + 1]].tobytes().decode()
             for i in range(len(p["p_partkey"]))]
    pdf = pd.DataFrame({"p_partkey": p["p_partkey"], "name": names})
    pdf = pdf[pdf.name.str.contains(color, regex=False)]
    li, ps, s, o = df(t["lineitem"]), df(t["partsupp"]), df(t["supplier"]), df(t["orders"])
    j = li.merge(pdf, left_on="l_partkey", right_on="p_partkey")
    j = j.merge(ps, left_on=["l_partkey", "l_suppkey"], right_on=["ps_partkey", "ps_suppkey"])
    j = j.merge(s, left_on="l_suppkey", right_on="s_suppkey").merge(o, left_on="l_orderkey", right_on="o_orderkey")
    j["year"] = pd.to_datetime(j.o_orderdate, unit="D").dt.year
    j["nation"] = [NAT[k] for k in j.s_nationkey]
    j["amount"] = j.l_extendedprice * (100 - j.l_discount) - j.ps_supplycost * j.l_quantity
    g = j.groupby(["nation", "year"]).amount.sum().reset_index().sort_values(["nation", "year"], ascending=[True, False])
    return [(r.nation, int(r.year), int(r.amount)) for r in g.itertuples()], len(j), len(pdf)


def test_q9_vs_pandas(data):
    sfm, t = data
    want, joined, ngreen = _q9_pandas(t)
    assert oracle.run_query("q9", t) == want
    assert len(want) == 175  # 25 nations x 7 years
    # each green lineitem joins exactly one partsupp, supplier and order by construction
    green = set(t["part"]["p_partkey"][[i for i in range(len(t["part"]["p_partkey"]))
                                        if b"green" in t["part"]["p_name_chars"][t["part"]["p_name_offsets"][i]:
                                                                                 t["part"]["p_name_offsets"][i + 1]].tobytes()]].tolist())
    assert joined == int(np.isin(t["lineitem"]["l_partkey"], list(green)).sum())


def _q18_pandas(t, qty_gt):
    li, o, c = df(t["lineitem"]), df(t["orders"]), df(t["customer"])
    s = li.groupby("l_orderkey").l_quantity.sum()
    big = set(s[s > qty_gt].index.tolist())
    j = c.merge(o[o.o_orderkey.isin(big)], left_on="c_custkey", right_on="o_custkey")
    j = j.merge(li, left_on="o_orderkey", right_on="l_orderkey")
    g = j.groupby(["c_custkey", "o_orderkey", "o_orderdate", "o_totalprice"]).l_quantity.sum().reset_index()
    g = g.sort_values(["o_totalprice", "o_orderdate", "o_orderkey"], ascending=[False, True, True])
    return [(oracle.c_name(int(r.c_custkey)), int(r.c_custkey), int(r.o_orderkey), int(r.o_orderdate),
             int(r.o_totalprice), int(r.l_quantity)) for r in g.itertuples()][:100], len(big)


@pytest.mark.parametrize("qty", [30000, 25000])
def test_q18_vs_pandas(data, qty):
    sfm, t = data
    want, nbig = _q18_pandas(t, qty)
    got = oracle.run_query("q18", t, oracle.default_params(q18_qty_gt=qty))
    assert got == want
    assert all(r[5] > qty for r in got)
    if qty == 25000:
        # P(order qualifies) for QUANTITY=250: (1/7) * P(sum of 7 U[1..50] >= 251) computed by convolution
        dist = np.zeros(351)
        dist[0] = 1.0
        for _ in range(7):
            nd = np.zeros(351)
            for v in range(1, 51):
                nd[v:] += dist[:351 - v] / 50
            dist = nd
        p = dist[251:].sum() / 7
        n = len(t["orders"]["o_orderkey"])
        assert abs(nbig - p * n) < 6 * math.sqrt(p * n) + 1
