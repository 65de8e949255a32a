"""Generator tests: exact row counts, determinism, shard union,
structural invariants and statistical closed forms."""
import math

import numpy as np
import pytest

import gen


@pytest.fixture(scope="module")
def sf01():
    return gen.cpu_tables(100, seed=42)  # SF 0.1


def test_sizes():
    assert gen.sizes(10) == {"supplier": 100, "customer": 1500, "part": 2000, "partsupp": 8000, "orders": 15000}
    assert gen.sizes(100000)["orders"] == 150_000_000
    assert gen.key_bytes_for(100000) == 4 and gen.key_bytes_for(1000000) == 8


def test_determinism_and_seed():
    a = gen.cpu_tables(10, seed=42)
    b = gen.cpu_tables(10, seed=42)
    c = gen.cpu_tables(10, seed=7)
    for t in a:
        for col in a[t]:
            assert np.array_equal(a[t][col], b[t][col]), (t, col)
    assert not np.array_equal(a["lineitem"]["l_quantity"], c["lineitem"]["l_quantity"])


def test_shard_union_equals_full():
    full = gen.cpu_tables(10, seed=1)
    parts = [gen.cpu_tables(10, seed=1, shard=(r, 3)) for r in range(3)]
    for t in full:
        for col in full[t]:
            if col == "p_name_offsets":
                continue
            cat = np.concatenate([p[t][col] for p in parts])
            assert np.array_equal(cat, full[t][col]), (t, col)


def test_row_counts_and_keys(sf01):
    o, li = sf01["orders"], sf01["lineitem"]
    n = len(o["o_orderkey"])
    assert n == 150_000
    i = np.arange(1, n + 1)
    assert np.array_equal(o["o_orderkey"], ((i >> 3) << 5) | (i & 7))  # 8 of every 32 keys
    # lineitem clustered by order; nlines in [1, 7]
    runs = np.diff(np.flatnonzero(np.r_[True, li["l_orderkey"][1:] != li["l_orderkey"][:-1], True]))
    assert len(runs) == n and runs.min() >= 1 and runs.max() <= 7
    assert abs(runs.mean() - 4.0) < 6 * math.sqrt(4.0 / n)  # U[1,7]: mean 4, var 4
    assert np.all(o["o_custkey"] % 3 != 0) and o["o_custkey"].min() >= 1
    assert o["o_custkey"].max() <= len(sf01["customer"]["c_custkey"])


def test_partsupp_structure(sf01):
    ps = sf01["partsupp"]
    pk, sk = ps["ps_partkey"], ps["ps_suppkey"]
    assert np.array_equal(pk, np.repeat(np.arange(1, len(pk) // 4 + 1), 4))
    sk4 = sk.reshape(-1, 4)
    assert np.all(np.sort(sk4, axis=1)[:, 1:] != np.sort(sk4, axis=1)[:, :-1])  # 4 distinct suppkeys per part
    li = sf01["lineitem"]
    ps_pairs = set(zip(pk.tolist(), sk.tolist()))
    li_pairs = set(zip(li["l_partkey"].tolist(), li["l_suppkey"].tolist()))
    assert li_pairs <= ps_pairs  # every lineitem (part, supp) exists in partsupp


def test_lineitem_value_ranges(sf01):
    li, o = sf01["lineitem"], sf01["orders"]
    od = np.repeat(o["o_orderdate"], np.diff(np.flatnonzero(
        np.r_[True, li["l_orderkey"][1:] != li["l_orderkey"][:-1], True])))
    d = li["l_shipdate"] - od
    assert d.min() >= 1 and d.max() <= 121
    assert set(np.unique(li["l_quantity"] // 100)) == set(range(1, 51)) and np.all(li["l_quantity"] % 100 == 0)
    assert li["l_discount"].min() == 0 and li["l_discount"].max() == 10
    assert li["l_tax"].min() == 0 and li["l_tax"].max() == 8
    rf, ls = li["l_returnflag"], li["l_linestatus"]
    assert set(np.unique(rf).tolist()) == {ord("A"), ord("N"), ord("R")}
    assert np.all(rf[ls == ord("O")] == ord("N"))  # O => shipdate > 9298 => receipt > 9298 => N
    price = 90000 + ((li["l_partkey"] // 10) % 20001) + 100 * (li["l_partkey"] % 1000)
    assert np.array_equal(li["l_extendedprice"], (li["l_quantity"] // 100) * price)


def test_statistical_closed_forms(sf01):
    """SURVEY App. C closed forms, each within 6 sigma (binomial / CLT)."""
    li = sf01["lineitem"]
    n = len(li["l_shipdate"])

    def close(k, p):
        assert abs(k / n - p) <= 6 * math.sqrt(p * (1 - p) / n), (k / n, p)

    s, disc, qty = li["l_shipdate"], li["l_discount"], li["l_quantity"]
    close(int(np.sum((s >= 8766) & (s < 9131) & (disc >= 5) & (disc <= 7) & (qty < 2400))), 0.019032)
    close(int(np.sum(s <= 10471)), 0.98593)
    close(int(np.sum(s > 9204)), 0.539069)
    q = qty / 100
    assert abs(q.mean() - 25.5) < 6 * math.sqrt((50**2 - 1) / 12 / n)


def _q1_group_probs():
    """Exact probabilities of each Q1 group among ALL lineitem rows, restricted to shipdate <= 10471,
    by enumerating the generator's distribution: orderdate U[8035,10440], ship = od + U[1,121],
    receipt = ship + U[1,30], rf = N if receipt > 9298 else R/A (1/2 each), ls = O iff ship > 9298.
    (SURVEY App. C quotes (A,F) .246779, (N,F) .006442, (N,O) .485934 of the same quantity.)"""
    od = np.arange(8035, 10441)[:, None, None]
    ship = od + np.arange(1, 122)[None, :, None]
    rec = ship + np.arange(1, 31)[None, None, :]
    w = 1.0 / (2406 * 121 * 30)
    q1 = np.broadcast_to(ship <= 10471, rec.shape)
    f = np.broadcast_to(ship <= 9298, rec.shape)
    n_rec = rec > 9298
    return {("A", "F"): 0.5 * w * np.sum(q1 & f & ~n_rec), ("R", "F"): 0.5 * w * np.sum(q1 & f & ~n_rec),
            ("N", "F"): w * np.sum(q1 & f & n_rec), ("N", "O"): w * np.sum(q1 & ~f)}


def test_q1_group_fractions(sf01):
    li = sf01["lineitem"]
    n = len(li["l_shipdate"])
    rf, ls, s = li["l_returnflag"], li["l_linestatus"], li["l_shipdate"]
    probs = _q1_group_probs()
    assert abs(probs[("A", "F")] - 0.246779) < 1e-5 and abs(probs[("N", "O")] - 0.485934) < 1e-5
    assert abs(probs[("N", "F")] - 0.006442) < 1e-5
    for (a, b), p in probs.items():
        k = int(np.sum((rf == ord(a)) & (ls == ord(b)) & (s <= 10471)))
        assert abs(k / n - p) <= 6 * math.sqrt(p * (1 - p) / n), (a, b, k / n, p)


def test_part_names(sf01):
    p = sf01["part"]
    words = {gen.cpu_lib().sxg_cpu_word(w).decode() for w in range(92)}
    assert len(words) == 92
    offs, chars = p["p_name_offsets"], p["p_name_chars"].tobytes()
    green = 0
    for r in range(len(p["p_partkey"])):
        name = chars[offs[r]:offs[r + 1]].decode()
        ws = name.split(" ")
        assert len(ws) == 5 and len(set(ws)) == 5 and set(ws) <= words
        green += "green" in name
    n = len(p["p_partkey"])
    pr = 5 / 92
    assert abs(green / n - pr) <= 6 * math.sqrt(pr * (1 - pr) / n)
    # only the word "green" contains the substring (reading R9)
    assert [w for w in words if "green" in w] == ["green"]
