"""CPU oracle (ctypes over oracle/liboracle.so).  TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module.  The product package
(paper_2508_04701_b200) never imports it; see oracle/oracle.h for what it
computes and the passages each function follows.

Result rows use the canonical Python form shared with the GPU-side decoder
(plain tuples of ints/floats/str; int128 values as Python ints):

* q1:  (returnflag, linestatus, sum_qty, sum_base_price, sum_disc_price, sum_charge,
        avg_qty, avg_price, avg_disc, count_order)
* q6:  (revenue | None,)
* q3:  (l_orderkey, revenue, o_orderdate, o_shippriority)
* q9:  (nation, o_year, sum_profit)
* q18: (c_name, c_custkey, o_orderkey, o_orderdate, o_totalprice, sum_qty)
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

NATIONS = [
    "ALGERIA", "ARGENTINA", "BRAZIL", "CANADA", "EGYPT", "ETHIOPIA", "FRANCE", "GERMANY",
    "INDIA", "INDONESIA", "IRAN", "IRAQ", "JAPAN", "JORDAN", "KENYA", "MOROCCO",
    "MOZAMBIQUE", "PERU", "CHINA", "ROMANIA", "SAUDI ARABIA", "VIETNAM", "RUSSIA",
    "UNITED KINGDOM", "UNITED STATES",
]


class I128(C.Structure):
    _fields_ = [("lo", C.c_uint64), ("hi", C.c_int64)]


def i128_to_int(v) -> int:
    return (int(v.hi) << 64) | int(v.lo)


def int_to_i128(x: int) -> I128:
    return I128(x & ((1 << 64) - 1), x >> 64)


_VP = C.c_void_p


class Tables(C.Structure):
    _fields_ = [
        ("n_lineitem", C.c_int64), ("l_orderkey", _VP), ("l_partkey", _VP), ("l_suppkey", _VP),
        ("l_quantity", _VP), ("l_extendedprice", _VP), ("l_discount", _VP), ("l_tax", _VP),
        ("l_returnflag", _VP), ("l_linestatus", _VP), ("l_shipdate", _VP),
        ("n_orders", C.c_int64), ("o_orderkey", _VP), ("o_custkey", _VP), ("o_orderdate", _VP),
        ("o_shippriority", _VP), ("o_totalprice", _VP),
        ("n_customer", C.c_int64), ("c_custkey", _VP), ("c_mktsegment", _VP),
        ("n_part", C.c_int64), ("p_partkey", _VP), ("p_name_offsets", _VP), ("p_name_chars", _VP),
        ("n_partsupp", C.c_int64), ("ps_partkey", _VP), ("ps_suppkey", _VP), ("ps_supplycost", _VP),
        ("n_supplier", C.c_int64), ("s_suppkey", _VP), ("s_nationkey", _VP),
    ]


class Params(C.Structure):
    _fields_ = [
        ("q1_shipdate_max", C.c_int32), ("q3_segment", C.c_int32), ("q3_date", C.c_int32),
        ("q6_date_lo", C.c_int32), ("q6_date_hi", C.c_int32), ("q6_disc_lo", C.c_int64),
        ("q6_disc_hi", C.c_int64), ("q6_qty_lt", C.c_int64), ("q9_color", C.c_char * 16),
        ("q18_qty_gt", C.c_int64),
    ]


class Q1Row(C.Structure):
    _fields_ = [("returnflag", C.c_uint8), ("linestatus", C.c_uint8), ("sum_qty", I128),
                ("sum_base_price", I128), ("sum_disc_price", I128), ("sum_charge", I128), ("sum_disc", I128),
                ("count_order", C.c_int64), ("avg_qty", C.c_double), ("avg_price", C.c_double),
                ("avg_disc", C.c_double)]


class Q6Row(C.Structure):
    _fields_ = [("revenue", I128), ("is_null", C.c_int32)]


class Q3Row(C.Structure):
    _fields_ = [("l_orderkey", C.c_int64), ("revenue", I128), ("o_orderdate", C.c_int32),
                ("o_shippriority", C.c_int32)]


class Q9Row(C.Structure):
    _fields_ = [("nationkey", C.c_int32), ("o_year", C.c_int32), ("sum_profit", I128)]


class Q18Row(C.Structure):
    _fields_ = [("c_custkey", C.c_int32), ("o_orderdate", C.c_int32), ("o_orderkey", C.c_int64),
                ("o_totalprice", C.c_int64), ("sum_qty", I128)]


class Pred(C.Structure):
    _fields_ = [("col", C.c_int32), ("op", C.c_int32), ("lo", C.c_int64), ("hi", C.c_int64)]


class Factor(C.Structure):
    _fields_ = [("col", C.c_int32), ("mul", C.c_int64), ("add", C.c_int64)]


class Term(C.Structure):
    _fields_ = [("coef", C.c_int64), ("nf", C.c_int32), ("f", Factor * 3)]


class Expr(C.Structure):
    _fields_ = [("nterms", C.c_int32), ("t", Term * 2)]


OPS = {"lt": 0, "le": 1, "gt": 2, "ge": 3, "eq": 4, "ne": 5, "between": 6}
AGGS = {"sum": 0, "count": 1, "min": 2, "max": 3, "avg": 4}


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make oracle`")
        L = C.CDLL(path)
        P = C.POINTER
        L.or_default_params.argtypes = [P(Params)]
        L.or_q1.argtypes = [P(Tables), P(Params), P(Q1Row), C.c_int64]
        L.or_q6.argtypes = [P(Tables), P(Params), P(Q6Row)]
        L.or_q3.argtypes = [P(Tables), P(Params), C.c_int64, P(Q3Row), C.c_int64]
        L.or_q9.argtypes = [P(Tables), P(Params), P(Q9Row), C.c_int64]
        L.or_q18.argtypes = [P(Tables), P(Params), C.c_int64, P(Q18Row), C.c_int64]
        for f in ("or_q1", "or_q6", "or_q3", "or_q9", "or_q18"):
            getattr(L, f).restype = C.c_int64
        L.or_filter.argtypes = [C.c_int64, _VP, P(Pred), C.c_int32, _VP]
        L.or_filter.restype = C.c_int64
        L.or_contains.argtypes = [C.c_int64, _VP, _VP, C.c_char_p, C.c_int32, _VP]
        L.or_contains.restype = C.c_int64
        L.or_eval_expr.argtypes = [C.c_int64, _VP, P(Expr), _VP]
        L.or_join.argtypes = [C.c_int64, _VP, C.c_int64, _VP, C.c_int32, _VP, _VP, C.c_int64]
        L.or_join.restype = C.c_int64
        L.or_groupby.argtypes = [C.c_int64, _VP, C.c_int32, _VP, C.c_int32, _VP, P(Expr), _VP, _VP, _VP, _VP,
                                 C.c_int64]
        L.or_groupby.restype = C.c_int64
        L.or_sort.argtypes = [C.c_int64, _VP, C.c_int32, _VP, C.c_int64, _VP]
        L.or_sort.restype = C.c_int64
        L.or_civil_year.argtypes = [C.c_int32]
        L.or_civil_year.restype = C.c_int32
        L.or_unmix64.argtypes = [C.c_uint64]
        L.or_unmix64.restype = C.c_uint64
        L.or_pair_mix.argtypes = [C.c_int64, C.c_int64]
        L.or_pair_mix.restype = C.c_uint64
        L.or_mb_join_closed.argtypes = [C.c_int64, C.c_int64, _VP, _VP, P(JoinSummary)]
        L.or_mb_join_hash.argtypes = [C.c_int64, _VP, _VP, C.c_int64, _VP, _VP, P(JoinSummary)]
        L.or_mb_groupby_direct.argtypes = [C.c_int64, _VP, _VP, C.c_int64, _VP, _VP, _VP, _VP]
        L.or_mb_groupby_direct.restype = C.c_int64
        _lib = L
    return _lib


def default_params(**over) -> Params:
    p = Params()
    lib().or_default_params(C.byref(p))
    for k, v in over.items():
        if k == "q9_color":
            v = v.encode() if isinstance(v, str) else v
        setattr(p, k, v)
    return p


def _c(a, dt):
    return np.ascontiguousarray(np.asarray(a), dtype=dt)


def make_tables(t: dict) -> tuple[Tables, list]:
    """numpy table dict (gen.cpu_tables layout) -> (Tables struct, keep-alive list)."""
    keep = []
    T = Tables()

    def put(field, arr, dt):
        a = _c(arr, dt)
        keep.append(a)
        setattr(T, field, a.ctypes.data)
        return len(a)

    li = t.get("lineitem")
    if li is not None:
        T.n_lineitem = len(li["l_shipdate"]) if "l_shipdate" in li else len(li["l_orderkey"])
        for f, dt in [("l_orderkey", np.int64), ("l_partkey", np.int32), ("l_suppkey", np.int32),
                      ("l_quantity", np.int64), ("l_extendedprice", np.int64), ("l_discount", np.int64),
                      ("l_tax", np.int64), ("l_returnflag", np.uint8), ("l_linestatus", np.uint8),
                      ("l_shipdate", np.int32)]:
            if f in li:
                put(f, li[f], dt)
    o = t.get("orders")
    if o is not None:
        T.n_orders = len(o["o_orderkey"])
        for f, dt in [("o_orderkey", np.int64), ("o_custkey", np.int32), ("o_orderdate", np.int32),
                      ("o_shippriority", np.int32), ("o_totalprice", np.int64)]:
            if f in o:
                put(f, o[f], dt)
    c = t.get("customer")
    if c is not None:
        T.n_customer = put("c_custkey", c["c_custkey"], np.int32)
        put("c_mktsegment", c["c_mktsegment"], np.uint8)
    p = t.get("part")
    if p is not None:
        T.n_part = put("p_partkey", p["p_partkey"], np.int32)
        put("p_name_offsets", p["p_name_offsets"], np.int64)
        chars = _c(p["p_name_chars"], np.uint8)
        if len(chars) == 0:
            chars = np.zeros(1, np.uint8)
        keep.append(chars)
        T.p_name_chars = chars.ctypes.data
    ps = t.get("partsupp")
    if ps is not None:
        T.n_partsupp = put("ps_partkey", ps["ps_partkey"], np.int32)
        put("ps_suppkey", ps["ps_suppkey"], np.int32)
        put("ps_supplycost", ps["ps_supplycost"], np.int64)
    s = t.get("supplier")
    if s is not None:
        T.n_supplier = put("s_suppkey", s["s_suppkey"], np.int32)
        put("s_nationkey", s["s_nationkey"], np.int32)
    return T, keep


def c_name(custkey: int) -> str:
    return "Customer#%09d" % custkey


def run_query(q: str, tables: dict, params: Params | None = None, limit: int | None = None) -> list:
    L = lib()
    T, keep = make_tables(tables)
    P = params or default_params()
    if q == "q1":
        out = (Q1Row * 64)()
        n = L.or_q1(C.byref(T), C.byref(P), out, 64)
        return [(chr(r.returnflag), chr(r.linestatus), i128_to_int(r.sum_qty), i128_to_int(r.sum_base_price),
                 i128_to_int(r.sum_disc_price), i128_to_int(r.sum_charge), r.avg_qty, r.avg_price, r.avg_disc,
                 r.count_order) for r in out[:n]]
    if q == "q6":
        out = Q6Row()
        L.or_q6(C.byref(T), C.byref(P), C.byref(out))
        return [(None if out.is_null else i128_to_int(out.revenue),)]
    if q == "q3":
        lim = 10 if limit is None else limit
        cap = max(lim, 0) if lim >= 0 else max(T.n_orders, 1)
        out = (Q3Row * max(cap, 1))()
        n = L.or_q3(C.byref(T), C.byref(P), lim, out, cap)
        assert n >= 0
        return [(r.l_orderkey, i128_to_int(r.revenue), r.o_orderdate, r.o_shippriority) for r in out[:n]]
    if q == "q9":
        out = (Q9Row * 4096)()
        n = L.or_q9(C.byref(T), C.byref(P), out, 4096)
        assert n >= 0
        return [(NATIONS[r.nationkey], r.o_year, i128_to_int(r.sum_profit)) for r in out[:n]]
    if q == "q18":
        lim = 100 if limit is None else limit
        cap = lim if lim >= 0 else max(T.n_orders, 1)
        out = (Q18Row * max(cap, 1))()
        n = L.or_q18(C.byref(T), C.byref(P), lim, out, cap)
        assert n >= 0
        return [(c_name(r.c_custkey), r.c_custkey, r.o_orderkey, r.o_orderdate, r.o_totalprice,
                 i128_to_int(r.sum_qty)) for r in out[:n]]
    raise ValueError(q)


# ---------------------------------------------------------------- operator oracles
def _ptrs(cols):
    arrs = [_c(c, np.int64) for c in cols]
    ptrs = (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])
    return arrs, ptrs


def filter(cols, preds) -> np.ndarray:
    """preds: list of (col, op_name, lo[, hi]). Returns ascending int32 row ids."""
    arrs, ptrs = _ptrs(cols)
    n = len(arrs[0]) if arrs else 0
    P = (Pred * max(len(preds), 1))(*[Pred(p[0], OPS[p[1]], p[2], p[3] if len(p) > 3 else 0) for p in preds])
    out = np.empty(max(n, 1), np.int32)
    k = lib().or_filter(n, ptrs, P, len(preds), out.ctypes.data)
    return out[:k]


def contains(offsets, chars, pattern: bytes) -> np.ndarray:
    off = _c(offsets, np.int64)
    ch = _c(chars, np.uint8)
    if len(ch) == 0:
        ch = np.zeros(1, np.uint8)
    n = len(off) - 1
    out = np.empty(max(n, 1), np.int32)
    k = lib().or_contains(n, off.ctypes.data, ch.ctypes.data, pattern, len(pattern), out.ctypes.data)
    return out[:k]


def make_expr(terms) -> Expr:
    """terms: list of (coef, [(col, mul, add), ...]) with <= 2 terms of <= 3 factors."""
    e = Expr()
    e.nterms = len(terms)
    for i, (coef, fs) in enumerate(terms):
        e.t[i].coef = coef
        e.t[i].nf = len(fs)
        for j, (col, mul, add) in enumerate(fs):
            e.t[i].f[j] = Factor(col, mul, add)
    return e


def eval_expr(cols, terms) -> list:
    arrs, ptrs = _ptrs(cols)
    n = len(arrs[0])
    out = (I128 * max(n, 1))()
    lib().or_eval_expr(n, ptrs, C.byref(make_expr(terms)), out)
    return [i128_to_int(v) for v in out[:n]]


def join(build_keys, probe_keys, jtype: str):
    """Returns (probe_idx, build_idx) for inner (probe-major), probe_idx for semi/anti."""
    b = _c(build_keys, np.int64)
    p = _c(probe_keys, np.int64)
    t = {"inner": 0, "semi": 1, "anti": 2}[jtype]
    mult = int(np.unique(b, return_counts=True)[1].max()) if len(b) else 1  # pairs <= probes x max multiplicity
    cap = len(p) if t else max(1, len(p) * mult)
    cap = max(cap, 1)
    op = np.empty(cap, np.int32)
    ob = np.empty(cap, np.int32)
    k = lib().or_join(len(b), b.ctypes.data, len(p), p.ctypes.data, t, op.ctypes.data, ob.ctypes.data, cap)
    assert k >= 0
    return (op[:k], ob[:k]) if t == 0 else op[:k]


def groupby(cols, key_cols, aggs):
    """aggs: list of (op_name, terms, avg_scale).  Returns list of rows sorted by key:
    (*keys, *agg values) with avg as float, others as int."""
    arrs, ptrs = _ptrs(cols)
    n = len(arrs[0]) if arrs else 0
    na = len(aggs)
    kc = (C.c_int32 * max(len(key_cols), 1))(*key_cols)
    ops = (C.c_int32 * max(na, 1))(*[AGGS[a[0]] for a in aggs])
    exprs = (Expr * max(na, 1))(*[make_expr(a[1]) for a in aggs])
    scales = (C.c_int32 * max(na, 1))(*[a[2] if len(a) > 2 else 0 for a in aggs])
    cap = max(n, 1)
    ok = [np.empty(cap, np.int64) for _ in key_cols]
    oa = [(I128 * cap)() for _ in aggs]
    oavg = [np.zeros(cap, np.float64) for _ in aggs]
    pk = (C.c_void_p * max(len(ok), 1))(*[a.ctypes.data for a in ok])
    pa = (C.c_void_p * max(na, 1))(*[C.addressof(a) for a in oa])
    pv = (C.c_void_p * max(na, 1))(*[a.ctypes.data for a in oavg])
    g = lib().or_groupby(n, ptrs, len(key_cols), kc, na, ops, exprs, scales, pk, pa, pv, cap)
    assert g >= 0
    rows = []
    for i in range(g):
        vals = []
        for a in range(na):
            vals.append(float(oavg[a][i]) if aggs[a][0] == "avg" else i128_to_int(oa[a][i]))
        rows.append(tuple(int(k[i]) for k in ok) + tuple(vals))
    return rows


def sort(keys, desc, k: int = -1) -> np.ndarray:
    """keys: list of integer sequences (any Python ints within int128); stable permutation (prefix k)."""
    n = len(keys[0]) if keys else 0
    arrs = []
    for col in keys:
        a = (I128 * max(n, 1))()
        for i, v in enumerate(col):
            a[i] = int_to_i128(int(v))
        arrs.append(a)
    ptrs = (C.c_void_p * max(len(arrs), 1))(*[C.addressof(a) for a in arrs])
    d = (C.c_int32 * max(len(desc), 1))(*desc)
    out = np.empty(max(n, 1), np.int32)
    m = lib().or_sort(n, ptrs, len(keys), d, k, out.ctypes.data)
    return out[:m]


def civil_year(days: int) -> int:
    return lib().or_civil_year(days)


# ---------------------------------------------------------------------------- operator µbenchmarks
class JoinSummary(C.Structure):
    _fields_ = [("count", C.c_int64), ("sum_build", I128), ("sum_probe", I128), ("pair_hash", C.c_uint64)]


def _summary(s: JoinSummary) -> dict:
    return {"count": int(s.count), "sum_build": i128_to_int(s.sum_build), "sum_probe": i128_to_int(s.sum_probe),
            "pair_hash": int(s.pair_hash)}


def unmix64(z: int) -> int:
    return int(lib().or_unmix64(z & (2**64 - 1)))


def pair_mix(b: int, p: int) -> int:
    return int(lib().or_pair_mix(b, p))


def mb_join_closed(nb: int, pkeys: np.ndarray, ppay: np.ndarray) -> dict:
    """Join µbench result summary by the closed form (build rows (mix64(i), i), i < nb)."""
    pk, pp = np.ascontiguousarray(pkeys, np.int64), np.ascontiguousarray(ppay, np.int64)
    s = JoinSummary()
    lib().or_mb_join_closed(nb, len(pk), pk.ctypes.data, pp.ctypes.data, C.byref(s))
    return _summary(s)


def mb_join_hash(bkeys, bpay, pkeys, ppay) -> dict:
    """Join µbench result summary by brute force (std::unordered_multimap)."""
    bk, bp = np.ascontiguousarray(bkeys, np.int64), np.ascontiguousarray(bpay, np.int64)
    pk, pp = np.ascontiguousarray(pkeys, np.int64), np.ascontiguousarray(ppay, np.int64)
    s = JoinSummary()
    lib().or_mb_join_hash(len(bk), bk.ctypes.data, bp.ctypes.data, len(pk), pk.ctypes.data, pp.ctypes.data,
                          C.byref(s))
    return _summary(s)


def mb_groupby_direct(keys, vals, G: int) -> dict:
    """Group-by µbench by direct array over g = mix64^-1(key): {g: (sum, count, min, max)} for present g."""
    k, v = np.ascontiguousarray(keys, np.int64), np.ascontiguousarray(vals, np.int64)
    sm = (I128 * G)()
    cnt = np.zeros(G, np.int64)
    mn = np.zeros(G, np.int64)
    mx = np.zeros(G, np.int64)
    r = lib().or_mb_groupby_direct(len(k), k.ctypes.data, v.ctypes.data, G, sm, cnt.ctypes.data, mn.ctypes.data,
                                   mx.ctypes.data)
    if r < 0:
        raise ValueError("a key is not mix64(g) for g < G")
    return {g: (i128_to_int(sm[g]), int(cnt[g]), int(mn[g]), int(mx[g])) for g in range(G) if cnt[g]}
