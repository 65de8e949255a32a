"""Test helpers: golden fixtures -> table dicts, canonical comparison."""
from __future__ import annotations

import json
import math
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

_DT = {
    "l_orderkey": np.int64, "l_partkey": np.int32, "l_suppkey": np.int32, "l_quantity": np.int64,
    "l_extendedprice": np.int64, "l_discount": np.int64, "l_tax": np.int64, "l_returnflag": np.uint8,
    "l_linestatus": np.uint8, "l_shipdate": np.int32,
    "o_orderkey": np.int64, "o_custkey": np.int32, "o_orderdate": np.int32, "o_shippriority": np.int32,
    "o_totalprice": np.int64, "c_custkey": np.int32, "c_mktsegment": np.uint8, "p_partkey": np.int32,
    "ps_partkey": np.int32, "ps_suppkey": np.int32, "ps_supplycost": np.int64, "s_suppkey": np.int32,
    "s_nationkey": np.int32,
}
_LI = ["l_orderkey", "l_partkey", "l_suppkey", "l_quantity", "l_extendedprice", "l_discount", "l_tax",
       "l_returnflag", "l_linestatus", "l_shipdate"]
_OR = ["o_orderkey", "o_custkey", "o_orderdate", "o_shippriority", "o_totalprice"]


def load_golden(name: str) -> dict:
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def golden_tables(spec: dict, key_dtype=np.int64) -> dict:
    """JSON table spec -> numpy table dict (gen.cpu_tables layout); missing lineitem/orders columns are 0."""
    out = {}
    for tname, cols in spec.items():
        t = {}
        if tname == "part":
            names = [s.encode() for s in cols["names"]]
            offs = np.zeros(len(names) + 1, np.int64)
            offs[1:] = np.cumsum([len(s) for s in names])
            t["p_partkey"] = np.asarray(cols["p_partkey"], np.int32)
            t["p_name_offsets"] = offs
            t["p_name_chars"] = np.frombuffer(b"".join(names), np.uint8).copy()
        else:
            for c, v in cols.items():
                if c in ("l_returnflag", "l_linestatus"):
                    v = [ord(x) for x in v]
                dt = _DT[c]
                if c in ("l_orderkey", "o_orderkey"):
                    dt = key_dtype
                t[c] = np.asarray(v, dt)
        out[tname] = t
    for tname, names in (("lineitem", _LI), ("orders", _OR)):
        if tname in out:
            n = len(next(iter(out[tname].values())))
            for c in names:
                if c not in out[tname]:
                    dt = key_dtype if c.endswith("orderkey") else _DT[c]
                    out[tname][c] = np.zeros(n, dt)
    return out


def rows_equal(a: list, b: list, rel: float = 1e-9) -> bool:
    """Exact for ints/str/None, relative tolerance for floats (north_star: avg within 1e-9)."""
    if len(a) != len(b):
        return False
    for ra, rb in zip(a, b):
        if len(ra) != len(rb):
            return False
        for x, y in zip(ra, rb):
            if isinstance(x, float) or isinstance(y, float):
                if x is None or y is None or not math.isclose(float(x), float(y), rel_tol=rel, abs_tol=0.0):
                    return False
            elif x != y:
                return False
    return True


def diff_rows(a: list, b: list) -> str:
    lines = [f"len {len(a)} vs {len(b)}"]
    for i, (ra, rb) in enumerate(zip(a, b)):
        if not rows_equal([ra], [rb]):
            lines.append(f"row {i}: {ra} != {rb}")
            if len(lines) > 10:
                break
    return "\n".join(lines)


def np_pair_mix(b: np.ndarray, p: np.ndarray) -> int:
    """Σ (mod 2^64) of the oracle's pair hash (oracle.or_pair_mix) over output pairs, in numpy (test side)."""
    with np.errstate(over="ignore"):
        z = b.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15) ^ p.astype(np.uint64)
        z = (z ^ (z >> np.uint64(32))) * np.uint64(0xD6E8FEB86659FD93)
        z = z ^ (z >> np.uint64(32))
        return int(z.sum(dtype=np.uint64))


def np_fmix64(k: np.ndarray) -> np.ndarray:
    """murmur3 fmix64 (the hash DESIGN.md R14 documents), in numpy (test side)."""
    k = k.astype(np.uint64)
    with np.errstate(over="ignore"):
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xFF51AFD7ED558CCD)
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xC4CEB9FE1A85EC53)
        k ^= k >> np.uint64(33)
    return k
