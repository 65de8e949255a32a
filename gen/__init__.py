"""Seeded TPC-H-shaped generator (shared by the CUDA path and the oracle).

Thin ctypes wrapper over ``gen/libsxgen.so`` (host fill) and
``gen/libsxgen_gpu.so`` (device fill).  Holds none of the method's
arithmetic: it only defines table contents (recipe in
DESIGN.md "Input recipe").

Tables are returned as ``{table: {column: array}}`` with numpy arrays (host) or
torch tensors (device).  ``sf_milli`` is the scale factor x 1000.  A shard
``(rank, world)`` generates a contiguous key range of every table, and of
orders (with their lineitems), so the union of all shards equals the world=1
tables row for row.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_cpu = None
_gpu = None

NATIONS = [
    "ALGERIA", "ARGENTINA", "BRAZIL", "CANADA", "EGYPT", "ETHIOPIA", "FRANCE", "GERMANY",
    "INDIA", "INDONESIA", "IRAN", "IRAQ", "JAPAN", "JORDAN", "KENYA", "MOROCCO",
    "MOZAMBIQUE", "PERU", "CHINA", "ROMANIA", "SAUDI ARABIA", "VIETNAM", "RUSSIA",
    "UNITED KINGDOM", "UNITED STATES",
]
SEGMENTS = ["AUTOMOBILE", "BUILDING", "FURNITURE", "MACHINERY", "HOUSEHOLD"]

LINEITEM_COLS = [
    ("l_orderkey", None), ("l_partkey", np.int32), ("l_suppkey", np.int32), ("l_quantity", np.int64),
    ("l_extendedprice", np.int64), ("l_discount", np.int64), ("l_tax", np.int64), ("l_returnflag", np.uint8),
    ("l_linestatus", np.uint8), ("l_shipdate", np.int32),
]
ORDERS_COLS = [
    ("o_orderkey", None), ("o_custkey", np.int32), ("o_orderdate", np.int32), ("o_shippriority", np.int32),
    ("o_totalprice", np.int64),
]


def sf_to_milli(sf: float) -> int:
    m = int(round(sf * 1000))
    if m <= 0 or abs(m - sf * 1000) > 1e-6:
        raise ValueError(f"scale factor {sf} is not a multiple of 0.001")
    return m


def cpu_lib():
    global _cpu
    if _cpu is None:
        path = os.path.join(_HERE, "libsxgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make gen` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        i64, u64, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        lib.sxg_cpu_sizes.argtypes = [i64, vp]
        lib.sxg_cpu_fill_supplier.argtypes = [u64, i64, i64, vp, vp]
        lib.sxg_cpu_fill_customer.argtypes = [u64, i64, i64, vp, vp, vp]
        lib.sxg_cpu_part_name_bytes.argtypes = [u64, i64, i64]
        lib.sxg_cpu_part_name_bytes.restype = i64
        lib.sxg_cpu_fill_part.argtypes = [u64, i64, i64, vp, vp, vp, vp]
        lib.sxg_cpu_fill_partsupp.argtypes = [u64, i64, i64, i64, vp, vp, vp]
        lib.sxg_cpu_lineitem_count.argtypes = [u64, i64, i64]
        lib.sxg_cpu_lineitem_count.restype = i64
        lib.sxg_cpu_fill_orders_lineitem.argtypes = [u64, i64, i64, i64, ctypes.c_int] + [vp] * 15
        lib.sxg_cpu_word.argtypes = [ctypes.c_int]
        lib.sxg_cpu_word.restype = ctypes.c_char_p
        _cpu = lib
    return _cpu


def sizes(sf_milli: int) -> dict:
    out = np.zeros(5, dtype=np.int64)
    cpu_lib().sxg_cpu_sizes(sf_milli, out.ctypes.data)
    return dict(zip(["supplier", "customer", "part", "partsupp", "orders"], (int(x) for x in out)))


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """1-based half-open key range [k0, k1) of shard `rank` of `world` over keys 1..n."""
    return 1 + (n * rank) // world, 1 + (n * (rank + 1)) // world


def key_bytes_for(sf_milli: int) -> int:
    """orderkey width: int32 while max orderkey < 2^31 (SF <= ~357), else int64 (SURVEY §8 header)."""
    n = sizes(sf_milli)["orders"]
    max_key = ((n >> 3) << 5) | 7
    return 4 if max_key < 2**31 else 8


def _p(a):
    return None if a is None else a.ctypes.data


TABLES = ("lineitem", "orders", "customer", "part", "partsupp", "supplier")


def cpu_tables(sf_milli: int, seed: int = 42, shard=(0, 1), tables=TABLES, key_bytes: int | None = None) -> dict:
    """Generate tables into host numpy arrays."""
    lib = cpu_lib()
    sz = sizes(sf_milli)
    rank, world = shard
    kb = key_bytes or key_bytes_for(sf_milli)
    kdt = np.int32 if kb == 4 else np.int64
    out = {}
    if "supplier" in tables:
        k0, k1 = shard_range(sz["supplier"], rank, world)
        t = {"s_suppkey": np.empty(k1 - k0, np.int32), "s_nationkey": np.empty(k1 - k0, np.int32)}
        lib.sxg_cpu_fill_supplier(seed, k0, k1, _p(t["s_suppkey"]), _p(t["s_nationkey"]))
        out["supplier"] = t
    if "customer" in tables:
        k0, k1 = shard_range(sz["customer"], rank, world)
        t = {"c_custkey": np.empty(k1 - k0, np.int32), "c_mktsegment": np.empty(k1 - k0, np.uint8)}
        lib.sxg_cpu_fill_customer(seed, k0, k1, _p(t["c_custkey"]), _p(t["c_mktsegment"]), None)
        out["customer"] = t
    if "part" in tables:
        k0, k1 = shard_range(sz["part"], rank, world)
        nbytes = lib.sxg_cpu_part_name_bytes(seed, k0, k1)
        t = {"p_partkey": np.empty(k1 - k0, np.int32), "p_name_offsets": np.empty(k1 - k0 + 1, np.int64),
             "p_name_chars": np.empty(max(nbytes, 1), np.uint8)}
        lib.sxg_cpu_fill_part(seed, k0, k1, _p(t["p_partkey"]), _p(t["p_name_offsets"]), _p(t["p_name_chars"]), None)
        t["p_name_chars"] = t["p_name_chars"][:nbytes]
        out["part"] = t
    if "partsupp" in tables:
        p0, p1 = shard_range(sz["part"], rank, world)
        n = 4 * (p1 - p0)
        t = {"ps_partkey": np.empty(n, np.int32), "ps_suppkey": np.empty(n, np.int32),
             "ps_supplycost": np.empty(n, np.int64)}
        lib.sxg_cpu_fill_partsupp(seed, sf_milli, p0, p1, _p(t["ps_partkey"]), _p(t["ps_suppkey"]),
                                  _p(t["ps_supplycost"]))
        out["partsupp"] = t
    if "orders" in tables or "lineitem" in tables:
        i0, i1 = shard_range(sz["orders"], rank, world)
        nl = lib.sxg_cpu_lineitem_count(seed, i0, i1)
        o = {c: np.empty(i1 - i0, dt or kdt) for c, dt in ORDERS_COLS}
        li = {c: np.empty(nl, dt or kdt) for c, dt in LINEITEM_COLS}
        lib.sxg_cpu_fill_orders_lineitem(seed, sf_milli, i0, i1, kb, *[_p(o[c]) for c, _ in ORDERS_COLS],
                                         *[_p(li[c]) for c, _ in LINEITEM_COLS])
        if "orders" in tables:
            out["orders"] = o
        if "lineitem" in tables:
            out["lineitem"] = li
    return out


def gpu_lib():
    global _gpu
    if _gpu is None:
        path = os.path.join(_HERE, "libsxgen_gpu.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make gen` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        i64, u64, vp, ci = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
        lib.sxg_gpu_fill_supplier.argtypes = [u64, i64, i64, vp, vp, vp]
        lib.sxg_gpu_fill_customer.argtypes = [u64, i64, i64, vp, vp, vp, vp]
        lib.sxg_gpu_part_offsets.argtypes = [u64, i64, i64, vp, vp, vp]
        lib.sxg_gpu_fill_part.argtypes = [u64, i64, i64, vp, vp, vp, vp, vp]
        lib.sxg_gpu_fill_partsupp.argtypes = [u64, i64, i64, i64, vp, vp, vp, vp]
        lib.sxg_gpu_line_offsets.argtypes = [u64, i64, i64, vp, vp, vp]
        lib.sxg_gpu_fill_orders_lineitem.argtypes = [u64, i64, i64, i64, ci, vp] + [vp] * 15 + [vp]
        for f in ("sxg_gpu_fill_supplier", "sxg_gpu_fill_customer", "sxg_gpu_part_offsets", "sxg_gpu_fill_part",
                  "sxg_gpu_fill_partsupp", "sxg_gpu_line_offsets", "sxg_gpu_fill_orders_lineitem"):
            getattr(lib, f).restype = ci
        _gpu = lib
    return _gpu


def gpu_tables(sf_milli: int, seed: int = 42, shard=(0, 1), tables=TABLES, device="cuda",
               key_bytes: int | None = None) -> dict:
    """Generate tables straight into device memory (torch tensors on `device`)."""
    import torch

    lib = gpu_lib()
    sz = sizes(sf_milli)
    rank, world = shard
    kb = key_bytes or key_bytes_for(sf_milli)
    kdt = torch.int32 if kb == 4 else torch.int64
    tdt = {np.int32: torch.int32, np.int64: torch.int64, np.uint8: torch.uint8}
    stream = torch.cuda.current_stream(device).cuda_stream

    def emp(n, dt):
        return torch.empty(max(int(n), 0), dtype=dt, device=device)

    def ptr(t):
        return None if t is None else t.data_ptr()

    def chk(rc):
        if rc != 0:
            raise RuntimeError(f"generator CUDA error {rc}")

    out = {}
    if "supplier" in tables:
        k0, k1 = shard_range(sz["supplier"], rank, world)
        t = {"s_suppkey": emp(k1 - k0, torch.int32), "s_nationkey": emp(k1 - k0, torch.int32)}
        chk(lib.sxg_gpu_fill_supplier(seed, k0, k1, ptr(t["s_suppkey"]), ptr(t["s_nationkey"]), stream))
        out["supplier"] = t
    if "customer" in tables:
        k0, k1 = shard_range(sz["customer"], rank, world)
        t = {"c_custkey": emp(k1 - k0, torch.int32), "c_mktsegment": emp(k1 - k0, torch.uint8)}
        chk(lib.sxg_gpu_fill_customer(seed, k0, k1, ptr(t["c_custkey"]), ptr(t["c_mktsegment"]), None, stream))
        out["customer"] = t
    if "part" in tables:
        k0, k1 = shard_range(sz["part"], rank, world)
        n = k1 - k0
        offs = emp(n + 1, torch.int64)
        tmp = emp(n // 1024 + 2, torch.int64)
        chk(lib.sxg_gpu_part_offsets(seed, k0, k1, ptr(offs), ptr(tmp), stream))
        nbytes = int(offs[n].item())
        t = {"p_partkey": emp(n, torch.int32), "p_name_offsets": offs, "p_name_chars": emp(nbytes, torch.uint8)}
        chk(lib.sxg_gpu_fill_part(seed, k0, k1, ptr(t["p_partkey"]), ptr(offs), ptr(t["p_name_chars"]), None, stream))
        out["part"] = t
    if "partsupp" in tables:
        p0, p1 = shard_range(sz["part"], rank, world)
        n = 4 * (p1 - p0)
        t = {"ps_partkey": emp(n, torch.int32), "ps_suppkey": emp(n, torch.int32),
             "ps_supplycost": emp(n, torch.int64)}
        chk(lib.sxg_gpu_fill_partsupp(seed, sf_milli, p0, p1, ptr(t["ps_partkey"]), ptr(t["ps_suppkey"]),
                                      ptr(t["ps_supplycost"]), stream))
        out["partsupp"] = t
    if "orders" in tables or "lineitem" in tables:
        i0, i1 = shard_range(sz["orders"], rank, world)
        n = i1 - i0
        offs = emp(n + 1, torch.int64)
        tmp = emp(n // 1024 + 2, torch.int64)
        chk(lib.sxg_gpu_line_offsets(seed, i0, i1, ptr(offs), ptr(tmp), stream))
        nl = int(offs[n].item())
        o = {c: emp(n, tdt.get(dt, kdt) if dt else kdt) for c, dt in ORDERS_COLS} if "orders" in tables else {}
        li = {c: emp(nl, tdt.get(dt, kdt) if dt else kdt) for c, dt in LINEITEM_COLS} if "lineitem" in tables else {}
        chk(lib.sxg_gpu_fill_orders_lineitem(seed, sf_milli, i0, i1, kb, ptr(offs),
                                             *[ptr(o.get(c)) for c, _ in ORDERS_COLS],
                                             *[ptr(li.get(c)) for c, _ in LINEITEM_COLS], stream))
        del offs, tmp
        if "orders" in tables:
            out["orders"] = o
        if "lineitem" in tables:
            out["lineitem"] = li
    torch.cuda.current_stream(device).synchronize()
    return out


def to_device(tables: dict, device="cuda") -> dict:
    import torch

    return {t: {c: torch.from_numpy(np.ascontiguousarray(a)).to(device) for c, a in cols.items()}
            for t, cols in tables.items()}


# ---------------------------------------------------------------------------- operator µbenchmarks
# C5a join (build 2^27 int64 key mix64(i) + payload i; probe keys from a uniform
# or Zipf(1.0) rank through an affine permutation, payload j), C5b group-by sweep (int64 key
# mix64(g), g ~ U[0, G); DEC64 value), and our sort µbench (uniform int64 keys + int32 payload).
# Readings R15-R17.  Host arrays (numpy) or device tensors; rows [r0, r1) of the
# infinite counter-based stream, so shards are contiguous row ranges.

def _mb_cpu():
    lib = cpu_lib()
    if not hasattr(lib, "_mb_ready"):
        i64, u64, vp, ci = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
        lib.sxg_cpu_fill_mb_build.argtypes = [i64, i64, vp, vp]
        lib.sxg_cpu_fill_mb_probe.argtypes = [u64, i64, ci, i64, i64, vp, vp]
        lib.sxg_cpu_fill_mb_groupby.argtypes = [u64, i64, i64, i64, vp, vp]
        lib.sxg_cpu_fill_mb_sort.argtypes = [u64, i64, i64, vp, vp]
        lib.sxg_cpu_mb_probe_rank.argtypes = [u64, i64, i64, ci]
        lib.sxg_cpu_mb_probe_rank.restype = i64
        lib._mb_ready = True
    return lib


def _mb_gpu():
    lib = gpu_lib()
    if not hasattr(lib, "_mb_ready"):
        i64, u64, vp, ci = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
        lib.sxg_gpu_fill_mb_build.argtypes = [i64, i64, vp, vp, vp]
        lib.sxg_gpu_fill_mb_probe.argtypes = [u64, i64, ci, i64, i64, vp, vp, vp]
        lib.sxg_gpu_fill_mb_groupby.argtypes = [u64, i64, i64, i64, vp, vp, vp]
        lib.sxg_gpu_fill_mb_sort.argtypes = [u64, i64, i64, vp, vp, vp]
        for f in ("sxg_gpu_fill_mb_build", "sxg_gpu_fill_mb_probe", "sxg_gpu_fill_mb_groupby", "sxg_gpu_fill_mb_sort"):
            getattr(lib, f).restype = ci
        lib._mb_ready = True
    return lib


def _mb_arrays(n, dtypes, device):
    if device is None:
        return [np.empty(int(n), dtype=d) for d in dtypes]
    import torch

    tm = {np.int64: torch.int64, np.int32: torch.int32}
    return [torch.empty(int(n), dtype=tm[d], device=device) for d in dtypes]


def _mb_ptr(a):
    return a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr()


def _mb_call(device, cpu_fn, gpu_fn, args, outs):
    if device is None:
        getattr(_mb_cpu(), cpu_fn)(*args, *[_mb_ptr(o) for o in outs])
    else:
        import torch

        rc = getattr(_mb_gpu(), gpu_fn)(*args, *[_mb_ptr(o) for o in outs], torch.cuda.current_stream(device).cuda_stream)
        if rc != 0:
            raise RuntimeError(f"generator CUDA error {rc}")
        torch.cuda.current_stream(device).synchronize()
    return outs


def mb_join_build(nb: int, r0: int = 0, r1: int | None = None, device=None):
    """Build side rows [r0, r1): (key int64 = mix64(i), payload int64 = i)."""
    r1 = nb if r1 is None else r1
    outs = _mb_arrays(r1 - r0, [np.int64, np.int64], device)
    return _mb_call(device, "sxg_cpu_fill_mb_build", "sxg_gpu_fill_mb_build", (r0, r1), outs)


def mb_join_probe(nb: int, nprobe: int, zipf: bool, seed: int = 42, r0: int = 0, r1: int | None = None, device=None):
    """Probe side rows [r0, r1): (key int64, payload int64 = j); nb a power of two."""
    assert nb >= 2 and nb & (nb - 1) == 0
    r1 = nprobe if r1 is None else r1
    outs = _mb_arrays(r1 - r0, [np.int64, np.int64], device)
    return _mb_call(device, "sxg_cpu_fill_mb_probe", "sxg_gpu_fill_mb_probe", (seed, nb, 1 if zipf else 0, r0, r1), outs)


def mb_probe_rank(j: int, nb: int, zipf: bool, seed: int = 42) -> int:
    return int(_mb_cpu().sxg_cpu_mb_probe_rank(seed, j, nb, 1 if zipf else 0))


def mb_groupby(n: int, G: int, seed: int = 42, r0: int = 0, r1: int | None = None, device=None):
    """Rows [r0, r1): (key int64 = mix64(g), value int64 DEC64 scale 2)."""
    r1 = n if r1 is None else r1
    outs = _mb_arrays(r1 - r0, [np.int64, np.int64], device)
    return _mb_call(device, "sxg_cpu_fill_mb_groupby", "sxg_gpu_fill_mb_groupby", (seed, G, r0, r1), outs)


def mb_sort(n: int, seed: int = 42, r0: int = 0, r1: int | None = None, device=None):
    """Rows [r0, r1): (key int64 uniform, payload int32 = i)."""
    r1 = n if r1 is None else r1
    outs = _mb_arrays(r1 - r0, [np.int64, np.int32], device)
    return _mb_call(device, "sxg_cpu_fill_mb_sort", "sxg_gpu_fill_mb_sort", (seed, r0, r1), outs)
