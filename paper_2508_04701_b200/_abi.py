"""ctypes mirror of include/sx.h (argument marshalling only; no compute here)."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsx.so")

# sx_status
SX_OK, SX_EINVAL, SX_ETYPE, SX_ENOMEM, SX_EINDEX, SX_EOVERFLOW, SX_EUNSUPPORTED, SX_ECUDA, SX_ENCCL = range(9)
STATUS_NAMES = ["SX_OK", "SX_EINVAL", "SX_ETYPE", "SX_ENOMEM", "SX_EINDEX", "SX_EOVERFLOW", "SX_EUNSUPPORTED",
                "SX_ECUDA", "SX_ENCCL"]
# sx_type
SX_U8, SX_I32, SX_I64, SX_DATE32, SX_DEC64, SX_I128, SX_F64, SX_STR = range(8)
# sx_cmp
SX_LT, SX_LE, SX_GT, SX_GE, SX_EQ, SX_NE, SX_BETWEEN, SX_CONTAINS = range(8)
# sx_aggop
SX_SUM, SX_COUNT, SX_MIN, SX_MAX, SX_AVG = range(5)
SX_KEY_IDENTITY, SX_KEY_YEAR = 0, 1
SX_INNER, SX_SEMI, SX_ANTI = 0, 1, 2
SX_MAX_COLS, SX_MAX_PREDS, SX_MAX_AGGS = 16, 8, 8

_VP = C.c_void_p


class Col(C.Structure):
    _fields_ = [("type", C.c_int32), ("scale", C.c_int32), ("len", C.c_int64), ("data", _VP),
                ("offsets", _VP), ("validity", _VP)]


class Sel(C.Structure):
    _fields_ = [("len", C.c_int64), ("idx", _VP)]


class Factor(C.Structure):
    _fields_ = [("col", C.c_int32), ("pad", C.c_int32), ("mul", C.c_int64), ("add", C.c_int64)]


class Term(C.Structure):
    _fields_ = [("coef", C.c_int64), ("nf", C.c_int32), ("pad", C.c_int32), ("f", Factor * 3)]


class Expr(C.Structure):
    _fields_ = [("nterms", C.c_int32), ("pad", C.c_int32), ("t", Term * 2)]


class Pred(C.Structure):
    _fields_ = [("col", C.c_int32), ("op", C.c_int32), ("lo", C.c_int64), ("hi", C.c_int64),
                ("pattern", C.c_char_p), ("pattern_len", C.c_int32), ("pad", C.c_int32)]


class Agg(C.Structure):
    _fields_ = [("op", C.c_int32), ("scale", C.c_int32), ("value", Expr)]


class Key(C.Structure):
    _fields_ = [("col", C.c_int32), ("fn", C.c_int32)]


class Having(C.Structure):
    _fields_ = [("agg", C.c_int32), ("op", C.c_int32), ("lo", C.c_int64), ("hi", C.c_int64)]


class SortKey(C.Structure):
    _fields_ = [("col", C.c_int32), ("desc", C.c_int32)]


TPCH_COLS = ["l_orderkey", "l_partkey", "l_suppkey", "l_quantity", "l_extendedprice", "l_discount", "l_tax",
             "l_returnflag", "l_linestatus", "l_shipdate", "o_orderkey", "o_custkey", "o_orderdate",
             "o_shippriority", "o_totalprice", "c_custkey", "c_mktsegment", "p_partkey", "p_name", "ps_partkey",
             "ps_suppkey", "ps_supplycost", "s_suppkey", "s_nationkey"]


class TpchTables(C.Structure):
    _fields_ = [(c, Col) for c in TPCH_COLS]


class TpchParams(C.Structure):
    _fields_ = [("q1_shipdate_max", C.c_int32), ("q3_segment", C.c_int32), ("q3_date", C.c_int32),
                ("q6_date_lo", C.c_int32), ("q6_date_hi", C.c_int32), ("q6_disc_lo", C.c_int64),
                ("q6_disc_hi", C.c_int64), ("q6_qty_lt", C.c_int64), ("q9_color", C.c_char * 16),
                ("q18_qty_gt", C.c_int64), ("q3_limit", C.c_int64), ("q18_limit", C.c_int64)]


class I128(C.Structure):
    _fields_ = [("lo", C.c_uint64), ("hi", C.c_int64)]


class Q1Row(C.Structure):
    _fields_ = [("returnflag", C.c_uint8), ("linestatus", C.c_uint8), ("pad", C.c_uint8 * 6), ("sum_qty", I128),
                ("sum_base_price", I128), ("sum_disc_price", I128), ("sum_charge", I128), ("avg_qty", C.c_double),
                ("avg_price", C.c_double), ("avg_disc", C.c_double), ("count_order", C.c_int64)]


class Q6Row(C.Structure):
    _fields_ = [("revenue", I128), ("is_null", C.c_int32), ("pad", C.c_int32)]


class Q3Row(C.Structure):
    _fields_ = [("l_orderkey", C.c_int64), ("revenue", I128), ("o_orderdate", C.c_int32),
                ("o_shippriority", C.c_int32)]


class Q9Row(C.Structure):
    _fields_ = [("nationkey", C.c_int32), ("o_year", C.c_int32), ("sum_profit", I128)]


class Q18Row(C.Structure):
    _fields_ = [("c_custkey", C.c_int32), ("o_orderdate", C.c_int32), ("o_orderkey", C.c_int64),
                ("o_totalprice", C.c_int64), ("sum_qty", I128)]


# every symbol include/sx.h declares (checked by tests/test_abi.py)
EXPORTS = ["sx_ctx_create", "sx_ctx_destroy", "sx_last_error", "sx_free", "sx_sync", "sx_memcpy", "sx_profile_enable",
           "sx_profile_read", "sx_launch_count", "sx_filter", "sx_groupby_agg", "sx_hash_build", "sx_hash_probe", "sx_ht_rows",
           "sx_ht_destroy", "sx_sort_topk", "sx_gather", "sx_tpch_default_params", "sx_tpch_q1", "sx_tpch_q6",
           "sx_tpch_q3", "sx_tpch_q9", "sx_tpch_q18", "sx_groupby_merge", "sx_avg", "sx_dest_rank",
           "sx_partition_by_rank", "sx_comm_unique_id", "sx_comm_init", "sx_comm_destroy", "sx_comm_rank",
           "sx_comm_size", "sx_shuffle", "sx_allgather", "sx_radix_of", "sx_radix_partition", "sx_hash_join",
           "sx_tpch_upload", "sx_tpch_tables_free"]


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise RuntimeError(f"libsx.so not found at {path}: build it with `make sx` "
                           "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(path)
    P = C.POINTER
    vp, i32, i64 = _VP, C.c_int, C.c_int64
    L.sx_ctx_create.argtypes = [i32, vp, P(vp)]
    L.sx_ctx_destroy.argtypes = [vp]
    L.sx_ctx_destroy.restype = None
    L.sx_last_error.argtypes = [vp]
    L.sx_last_error.restype = C.c_char_p
    L.sx_free.argtypes = [vp, vp]
    L.sx_sync.argtypes = [vp]
    L.sx_memcpy.argtypes = [vp, vp, vp, C.c_size_t]
    L.sx_profile_enable.argtypes = [vp, i32]
    L.sx_launch_count.argtypes = [vp, i32]
    L.sx_launch_count.restype = i64
    L.sx_profile_read.argtypes = [vp, vp, vp, vp, i32, P(C.c_int)]
    L.sx_filter.argtypes = [vp, P(Col), i32, P(Pred), i32, P(Sel), vp, i32, P(Sel), P(Col)]
    L.sx_groupby_agg.argtypes = [vp, P(Col), i32, P(Key), i32, P(Sel), P(Pred), i32, P(Agg), i32, P(Having), i64,
                                 P(Col), P(Col), P(C.c_int64)]
    L.sx_hash_build.argtypes = [vp, P(Col), i32, vp, i32, P(Sel), P(Pred), i32, i32, P(vp)]
    L.sx_hash_probe.argtypes = [vp, vp, P(Col), i32, vp, i32, P(Sel), P(Pred), i32, i32, P(Col), i32, vp, i32, vp,
                                i32, P(Sel), P(Sel), P(Col)]
    L.sx_ht_rows.argtypes = [vp]
    L.sx_ht_rows.restype = i64
    L.sx_ht_destroy.argtypes = [vp, vp]
    L.sx_ht_destroy.restype = None
    L.sx_sort_topk.argtypes = [vp, P(Col), i32, P(SortKey), i32, P(Sel), i64, P(Sel)]
    L.sx_gather.argtypes = [vp, P(Col), P(Sel), P(Col)]
    L.sx_tpch_default_params.argtypes = [P(TpchParams)]
    L.sx_tpch_default_params.restype = None
    for q, row in (("q1", Q1Row), ("q3", Q3Row), ("q9", Q9Row), ("q18", Q18Row)):
        getattr(L, f"sx_tpch_{q}").argtypes = [vp, P(TpchTables), P(TpchParams), P(row), i64, P(C.c_int64)]
    L.sx_tpch_q6.argtypes = [vp, P(TpchTables), P(TpchParams), P(Q6Row), P(C.c_int64)]
    L.sx_groupby_merge.argtypes = [vp, P(Col), i32, P(Col), vp, i32, P(Having), i64, P(Col), P(Col), P(C.c_int64)]
    L.sx_avg.argtypes = [vp, P(Col), P(Col), i32, P(Col)]
    L.sx_dest_rank.argtypes = [C.c_uint64, i32]
    L.sx_dest_rank.restype = i32
    L.sx_partition_by_rank.argtypes = [vp, P(Col), i32, vp, i32, P(Sel), i32, P(Col), vp]
    L.sx_comm_unique_id.argtypes = [vp]
    L.sx_comm_init.argtypes = [vp, vp, i32, i32, P(vp)]
    L.sx_comm_destroy.argtypes = [vp]
    L.sx_comm_destroy.restype = None
    L.sx_comm_rank.argtypes = [vp]
    L.sx_comm_size.argtypes = [vp]
    L.sx_shuffle.argtypes = [vp, vp, P(Col), i32, vp, i32, P(Sel), P(Col), P(C.c_int64)]
    L.sx_allgather.argtypes = [vp, vp, P(Col), i32, P(Col), P(C.c_int64)]
    L.sx_tpch_upload.argtypes = [vp, P(TpchTables), P(TpchTables)]
    L.sx_tpch_tables_free.argtypes = [vp, P(TpchTables)]
    L.sx_tpch_tables_free.restype = None
    L.sx_radix_of.argtypes = [C.c_uint64, i32]
    L.sx_radix_of.restype = C.c_uint32
    L.sx_radix_partition.argtypes = [vp, P(Col), i32, vp, i32, P(Sel), i32, P(Col), P(Sel), vp]
    L.sx_hash_join.argtypes = [vp, P(Col), i32, vp, P(Sel), i32, P(Col), i32, vp, P(Sel), i32, i32, vp, i32, vp, i32,
                               i32, P(Sel), P(Sel), P(Col), P(C.c_int)]
    return L
