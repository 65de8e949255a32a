"""sx — B200-native relational hot path of Sirius (arXiv 2508.04701).

Thin Python binding over ``libsx.so`` (include/sx.h): argument marshalling only.
Every operator step runs in the library's sm_100a CUDA kernels; there is no CPU
fallback — importing works anywhere, but creating a ``Ctx`` needs a CUDA device
and the built library, and fails loudly otherwise.

PyTorch supplies device memory (tensors in), streams and process groups; the
library returns its own pool-allocated buffers, which the binding copies into
torch tensors and releases.
"""
from __future__ import annotations

import ctypes as C

from . import _abi as A

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = A.load()
    return _lib


class SxError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{A.STATUS_NAMES[status] if 0 <= status < len(A.STATUS_NAMES) else status}: {msg}")
        self.status = status


_DTYPE_TYPE = {"torch.uint8": A.SX_U8, "torch.int32": A.SX_I32, "torch.int64": A.SX_I64,
               "torch.float64": A.SX_F64}
_TYPE_DTYPE = {}


def _torch():
    import torch

    if not _TYPE_DTYPE:
        _TYPE_DTYPE.update({A.SX_U8: torch.uint8, A.SX_I32: torch.int32, A.SX_DATE32: torch.int32,
                            A.SX_I64: torch.int64, A.SX_DEC64: torch.int64, A.SX_F64: torch.float64,
                            A.SX_I128: torch.int64})
    return torch


def col(t, type: int | None = None, scale: int = 0, offsets=None) -> A.Col:
    """torch CUDA tensor -> sx_col (borrowed).  SX_I128 columns are int64 tensors of shape (n, 2);
    SX_STR columns pass the uint8 chars tensor and an int64 offsets tensor."""
    if type is None:
        type = _DTYPE_TYPE[str(t.dtype)]
    n = t.shape[0] if type != A.SX_STR else offsets.shape[0] - 1
    # sx.h: buffers are dense and 16-byte aligned (the kernels load 16 bytes at a time); a strided or
    # offset view would be misread or fault, so it is rejected here rather than copied silently
    for x in (t, offsets):
        if x is not None and x.numel():
            if not x.is_contiguous():
                raise SxError(A.SX_EINVAL, "column tensor is not contiguous (pass .contiguous())")
            if x.data_ptr() % (8 if x is offsets else (1 if type == A.SX_STR else 16)):
                raise SxError(A.SX_EINVAL, f"column tensor at {x.data_ptr():#x} is not 16-byte aligned (pass .clone())")
    c = A.Col(type, scale, n, t.data_ptr() if t.numel() else None,
              offsets.data_ptr() if offsets is not None else None, None)
    c._keep = (t, offsets)  # the struct borrows the tensors' memory: keep them alive with it
    return c


def expr(terms) -> A.Expr:
    """terms: [(coef, [(col, mul, add), ...]), ...] (<= 2 terms of <= 3 factors)."""
    e = A.Expr()
    e.nterms = len(terms)
    for i, (coef, fs) in enumerate(terms):
        e.t[i].coef = coef
        e.t[i].nf = len(fs)
        for j, (c, m, a) in enumerate(fs):
            e.t[i].f[j] = A.Factor(c, 0, m, a)
    return e


_OPS = {"lt": A.SX_LT, "le": A.SX_LE, "gt": A.SX_GT, "ge": A.SX_GE, "eq": A.SX_EQ, "ne": A.SX_NE,
        "between": A.SX_BETWEEN, "contains": A.SX_CONTAINS}
_AGGS = {"sum": A.SX_SUM, "count": A.SX_COUNT, "min": A.SX_MIN, "max": A.SX_MAX, "avg": A.SX_AVG}
_JOINS = {"inner": A.SX_INNER, "semi": A.SX_SEMI, "anti": A.SX_ANTI}


def preds(ps):
    """[(col, op, lo[, hi])] or (col, 'contains', b'pattern') -> (array, keepalive)."""
    arr = (A.Pred * max(len(ps), 1))()
    keep = []
    for i, p in enumerate(ps):
        if p[1] == "contains":
            pat = p[2] if isinstance(p[2], bytes) else p[2].encode()
            keep.append(pat)
            arr[i] = A.Pred(p[0], A.SX_CONTAINS, 0, 0, pat, len(pat), 0)
        else:
            arr[i] = A.Pred(p[0], _OPS[p[1]], int(p[2]), int(p[3]) if len(p) > 3 else 0, None, 0, 0)
    return arr, keep


class Ctx:
    """One sx_ctx bound to a CUDA device and the current torch stream."""

    def __init__(self, device: int = 0, stream=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise SxError(A.SX_ECUDA, "no CUDA device: libsx has no CPU fallback")
        self.L = lib()
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = C.c_void_p()
        st = self.L.sx_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h))
        if st != A.SX_OK:
            raise SxError(st, "sx_ctx_create failed")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.sx_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st: int):
        if st != A.SX_OK:
            raise SxError(st, self.L.sx_last_error(self.h).decode())

    # --------------------------------------------------------------- buffer helpers
    def take_col(self, c: A.Col):
        """Library-owned output column -> torch tensor (copied), library buffer freed."""
        torch = _torch()
        n = c.len
        if c.type == A.SX_I128:
            t = torch.empty((n, 2), dtype=torch.int64, device=self.device)
        else:
            t = torch.empty(n, dtype=_TYPE_DTYPE[c.type], device=self.device)
        if n:
            self.check(self.L.sx_memcpy(self.h, C.c_void_p(t.data_ptr()), C.c_void_p(c.data), t.numel() * t.element_size()))
        if c.data:
            self.check(self.L.sx_free(self.h, C.c_void_p(c.data)))
        return t

    def take_sel(self, s: A.Sel):
        torch = _torch()
        t = torch.empty(s.len, dtype=torch.int32, device=self.device)
        if s.len:
            self.check(self.L.sx_memcpy(self.h, C.c_void_p(t.data_ptr()), C.c_void_p(s.idx), s.len * 4))
        if s.idx:
            self.check(self.L.sx_free(self.h, C.c_void_p(s.idx)))
        return t

    @staticmethod
    def sel(t) -> A.Sel:
        return A.Sel(t.shape[0], t.data_ptr() if t.numel() else None)

    def sync(self):
        self.check(self.L.sx_sync(self.h))

    # --------------------------------------------------------------- operators
    def filter(self, cols, conj, in_sel=None, gather=()):
        """-> (sel int32 tensor, [gathered tensors])"""
        ca = (A.Col * max(len(cols), 1))(*cols)
        pa, keep = preds(conj)
        g = (C.c_int32 * max(len(gather), 1))(*gather)
        outs = (A.Col * max(len(gather), 1))()
        osel = A.Sel()
        isel = self.sel(in_sel) if in_sel is not None else None
        self.check(self.L.sx_filter(self.h, ca, len(cols), pa, len(conj), C.byref(isel) if isel else None, g,
                                    len(gather), C.byref(osel), outs))
        return self.take_sel(osel), [self.take_col(outs[i]) for i in range(len(gather))]

    def groupby(self, cols, keys, aggs, where=(), in_sel=None, having=None, groups_hint=0, raw=False):
        """keys: [(col, 'id'|'year')]; aggs: [(op, terms, scale)]; having: (agg, op, lo[, hi]).
        -> (key tensors, agg tensors, ngroups); raw=True: the library-owned sx_cols (free_ptr them)."""
        ca = (A.Col * max(len(cols), 1))(*cols)
        ka = (A.Key * max(len(keys), 1))(*[A.Key(c, A.SX_KEY_YEAR if fn == "year" else A.SX_KEY_IDENTITY)
                                           for c, fn in keys])
        aa = (A.Agg * max(len(aggs), 1))(*[A.Agg(_AGGS[a[0]], a[2] if len(a) > 2 else 0, expr(a[1])) for a in aggs])
        pa, keep = preds(where)
        hv = None
        if having is not None:
            hv = A.Having(having[0], _OPS[having[1]], int(having[2]), int(having[3]) if len(having) > 3 else 0)
        ok = (A.Col * 2)()
        oa = (A.Col * max(len(aggs), 1))()
        ng = C.c_int64()
        isel = self.sel(in_sel) if in_sel is not None else None
        self.check(self.L.sx_groupby_agg(self.h, ca, len(cols), ka, len(keys), C.byref(isel) if isel else None, pa,
                                         len(where), aa, len(aggs), C.byref(hv) if hv else None, groups_hint, ok, oa,
                                         C.byref(ng)))
        if raw:
            return [ok[i] for i in range(len(keys))], [oa[i] for i in range(len(aggs))], ng.value
        return [self.take_col(ok[i]) for i in range(len(keys))], [self.take_col(oa[i]) for i in range(len(aggs))], ng.value

    def hash_build(self, cols, key_cols, in_sel=None, where=(), unique=False, membership=False):
        ca = (A.Col * max(len(cols), 1))(*cols)
        kc = (C.c_int32 * len(key_cols))(*key_cols)
        pa, keep = preds(where)
        h = C.c_void_p()
        isel = self.sel(in_sel) if in_sel is not None else None
        self.check(self.L.sx_hash_build(self.h, ca, len(cols), kc, len(key_cols), C.byref(isel) if isel else None, pa,
                                        len(where), (1 if unique else 0) | (2 if membership else 0), C.byref(h)))
        return HashTable(self, h)

    def hash_probe(self, ht, cols, key_cols, jtype, in_sel=None, where=(), build_cols=(), bp=(), pp=()):
        """-> (probe sel, build sel | None, payload tensors)"""
        ca = (A.Col * max(len(cols), 1))(*cols)
        kc = (C.c_int32 * len(key_cols))(*key_cols)
        pa, keep = preds(where)
        ba = (A.Col * max(len(build_cols), 1))(*build_cols)
        bpa = (C.c_int32 * max(len(bp), 1))(*bp)
        ppa = (C.c_int32 * max(len(pp), 1))(*pp)
        op, ob = A.Sel(), A.Sel()
        outs = (A.Col * max(len(bp) + len(pp), 1))()
        isel = self.sel(in_sel) if in_sel is not None else None
        jt = _JOINS[jtype]
        self.check(self.L.sx_hash_probe(self.h, ht.h, ca, len(cols), kc, len(key_cols), C.byref(isel) if isel else None,
                                        pa, len(where), jt, ba, len(build_cols), bpa, len(bp), ppa, len(pp),
                                        C.byref(op), C.byref(ob) if jt == A.SX_INNER else None, outs))
        p = self.take_sel(op)
        b = self.take_sel(ob) if jt == A.SX_INNER else None
        return p, b, [self.take_col(outs[i]) for i in range(len(bp) + len(pp))]

    def sort_topk(self, cols, keys, k=-1, in_sel=None, raw=False):
        """keys: [(col, desc)] -> int32 permutation tensor"""
        ca = (A.Col * max(len(cols), 1))(*cols)
        ks = (A.SortKey * len(keys))(*[A.SortKey(c, 1 if d else 0) for c, d in keys])
        out = A.Sel()
        isel = self.sel(in_sel) if in_sel is not None else None
        self.check(self.L.sx_sort_topk(self.h, ca, len(cols), ks, len(keys), C.byref(isel) if isel else None, k,
                                       C.byref(out)))
        return out if raw else self.take_sel(out)

    def gather(self, c: A.Col, sel_t):
        out = A.Col()
        s = self.sel(sel_t)
        self.check(self.L.sx_gather(self.h, C.byref(c), C.byref(s), C.byref(out)))
        return self.take_col(out)

    def groupby_merge(self, keys, parts, ops, having=None, groups_hint=0):
        """keys/parts: sx_col lists (partials); ops: 'sum'|'count'|'min'|'max' -> (keys, parts, n)"""
        ka = (A.Col * len(keys))(*keys)
        pa = (A.Col * max(len(parts), 1))(*parts)
        oa = (C.c_int32 * max(len(ops), 1))(*[_AGGS[o] for o in ops])
        hv = None
        if having is not None:
            hv = A.Having(having[0], _OPS[having[1]], int(having[2]), int(having[3]) if len(having) > 3 else 0)
        ok = (A.Col * 2)()
        op = (A.Col * max(len(parts), 1))()
        ng = C.c_int64()
        self.check(self.L.sx_groupby_merge(self.h, ka, len(keys), pa, oa, len(parts), C.byref(hv) if hv else None,
                                           groups_hint, ok, op, C.byref(ng)))
        return [self.take_col(ok[i]) for i in range(len(keys))], [self.take_col(op[i]) for i in range(len(parts))], ng.value

    def avg(self, sum_col: A.Col, count_col: A.Col, scale: int):
        out = A.Col()
        self.check(self.L.sx_avg(self.h, C.byref(sum_col), C.byref(count_col), scale, C.byref(out)))
        return self.take_col(out)

    def partition_by_rank(self, cols, key_cols, nranks, in_sel=None):
        """-> (partitioned tensors, counts list)"""
        ca = (A.Col * len(cols))(*cols)
        kc = (C.c_int32 * len(key_cols))(*key_cols)
        outs = (A.Col * len(cols))()
        cnt = (C.c_int64 * nranks)()
        isel = self.sel(in_sel) if in_sel is not None else None
        self.check(self.L.sx_partition_by_rank(self.h, ca, len(cols), kc, len(key_cols), C.byref(isel) if isel else None,
                                               nranks, outs, cnt))
        return [self.take_col(outs[i]) for i in range(len(cols))], [int(x) for x in cnt]

    def radix_partition(self, cols, key_cols, bits, in_sel=None, rows=False):
        """H5 (sx_radix_partition) -> (partitioned tensors, row ids | None, offsets list of 2^bits + 1)"""
        ca = (A.Col * len(cols))(*cols)
        kc = (C.c_int32 * len(key_cols))(*key_cols)
        outs = (A.Col * len(cols))()
        orow = A.Sel()
        offs = (C.c_int64 * ((1 << bits) + 1))()
        isel = self.sel(in_sel) if in_sel is not None else None
        self.check(self.L.sx_radix_partition(self.h, ca, len(cols), kc, len(key_cols), C.byref(isel) if isel else None,
                                             bits, outs, C.byref(orow) if rows else None, offs))
        r = self.take_sel(orow) if rows else None
        return [self.take_col(outs[i]) for i in range(len(cols))], r, [int(x) for x in offs]

    def hash_join(self, build_cols, build_keys, probe_cols, probe_keys, jtype="inner", unique=True, bp=(), pp=(),
                  strategy=0, build_sel=None, probe_sel=None, rows=(True, True), raw=False):
        """Build + probe (sx_hash_join).  -> (probe sel | None, build sel | None, payloads, strategy used).
        raw=True returns the library-owned sx_sel / sx_col structs (free them with free_ptr)."""
        ba = (A.Col * len(build_cols))(*build_cols)
        pa = (A.Col * len(probe_cols))(*probe_cols)
        bk = (C.c_int32 * len(build_keys))(*build_keys)
        pk = (C.c_int32 * len(probe_keys))(*probe_keys)
        bpa = (C.c_int32 * max(len(bp), 1))(*bp)
        ppa = (C.c_int32 * max(len(pp), 1))(*pp)
        op, ob = A.Sel(), A.Sel()
        outs = (A.Col * max(len(bp) + len(pp), 1))()
        used = C.c_int()
        bs = self.sel(build_sel) if build_sel is not None else None
        ps = self.sel(probe_sel) if probe_sel is not None else None
        jt = _JOINS[jtype]
        self.check(self.L.sx_hash_join(self.h, ba, len(build_cols), bk, C.byref(bs) if bs else None, 1 if unique else 0,
                                       pa, len(probe_cols), pk, C.byref(ps) if ps else None, len(build_keys), jt,
                                       bpa, len(bp), ppa, len(pp), strategy,
                                       C.byref(op) if rows[0] else None,
                                       C.byref(ob) if (rows[1] and jt == A.SX_INNER) else None, outs, C.byref(used)))
        npay = len(bp) + len(pp)
        if raw:
            return (op if rows[0] else None), (ob if rows[1] and jt == A.SX_INNER else None), \
                [outs[i] for i in range(npay)], used.value
        p = self.take_sel(op) if rows[0] else None
        b = self.take_sel(ob) if (rows[1] and jt == A.SX_INNER) else None
        return p, b, [self.take_col(outs[i]) for i in range(npay)], used.value

    def free_ptr(self, p):
        if p:
            self.check(self.L.sx_free(self.h, C.c_void_p(p)))

    def copy_into(self, dst, dst_off: int, src, n: int):
        """dst[dst_off:dst_off+n] = src[:n] (stream-ordered device copy; rows of any width)."""
        if n <= 0:
            return
        w = src.element_size() * (src.shape[1] if src.dim() > 1 else 1)
        self.check(self.L.sx_memcpy(self.h, C.c_void_p(dst.data_ptr() + dst_off * w), C.c_void_p(src.data_ptr()), n * w))

    # --------------------------------------------------------------- profiling
    def profile(self, on: bool = True):
        self.check(self.L.sx_profile_enable(self.h, 1 if on else 0))

    def profile_read(self, with_bytes: bool = False):
        """[(name, ms)] (or [(name, ms, algorithmic bytes)]) of the sx calls since the last read."""
        cap = 4096
        names = (C.c_char * 32 * cap)()
        ms = (C.c_float * cap)()
        nb = (C.c_double * cap)()
        n = C.c_int()
        self.check(self.L.sx_profile_read(self.h, names, ms, nb, cap, C.byref(n)))
        out = [(bytes(names[i]).split(b"\0")[0].decode(), float(ms[i]), float(nb[i])) for i in range(n.value)]
        return out if with_bytes else [o[:2] for o in out]


class HashTable:
    def __init__(self, ctx: Ctx, h):
        self.ctx, self.h = ctx, h

    @property
    def rows(self) -> int:
        return self.ctx.L.sx_ht_rows(self.h)

    def close(self):
        if self.h:
            self.ctx.L.sx_ht_destroy(self.ctx.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


from .tpch import Tpch, QUERIES  # noqa: E402
