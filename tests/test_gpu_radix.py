"""H5 parity: sx_radix_partition and sx_hash_join (flat and radix-partitioned) through the C ABI
vs the CPU oracle (join µbench closed form / brute force, or_join) and vs properties that pin the
partition function (SURVEY.md §8(a) H5, §8(c) "µbench join"; reading R14)."""
import numpy as np
import pytest

import gen
import oracle
from tests.helpers import np_fmix64, np_pair_mix

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2508_04701_b200 as sx  # noqa: E402
from paper_2508_04701_b200 import _abi as A  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return sx.Ctx(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n,bits,key_t", [(0, 3, np.int64), (1, 1, np.int32), (5000, 4, np.int32),
                                          (100_003, 8, np.int64), (300_001, 10, np.int32)])
def test_radix_partition(ctx, n, bits, key_t):
    rng = np.random.default_rng(n + bits)
    keys = rng.integers(-2**31, 2**31 - 1, n, dtype=np.int64).astype(key_t)
    pay = rng.integers(-2**62, 2**62, n, dtype=np.int64)
    cols = [sx.col(dev(keys)), sx.col(dev(pay))]
    (pk, pp), rows, offs = ctx.radix_partition(cols, [0], bits, rows=True)
    pk, pp, rows = pk.cpu().numpy(), pp.cpu().numpy(), rows.cpu().numpy()
    P = 1 << bits
    # the documented partition function: (fmix64(key as u64, sign-extended) >> 48) & (2^bits - 1)
    part = ((np_fmix64(keys.astype(np.int64).view(np.uint64)) >> np.uint64(48)) & np.uint64(P - 1)).astype(np.int64)
    assert offs[0] == 0 and offs[-1] == n and all(offs[i] <= offs[i + 1] for i in range(P))
    assert np.array_equal(np.diff(offs), np.bincount(part, minlength=P))
    assert np.array_equal(np.sort(rows), np.arange(n))  # a permutation of the input rows
    assert np.array_equal(pk, keys[rows]) and np.array_equal(pp, pay[rows])
    for p in range(P):
        assert (part[rows[offs[p]:offs[p + 1]]] == p).all()
    for k in keys[:20]:
        assert sx.lib().sx_radix_of(int(k) & (2**64 - 1), bits) == part[list(keys).index(k)]


@pytest.mark.parametrize("n,bits,key_t", [(70_001, 3, np.int64), (1_000_003, 10, np.int64), (4_097, 9, np.int64),
                                          (500_000, 7, np.int32)])
def test_radix_partition_register_path(ctx, n, bits, key_t):
    """No row ids: K7r (the register-resident scatter, shared-atomic ranks) — each partition holds
    exactly its rows' (key, payload) pairs."""
    rng = np.random.default_rng(n + bits)
    keys = rng.integers(-2**40, 2**40, n, dtype=np.int64).astype(key_t)
    pay = rng.integers(-2**62, 2**62, n, dtype=np.int64)
    (pk, pp), _, offs = ctx.radix_partition([sx.col(dev(keys)), sx.col(dev(pay))], [0], bits, rows=False)
    pk, pp = pk.cpu().numpy(), pp.cpu().numpy()
    P = 1 << bits
    part = ((np_fmix64(keys.astype(np.int64).view(np.uint64)) >> np.uint64(48)) & np.uint64(P - 1)).astype(np.int64)
    assert offs[0] == 0 and offs[-1] == n
    assert np.array_equal(np.diff(offs), np.bincount(part, minlength=P))
    for p_ in range(P):
        lo, hi = offs[p_], offs[p_ + 1]
        got = sorted(zip(pk[lo:hi].tolist(), pp[lo:hi].tolist()))
        want = sorted(zip(keys[part == p_].tolist(), pay[part == p_].tolist()))
        assert got == want, p_


def test_radix_partition_with_selection(ctx):
    n = 70_001
    keys = np.arange(n, dtype=np.int32) * 7
    sel = np.nonzero(keys % 3 == 1)[0].astype(np.int32)
    (pk,), rows, offs = ctx.radix_partition([sx.col(dev(keys))], [0], 5, in_sel=dev(sel), rows=True)
    rows = rows.cpu().numpy()
    assert np.array_equal(np.sort(rows), sel)
    assert np.array_equal(pk.cpu().numpy(), keys[rows])


@pytest.mark.parametrize("zipf", [False, True])
@pytest.mark.parametrize("strategy", [1, 2])
def test_join_mbench_vs_closed_form(ctx, zipf, strategy):
    nb, np_ = 1 << 16, (1 << 20) + 13
    bk, bp = gen.mb_join_build(nb, device="cuda")
    pk, pp = gen.mb_join_probe(nb, np_, zipf, seed=11, device="cuda")
    want = oracle.mb_join_closed(nb, pk.cpu().numpy(), pp.cpu().numpy())
    prow, brow, (gb, gp), used = ctx.hash_join([sx.col(bk), sx.col(bp)], [0], [sx.col(pk), sx.col(pp)], [0],
                                               "inner", unique=True, bp=[1], pp=[1], strategy=strategy)
    assert used == strategy
    gb, gp = gb.cpu().numpy(), gp.cpu().numpy()
    got = {"count": len(gb), "sum_build": int(gb.sum()), "sum_probe": int(gp.sum()), "pair_hash": np_pair_mix(gb, gp)}
    assert got == want
    # row ids are consistent with the payloads (payload = row id in this workload)
    assert np.array_equal(prow.cpu().numpy().astype(np.int64), gp)
    assert np.array_equal(brow.cpu().numpy().astype(np.int64), gb)


@pytest.mark.parametrize("strategy", [2, 3])
@pytest.mark.parametrize("zipf", [False, True])
def test_join_mbench_inline_payloads(ctx, zipf, strategy):
    """The µbench's own call shape (payload pairs only, no row ids): the partitioned join's
    inline-value path (K8i) and the flat inline table (K8f) vs the closed form."""
    nb, np_ = 1 << 17, (1 << 21) + 7
    bk, bp = gen.mb_join_build(nb, device="cuda")
    pk, pp = gen.mb_join_probe(nb, np_, zipf, seed=5, device="cuda")
    want = oracle.mb_join_closed(nb, pk.cpu().numpy(), pp.cpu().numpy())
    _, _, (gb, gp), used = ctx.hash_join([sx.col(bk), sx.col(bp)], [0], [sx.col(pk), sx.col(pp)], [0], "inner",
                                         unique=True, bp=[1], pp=[1], strategy=strategy, rows=(False, False))
    assert used == strategy
    gb, gp = gb.cpu().numpy(), gp.cpu().numpy()
    got = {"count": len(gb), "sum_build": int(gb.sum()), "sum_probe": int(gp.sum()), "pair_hash": np_pair_mix(gb, gp)}
    assert got == want


def test_flat_inline_join_reserved_key(ctx):
    """K8f: int64 keys including -1 (the table's EMPTY marker: side cell), 0 and the extremes,
    misses on both sides, payload widths 4 and 8 — against the oracle's join."""
    rng = np.random.default_rng(4)
    nb, np_ = 50_000, 300_001
    bkey = np.unique(rng.integers(-(2**63), 2**63 - 1, nb * 2, dtype=np.int64))[:nb]
    bkey[:4] = [-1, 0, -(2**63), 2**63 - 1]
    bkey = rng.permutation(bkey)
    pkey = np.where(rng.random(np_) < 0.6, bkey[rng.integers(0, nb, np_)], rng.integers(-(2**63), 2**63 - 1, np_, dtype=np.int64))
    pkey[:3] = [-1, -1, 5]
    bpay = rng.integers(-(2**31), 2**31 - 1, nb).astype(np.int32)
    ppay = rng.integers(-(2**62), 2**62, np_)
    _, _, (gb, gp), used = ctx.hash_join([sx.col(dev(bkey)), sx.col(dev(bpay))], [0], [sx.col(dev(pkey)), sx.col(dev(ppay))],
                                         [0], "inner", unique=True, bp=[1], pp=[1], strategy=3, rows=(False, False))
    assert used == 3
    op, ob = oracle.join(bkey, pkey, "inner")
    assert sorted(zip(gb.cpu().numpy().tolist(), gp.cpu().numpy().tolist())) == sorted(zip(bpay[ob].tolist(), ppay[op].tolist()))


@pytest.mark.parametrize("inline", ["1", "0"])
def test_partitioned_join_reserved_key(ctx, monkeypatch, inline):
    """int64 keys including -1 (all ones: the inline table's EMPTY marker, kept in a side cell),
    0, and the extremes; misses on both sides; payload outputs of widths 4 and 8."""
    monkeypatch.setenv("SX_PJ_INLINE", inline)
    rng = np.random.default_rng(3)
    nb, np_ = 30_000, 200_001
    bkey = np.unique(rng.integers(-(2**63), 2**63 - 1, nb * 2, dtype=np.int64))[:nb]
    bkey[:4] = [-1, 0, -(2**63), 2**63 - 1]
    bkey = rng.permutation(bkey)
    pkey = np.where(rng.random(np_) < 0.6, bkey[rng.integers(0, nb, np_)], rng.integers(-(2**63), 2**63 - 1, np_, dtype=np.int64))
    pkey[:3] = [-1, -1, 5]
    bpay = rng.integers(-(2**31), 2**31 - 1, nb).astype(np.int32)
    ppay = rng.integers(-(2**62), 2**62, np_)
    _, _, (gb, gp), used = ctx.hash_join([sx.col(dev(bkey)), sx.col(dev(bpay))], [0], [sx.col(dev(pkey)), sx.col(dev(ppay))],
                                         [0], "inner", unique=True, bp=[1], pp=[1], strategy=2, rows=(False, False))
    assert used == 2
    op, ob = oracle.join(bkey, pkey, "inner")
    assert sorted(zip(gb.cpu().numpy().tolist(), gp.cpu().numpy().tolist())) == sorted(zip(bpay[ob].tolist(), ppay[op].tolist()))


@pytest.mark.parametrize("inline", ["1", "0"])
@pytest.mark.parametrize("nkeys", [1, 2])
def test_partitioned_join_vs_or_join(ctx, monkeypatch, nkeys, inline):
    """Partitioned INNER join on a unique build with misses, int32 / packed two-key columns, a
    selection on each side: the multiset of (probe row, build row) pairs equals or_join's."""
    monkeypatch.setenv("SX_PJ_INLINE", inline)
    rng = np.random.default_rng(nkeys)
    nb, np_ = 40_000, 250_003
    if nkeys == 1:
        bkey = rng.permutation(np.arange(-nb, nb * 3, dtype=np.int32))[:nb]
        pkey = rng.integers(-nb * 2, nb * 4, np_, dtype=np.int64).astype(np.int32)
        bcols, pcols = [sx.col(dev(bkey))], [sx.col(dev(pkey))]
        bk64, pk64 = bkey.astype(np.int64), pkey.astype(np.int64)
        keys = [0]
    else:
        u = rng.permutation(np.arange(nb * 2, dtype=np.int64))[:nb]
        b0, b1 = (u // 7).astype(np.int32), (u % 7).astype(np.int32)
        pu = rng.integers(0, nb * 3, np_, dtype=np.int64)
        p0, p1 = (pu // 7).astype(np.int32), (pu % 7).astype(np.int32)
        bcols, pcols = [sx.col(dev(b0)), sx.col(dev(b1))], [sx.col(dev(p0)), sx.col(dev(p1))]
        bk64 = (b0.astype(np.int64) << 32) | b1.astype(np.int64)
        pk64 = (p0.astype(np.int64) << 32) | p1.astype(np.int64)
        keys = [0, 1]
    bsel = np.nonzero(rng.random(nb) < 0.9)[0].astype(np.int32)
    psel = np.nonzero(rng.random(np_) < 0.7)[0].astype(np.int32)
    prow, brow, _, used = ctx.hash_join(bcols, keys, pcols, keys, "inner", unique=True, strategy=2,
                                        build_sel=dev(bsel), probe_sel=dev(psel))
    assert used == 2
    got = sorted(zip(prow.cpu().numpy().tolist(), brow.cpu().numpy().tolist()))
    op, ob = oracle.join(bk64[bsel], pk64[psel], "inner")
    want = sorted(zip(psel[op].tolist(), bsel[ob].tolist()))
    assert got == want


def test_join_empty_sides(ctx):
    e64 = dev(np.zeros(0, np.int64))
    k = dev(np.arange(10, dtype=np.int64))
    for b, p in ((e64, k), (k, e64), (e64, e64)):
        for strategy in (1, 2):
            prow, brow, _, _ = ctx.hash_join([sx.col(b)], [0], [sx.col(p)], [0], "inner", strategy=strategy)
            assert len(prow) == 0 and len(brow) == 0
