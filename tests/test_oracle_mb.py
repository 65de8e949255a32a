"""Pins of the operator-µbenchmark oracle (oracle.or_mb_*) and generator (SURVEY.md §8(c)
"µbench join" / "µbench group-by", §8(d) C5a/C5b; readings R15-R17).

The closed forms rest on the build keys being mix64(i) with mix64 a bijection: they are pinned
against brute force (std::unordered_multimap, pandas) and against the identities the generator
fixes (every probe matches exactly one build row; Σ probe payload = Σ j; Zipf mass below 2^20
of 2^27 ranks = 20/27)."""
import numpy as np
import pandas as pd
import pytest

import gen
import oracle
from tests.helpers import np_pair_mix


def test_unmix64_inverts_the_generator_keys():
    k, p = gen.mb_join_build(1 << 12)
    for key, i in zip(k[::97], p[::97]):
        assert oracle.unmix64(int(key)) == int(i)
    rng = np.random.default_rng(5)
    for x in rng.integers(0, 2**63, 50, dtype=np.int64):
        assert oracle.unmix64(int(gen.mb_join_build(int(x) + 1, r0=int(x))[0][0]) & (2**64 - 1)) == int(x)


@pytest.mark.parametrize("zipf", [False, True])
def test_join_closed_form_equals_brute_force(zipf):
    nb, np_ = 1 << 10, 1 << 15
    bk, bp = gen.mb_join_build(nb)
    pk, pp = gen.mb_join_probe(nb, np_, zipf, seed=7)
    # add probes that match nothing (keys of rows >= nb) and a ragged tail
    xk, _ = gen.mb_join_build(nb + 100, r0=nb)
    pk = np.concatenate([pk, xk])
    pp = np.concatenate([pp, np.arange(np_, np_ + 100, dtype=np.int64)])
    closed = oracle.mb_join_closed(nb, pk, pp)
    brute = oracle.mb_join_hash(bk, bp, pk, pp)
    assert closed == brute
    assert closed["count"] == np_  # every generated probe matches exactly one build row
    assert closed["sum_probe"] == np_ * (np_ - 1) // 2
    # the pair hash also agrees with an independent numpy evaluation over the matched pairs
    m = pp < np_
    bpay = np.array([oracle.unmix64(int(x) & (2**64 - 1)) for x in pk[m]], dtype=np.int64)
    assert closed["pair_hash"] == np_pair_mix(bpay, pp[m])
    assert closed["sum_build"] == int(bpay.sum())


def test_join_brute_force_duplicates_and_misses():
    bk = np.array([5, 5, 7, -1, 0], np.int64)
    bp = np.array([10, 11, 12, 13, 14], np.int64)
    pk = np.array([5, 6, 0, -1, 5], np.int64)
    pp = np.array([100, 101, 102, 103, 104], np.int64)
    s = oracle.mb_join_hash(bk, bp, pk, pp)
    pairs = [(10, 100), (11, 100), (14, 102), (13, 103), (10, 104), (11, 104)]
    assert s["count"] == 6
    assert s["sum_build"] == sum(b for b, _ in pairs) and s["sum_probe"] == sum(p for _, p in pairs)
    assert s["pair_hash"] == sum(oracle.pair_mix(b, p) for b, p in pairs) % 2**64


def test_zipf_mass_and_uniform_mean():
    nb = 1 << 27
    js = range(0, 400_000)
    rz = np.array([gen.mb_probe_rank(j, nb, True) for j in js])
    assert abs((rz < (1 << 20)).mean() - 20 / 27) < 0.005  # log-uniform: P(r+1 < 2^k) = k / log2(nb)
    assert abs((rz < 1).mean() - 1 / 27) < 0.002             # octave 0 (r + 1 in [1, 2)) is rank 0 alone
    assert rz.min() >= 0 and rz.max() < nb
    ru = np.array([gen.mb_probe_rank(j, nb, False) for j in range(100_000)])
    assert abs(ru.mean() / nb - 0.5) < 0.005


@pytest.mark.parametrize("G", [1, 4, 1000])
def test_groupby_direct_equals_pandas(G):
    n = 50_000
    k, v = gen.mb_groupby(n, G, seed=3)
    d = oracle.mb_groupby_direct(k, v, G)
    df = pd.DataFrame({"k": k, "v": v}).groupby("k")["v"].agg(["sum", "count", "min", "max"])
    assert len(d) == len(df)
    for g, (s, c, mn, mx) in d.items():
        key = int(gen.mb_join_build(g + 1, r0=g)[0][0])  # mix64(g)
        row = df.loc[key]
        assert (s, c, mn, mx) == (int(row["sum"]), int(row["count"]), int(row["min"]), int(row["max"]))
    assert v.min() >= 100 and v.max() <= 10_000_000
