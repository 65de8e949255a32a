"""Sharded path (H10) on one B200: g logical ranks with the loopback communicator, and a 1-rank
NCCL communicator (exercises libsx's NCCL exchange).  result(g) must equal the CPU oracle (and so
result(1)) bit-exactly; the shuffle must conserve rows and place each at sx_dest_rank(key)."""
import numpy as np
import pytest

import gen
import oracle
from tests.helpers import diff_rows, rows_equal

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2508_04701_b200 as sx  # noqa: E402
from paper_2508_04701_b200 import _abi as A  # noqa: E402
from paper_2508_04701_b200.sharded import LoopbackComm, NcclComm, ShardedTpch, typed  # noqa: E402

QUERIES = ["q1", "q6", "q3", "q9", "q18"]


@pytest.fixture(scope="module")
def ctx():
    return sx.Ctx(0)


@pytest.fixture(scope="module")
def oracle_answers():
    host = gen.cpu_tables(100, seed=42)
    return {q: oracle.run_query(q, host) for q in QUERIES}


@pytest.mark.parametrize("g", [1, 2, 3, 4])
def test_loopback_sharded_queries(ctx, oracle_answers, g):
    shards = [gen.gpu_tables(100, seed=42, shard=(r, g)) for r in range(g)]
    st = ShardedTpch(ctx, LoopbackComm(ctx, g), shards)
    for q in QUERIES:
        got = st.run(q)
        assert rows_equal(got, oracle_answers[q]), f"g={g} {q}: " + diff_rows(got, oracle_answers[q])


@pytest.mark.parametrize("g", [2, 4])
@pytest.mark.parametrize("q", ["q3", "q9", "q18"])
def test_loopback_with_shuffle(ctx, oracle_answers, g, q):
    """co_located=False: every orderkey join / group-by goes through sx_partition_by_rank (the
    shuffle's one-pass partition) before it runs, as on a cluster without co-partitioned tables."""
    shards = [gen.gpu_tables(100, seed=42, shard=(r, g)) for r in range(g)]
    st = ShardedTpch(ctx, LoopbackComm(ctx, g), shards, co_located=False)
    got = st.run(q)
    assert rows_equal(got, oracle_answers[q]), diff_rows(got, oracle_answers[q])


@pytest.mark.parametrize("n,g,with_sel", [(100_003, 5, False), (1, 3, False), (0, 2, False), (4096, 64, False),
                                          (70_001, 8, True), (2047, 1, False)])
def test_partition_by_rank_contract(ctx, n, g, with_sel):
    """One pass (histogram, scan, stable scatter) over ragged tiles: counts = host histogram of
    sx_dest_rank, and every destination segment keeps input order (bit-exact)."""
    rng = np.random.default_rng(3 + n)
    k = rng.integers(-(2**40), 2**40, n).astype(np.int64)
    v = np.arange(n, dtype=np.int32)
    sel = None
    if with_sel:
        idx = np.sort(rng.choice(n, n // 3, replace=False)).astype(np.int32)
        sel = torch.from_numpy(idx).cuda()
        k, v = k[idx], v[idx]
        kk = np.zeros(n, np.int64)
        kk[idx] = k
        vv = np.zeros(n, np.int32)
        vv[idx] = v
        dev = [sx.col(torch.from_numpy(kk).cuda()), sx.col(torch.from_numpy(vv).cuda())]
    else:
        dev = [sx.col(torch.from_numpy(k).cuda()), sx.col(torch.from_numpy(v).cuda())]
    parts, counts = ctx.partition_by_rank(dev, [0], g, in_sel=sel)
    dest = np.array([sx.lib().sx_dest_rank(int(x) & ((1 << 64) - 1), g) for x in k])
    assert counts == [int((dest == d).sum()) for d in range(g)]
    pk, pv = parts[0].cpu().numpy(), parts[1].cpu().numpy()
    off = 0
    for d in range(g):
        seg = pv[off:off + counts[d]]
        assert np.array_equal(seg, v[dest == d])  # input order kept within a destination
        assert np.array_equal(pk[off:off + counts[d]], k[dest == d])
        off += counts[d]


def test_nccl_single_rank_exchange(ctx):
    comm = NcclComm(ctx, 0, 1, NcclComm.unique_id())
    rng = np.random.default_rng(4)
    k = torch.from_numpy(rng.integers(0, 10**6, 5000).astype(np.int32)).cuda()
    v = torch.from_numpy(rng.integers(0, 10**9, 5000).astype(np.int64)).cuda()
    (out,) = comm.shuffle([[typed(k, A.SX_I32), typed(v, A.SX_I64)]], [0])
    assert torch.equal(out[0][0], k) and torch.equal(out[1][0], v)
    (g,) = comm.allgather([[typed(k, A.SX_I32)]])
    assert torch.equal(g[0][0], k)
    shards = [gen.gpu_tables(10, seed=42)]
    st = ShardedTpch(ctx, comm, shards, co_located=False)
    host = gen.cpu_tables(10, seed=42)
    for q in ("q1", "q3", "q18"):
        got, want = st.run(q), oracle.run_query(q, host)
        assert rows_equal(got, want), diff_rows(got, want)
    comm.close()
