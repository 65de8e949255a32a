"""Host-side logic of the N>1 path on CPU with a world_size-2 gloo process group (no GPU):

* shard placement: the union of the ranks' generated shards is the world=1 table, and orders and
  their lineitems land on the same rank (the co-partitioning the sharded plans rely on);
* the shuffle contract: every rank routes each key to sx_dest_rank(key, g) (libsx's host mirror
  of the device function; loading libsx needs no GPU), the counts matrix gives every rank its
  receive sizes, and after the exchange (here torch.distributed all_to_all over gloo, the same
  schedule sx_shuffle runs with NCCL) rows are conserved and each sits on its destination;
* the merge contract: per-rank partial aggregates combined on every rank equal the global ones.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.conftest import ROOT, build


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        import sys

        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import gen
        from paper_2508_04701_b200 import _abi

        L = _abi.load()
        # --- placement: co-partitioned orders/lineitem shard
        t = gen.cpu_tables(20, seed=5, shard=(rank, world), tables=("orders", "lineitem"))
        ok = set(t["orders"]["o_orderkey"].tolist())
        assert set(t["lineitem"]["l_orderkey"].tolist()) <= ok
        # --- shuffle contract on this rank's keys
        rng = np.random.default_rng(rank)
        keys = rng.integers(0, 2**31 - 1, 10_000).astype(np.int64)
        dest = np.array([L.sx_dest_rank(int(k), world) for k in keys])
        order = np.argsort(dest, kind="stable")
        send_counts = torch.tensor([int((dest == d).sum()) for d in range(world)], dtype=torch.int64)
        all_counts = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(all_counts, send_counts)
        recv_counts = [int(all_counts[s][rank]) for s in range(world)]
        sendbuf = torch.from_numpy(keys[order])
        recv = [torch.zeros(c, dtype=torch.int64) for c in recv_counts]
        # the schedule sx_shuffle issues inside one ncclGroupStart/End: a send and a recv per peer
        chunks = list(torch.split(sendbuf, send_counts.tolist()))
        reqs = []
        for peer in range(world):
            if peer == rank:
                recv[peer].copy_(chunks[peer])
                continue
            if send_counts[peer] > 0:
                reqs.append(dist.isend(chunks[peer].contiguous(), peer))
            if recv_counts[peer] > 0:
                reqs.append(dist.irecv(recv[peer], peer))
        for r in reqs:
            r.wait()
        got = torch.cat(recv).numpy()
        assert all(L.sx_dest_rank(int(k), world) == rank for k in got)
        tot = torch.tensor([len(keys), len(got)], dtype=torch.int64)
        dist.all_reduce(tot)
        assert tot[0] == tot[1]  # conservation
        # --- merge contract: partial (key, sum, count) per rank -> allgather -> combine
        vals = rng.integers(-100, 100, len(keys))
        part = {}
        for k, v in zip(keys % 7, vals):
            s, c = part.get(int(k), (0, 0))
            part[int(k)] = (s + int(v), c + 1)
        gathered = [None] * world
        dist.all_gather_object(gathered, part)
        merged = {}
        for pp in gathered:
            for k, (s, c) in pp.items():
                ms, mc = merged.get(k, (0, 0))
                merged[k] = (ms + s, mc + c)
        full = [None] * world
        dist.all_gather_object(full, (keys.tolist(), vals.tolist()))
        direct = {}
        for ks, vs in full:
            for k, v in zip(ks, vs):
                s, c = direct.get(k % 7, (0, 0))
                direct[k % 7] = (s + v, c + 1)
        assert merged == direct
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_world2_gloo_host_logic():
    build("sx")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res
