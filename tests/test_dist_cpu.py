"""Multi-process (world_size 2, gloo, CPU) tests of the N > 1 host logic: bank shards, pair
assignment, NCCL-id broadcast, max/sum over ranks, and the bank-shard decomposition of the
window distances summed with a real all-reduce (the exchange libbn does over NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_12620_b200.dist import (broadcast_unique_id, max_over_ranks, pairs_of_rank, shard_range,
                                        sum_over_ranks)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions():
    for T in (2, 7, 64, 1000, 8192):
        for world in (1, 2, 3, 8):
            if T < world:
                continue
            r = [shard_range(T, k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == T
            assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(1, 0, 2)


def test_pairs_round_robin():
    for world in (1, 2, 4, 8):
        got = sorted(j for r in range(world) for j in pairs_of_rank(8, r, world))
        assert got == list(range(8))


def _partial_distances(c, L, R=7):
    """Plain window distances D(p, p+o) over the half window from counts c[P][T] (test helper)."""
    P = L * L
    img = c.reshape(L, L, -1).astype(np.int64)
    out = []
    offs = [(ox, 0) for ox in range(1, R + 1)] + [(ox, oy) for oy in range(1, R + 1) for ox in range(-R, R + 1)]
    for ox, oy in offs:
        nb = np.roll(img, (-oy, -ox), axis=(0, 1))
        out.append(((img - nb) ** 2).sum(-1).reshape(P))
    return np.stack(out, 1)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = broadcast_unique_id(bytes(range(128)) if rank == 0 else None)
        assert uid == bytes(range(128))
        assert max_over_ranks(1.5 + rank) == 1.5 + world - 1
        assert sum_over_ranks(rank + 1) == world * (world + 1) // 2
        # bank-shard decomposition with a real all-reduce: partial distances over disjoint
        # integrand shards sum to the full-bank distances (what bn_comm_init's all-reduce does)
        import synth
        from oracle import oracle

        L, T = 16, 40
        a, b, px, py = synth.make_bank(T, 3)
        U = synth.make_tile(L, 4)
        t0, t1 = shard_range(T, rank, world)
        pb = oracle.OracleProblem(L, t1 - t0, (16,), synth.D1, synth.D2, a[t0:t1], b[t0:t1], px[t0:t1], py[t0:t1])
        part = torch.from_numpy(_partial_distances(pb.counts(U)[0], L))
        dist.all_reduce(part)
        full_pb = oracle.OracleProblem(L, T, (16,), synth.D1, synth.D2, a, b, px, py)
        full = _partial_distances(full_pb.counts(U)[0], L)
        assert np.array_equal(part.numpy(), full)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
