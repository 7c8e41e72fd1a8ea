"""Multi-rank host logic on CPU (gloo, world size 2): contiguous sharding and
the stats all-reduce (SUM of int64 tallies, MIN of the fp64 min distance).
Also checks, with the oracle, that sharded tallies equal the whole run's."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_12415_b200 import shard


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 4096, 1 << 24):
        for w in (1, 2, 3, 4, 8):
            spans = [shard.shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0
            assert sum(c for _, c in spans) == n
            for (lo, c), (lo2, _) in zip(spans, spans[1:]):
                assert lo + c == lo2
    with pytest.raises(ValueError):
        shard.shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    stats = torch.zeros(7, dtype=torch.int64)
    stats[:6] = torch.tensor([10 + rank, 2 * rank, 3, rank, 5, 7 * rank])
    stats[6:].view(torch.float64)[0] = 0.5 / (rank + 1)
    shard.allreduce_stats(stats)
    q.put((rank, shard.stats_dict(stats)))
    dist.destroy_process_group()


def test_allreduce_stats_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        d = res[r]
        assert (d["iterative"], d["comparison"], d["fallback"], d["degenerate"], d["contacts"],
                d["intersecting"]) == (21, 2, 6, 1, 10, 7)
        assert d["min_distance"] == 0.25


def test_sharded_tallies_equal_whole(oracle_lib, golden_inputs):
    """The reduction is order-independent: W shards give the whole run's tallies."""
    A, B = golden_inputs["cfg0_A"], golden_inputs["cfg0_B"]
    p = oracle_lib.make_params(n_iterative=16, epsilon=1e-6)
    whole, counts, _ = oracle_lib.hybrid(A, B, p, 1e-6)
    for w in (2, 3, 8):
        tot = np.zeros(4, np.int64)
        mins = []
        for r in range(w):
            lo, c = shard.shard_range(len(A), r, w)
            o, cnt, _ = oracle_lib.hybrid(A[lo:lo + c], B[lo:lo + c], p, 1e-6)
            tot += cnt
            mins.append(o["distance"].min())
            for k in o:
                assert np.array_equal(o[k], whole[k][lo:lo + c])
        assert np.array_equal(tot, counts)
        assert min(mins) == whole["distance"].min()
