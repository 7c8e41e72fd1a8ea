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


@pytest.mark.gpu
def test_c_abi_allreduce_stats_one_rank():
    """tc_allreduce_stats (the C-ABI reduction for non-torch hosts) on a
    1-rank NCCL communicator: the grouped SUM / MIN leaves the record as is;
    a NULL communicator is TC_EINVAL."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import ctypes
    from paper_2105_12415_b200 import _abi, device as D
    nccl = ctypes.CDLL("libnccl.so.2", mode=ctypes.RTLD_GLOBAL)

    class UniqueId(ctypes.Structure):
        _fields_ = [("internal", ctypes.c_char * 128)]

    uid = UniqueId()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()
    torch.cuda.set_device(0)
    assert nccl.ncclCommInitRank(ctypes.byref(comm), 1, uid, 0) == 0
    try:
        st = D.new_stats()
        st[:6] = torch.tensor([5, 4, 4, 1, 3, 2], dtype=torch.int64)
        st[6:].view(torch.float64)[0] = 0.25
        before = st.clone()
        lib = _abi.load()
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        assert lib.tc_allreduce_stats(ctypes.c_void_p(st.data_ptr()), comm, s) == 0
        torch.cuda.synchronize()
        assert torch.equal(st, before)
        assert lib.tc_allreduce_stats(ctypes.c_void_p(st.data_ptr()), None, s) == 1   # TC_EINVAL
    finally:
        nccl.ncclCommDestroy(comm)
