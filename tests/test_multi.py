"""Multi-rank host logic on CPU (gloo, world sizes 2-4): the survivor rebalancing plan
(libdycl's dycl_rebalance_plan) computed independently on every rank from all-gathered counts
must agree across ranks (sends == peers' receives, rows conserved, surplus ranks drop to
T = ceil(S/G)); the bench's shards tile the global batch.  The exchange itself runs inside
dycl_run (NCCL / in-process transport) and is tested on the GPU (tests/test_gpu_multi.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_04963_b200 import dycl as D


@pytest.mark.parametrize("counts", [[10, 3, 7, 0], [5, 5, 5, 5], [9, 0], [0, 0, 0], [1, 2, 3, 100], [7]])
def test_plan_invariants(counts):
    w = len(counts)
    S = sum(counts)
    T = -(-S // w)
    send = np.zeros((w, w), int)
    recv = np.zeros((w, w), int)
    new = []
    for r in range(w):
        s, rc, n = D.dycl_rebalance_plan(counts, r)
        send[r], recv[r] = s, rc
        new.append(n)
        assert not (s.any() and rc.any())                   # a rank only sends or only receives
    assert np.array_equal(send, recv.T)                     # what r sends to j, j receives from r
    assert sum(new) == S and max(new, default=0) <= max(T, max(counts) if S == 0 else T)
    for r in range(w):
        if counts[r] > T:
            assert new[r] == T                              # surplus ranks drop exactly to T
        assert new[r] <= max(T, counts[r])
    # deterministic
    assert all(np.array_equal(D.dycl_rebalance_plan(counts, r)[0], send[r]) for r in range(w))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, counts, q):
    """One rank: all-gather the survivor counts over gloo, compute this rank's plan with the
    C-ABI host function (what dycl_run does between the all-gather and the exchange), and
    check that every rank's sends match its peers' receives and the data volume is conserved."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = torch.tensor([counts[rank]], dtype=torch.int32)
    allc = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(allc, t)
    seen = [int(x) for x in allc]
    send, recv, new = D.dycl_rebalance_plan(seen, rank)
    sends = [torch.zeros(world, dtype=torch.int32) for _ in range(world)]
    dist.all_gather(sends, torch.from_numpy(send))
    matrix = torch.stack(sends).numpy()                       # matrix[r, j] = rows r sends to j
    ok = seen == list(counts)
    ok &= bool(np.array_equal(matrix[:, rank], recv))        # my receives are my peers' sends to me
    ok &= new == counts[rank] - int(send.sum()) + int(recv.sum())
    # rows a surplus rank sends are its LAST ones, destination ascending: the row ranges
    # [keep + sum(send[:j]), keep + sum(send[:j+1])) tile [keep, count) exactly
    keep = counts[rank] - int(send.sum())
    ok &= keep >= 0 and (keep == counts[rank] or int(recv.sum()) == 0)
    held = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(held, torch.tensor([new], dtype=torch.int64))
    q.put((rank, ok, [int(h) for h in held], int(send.sum()), int(recv.sum())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("counts", [[30, 4], [5, 17, 2], [0, 9], [3, 3], [100, 0, 0, 1]])
def test_gloo_plan_agreement(counts):
    world = len(counts)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, counts, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    T = -(-sum(counts) // world)
    for rank, ok, held, ns, nr in res:
        assert ok, (rank, held)
        assert sum(held) == sum(counts) and max(held) == T


@pytest.mark.parametrize("B,world", [(65536, 1), (65536, 2), (65536, 8), (65536, 3), (5, 8), (2048, 6)])
def test_bench_shards_tile_the_global_batch(B, world):
    """bench.py's shards: contiguous [r*B/G, (r+1)*B/G), disjoint, covering the global batch."""
    import bench
    lo_hi = [bench.shard(B, world, r) for r in range(world)]
    assert lo_hi[0][0] == 0 and lo_hi[-1][1] == B
    assert all(a[1] == b[0] for a, b in zip(lo_hi, lo_hi[1:]))
    sizes = [h - l for l, h in lo_hi]
    assert max(sizes) - min(sizes) <= 1
