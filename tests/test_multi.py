"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): the survivor rebalancing plan
(libdycl's dycl_rebalance_plan) and the exchange / return protocol (rebalance.py)."""
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
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2307_04963_b200 import rebalance as RB
    B = 64                                                  # local batch per rank
    n = counts[rank]
    cap = B
    # survivors: global ids of this rank's surviving samples, rows = f(id)
    ids = torch.full((cap,), -1, dtype=torch.int64)
    ids[:n] = rank * B + torch.arange(n) * 2                  # every other sample survived
    rows = torch.zeros((cap, 5), dtype=torch.float32)
    rows[:n] = ids[:n, None].float() * torch.tensor([1.0, -2.0, 0.5, 3.0, 7.0])
    new_n, send, recv = RB.exchange([rows, ids], n)
    ok = True
    # content integrity: every held row still matches its id
    ok &= bool(torch.equal(rows[:new_n], ids[:new_n, None].float() * torch.tensor([1.0, -2.0, 0.5, 3.0, 7.0])))
    # "compute" on the holding rank, return results home, compare to local compute
    res = rows[:new_n].sum(dim=1, keepdim=True) * 3.0 + 1.0
    out = torch.full((B, 1), float("nan"))
    RB.return_results(res, ids, new_n, B, out)
    mine = rank * B + torch.arange(n) * 2
    expect = (mine[:, None].float() * torch.tensor([1.0, -2.0, 0.5, 3.0, 7.0])).sum(1, keepdim=True) * 3.0 + 1.0
    ok &= bool(torch.equal(out[(mine - rank * B)], expect))
    ok &= bool(torch.isnan(out[1::2]).all()) if n else True
    held = torch.tensor([new_n])
    allh = [torch.zeros_like(held) for _ in range(world)]
    dist.all_gather(allh, held)
    q.put((rank, ok, [int(h) for h in allh], int(send.sum()), int(recv.sum())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("counts", [[30, 4], [5, 17, 2], [0, 9]])
def test_gloo_exchange_and_return(counts):
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
