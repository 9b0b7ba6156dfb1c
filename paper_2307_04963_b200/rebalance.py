"""Survivor rebalancing across ranks after an exit point.

Samples are independent (Eq. 2 is per-x), so the batch shards over
GPUs with no collective; but early exits leave ranks with unequal numbers of
survivors.  After an exit point:

  1. all-gather the survivor counts (world int32);
  2. plan = dycl_rebalance_plan(counts, rank) (libdycl, deterministic): surplus ranks
     send their LAST (count - T) rows, in order, to deficit ranks in rank order,
     T = ceil(sum / world);
  3. batched point-to-point send / recv of the rows and their GLOBAL sample ids
     (torch.distributed: NCCL for CUDA tensors over NVLink, gloo for CPU tensors);
     received rows are appended after the kept rows in source-rank order;
  4. at the end, results of rows computed away from home go back to the home rank
     (return_results), which scatters them by global id -- output order stays the
     original order (reading R17).

The plan is the C-ABI host function; this module only moves bytes.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import dycl as D


def _all_gather_int(v: int, device) -> np.ndarray:
    world = dist.get_world_size()
    t = torch.tensor([int(v)], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return np.array([int(x.item()) for x in out], dtype=np.int32)


def exchange(tensors, count: int):
    """Rebalance the first `count` rows of every tensor in `tensors` (same leading dim,
    capacity >= the planned new count).  Returns (new_count, send, recv)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = tensors[0].device
    counts = _all_gather_int(count, dev)
    send, recv, new_count = D.dycl_rebalance_plan(counts, rank)
    ops = []
    if send.sum():
        off = count - int(send.sum())                     # the tail, destination rank ascending
        for j in range(world):
            n = int(send[j])
            if n:
                for t in tensors:
                    ops.append(dist.P2POp(dist.isend, t[off:off + n].contiguous(), j))
                off += n
    recv_bufs = []
    if recv.sum():
        pos = count                                       # appended after the kept rows
        for j in range(world):
            n = int(recv[j])
            if n:
                for t in tensors:
                    buf = torch.empty_like(t[pos:pos + n])
                    recv_bufs.append((t, pos, n, buf))
                    ops.append(dist.P2POp(dist.irecv, buf, j))
                pos += n
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for t, pos, n, buf in recv_bufs:
        t[pos:pos + n].copy_(buf)
    return new_count, send, recv


def return_results(results: torch.Tensor, ids: torch.Tensor, n: int, local_batch: int, out: torch.Tensor):
    """Scatter the first n result rows to their home ranks' `out` by global id.
    Home of id g = g // local_batch; local position = g % local_batch."""
    rank, world = dist.get_rank(), dist.get_world_size()
    ids = ids[:n]
    home = torch.div(ids, local_batch, rounding_mode="floor")
    order = torch.argsort(home * (local_batch * world) + ids)      # group by home rank, stable by id
    res_s, ids_s, home_s = results[:n][order], ids[order], home[order]
    per_dst = torch.bincount(home_s.long(), minlength=world).to(torch.int64)
    mat = [torch.zeros_like(per_dst) for _ in range(world)]
    dist.all_gather(mat, per_dst)                                   # mat[src][dst]
    ops, bufs = [], []
    off = 0
    for j in range(world):
        c = int(per_dst[j])
        if c and j != rank:
            ops.append(dist.P2POp(dist.isend, res_s[off:off + c].contiguous(), j))
            ops.append(dist.P2POp(dist.isend, ids_s[off:off + c].contiguous(), j))
        elif c:
            out[(ids_s[off:off + c] - rank * local_batch).long()] = res_s[off:off + c]
        off += c
    for j in range(world):
        c = int(mat[j][rank])
        if c and j != rank:
            rb = torch.empty((c,) + tuple(results.shape[1:]), dtype=results.dtype, device=results.device)
            ib = torch.empty(c, dtype=ids.dtype, device=ids.device)
            ops.append(dist.P2POp(dist.irecv, rb, j))
            ops.append(dist.P2POp(dist.irecv, ib, j))
            bufs.append((rb, ib))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for rb, ib in bufs:
        out[(ib - rank * local_batch).long()] = rb
