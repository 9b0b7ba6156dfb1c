"""Multi-GPU plumbing: hand the job's NCCL communicator to libdycl (argument marshalling only).

One process per GPU under torchrun; torch.distributed (backend "nccl") owns the process group.
`attach` passes its ncclComm_t (ProcessGroupNCCL._comm_ptr()) to dycl_set_comm, so the survivor
rebalancing inside dycl_run runs over the same communicator on NVLink / NVSwitch.
Without an initialised NCCL process group this raises -- there is no fallback transport.
"""
from __future__ import annotations

from . import dycl as D


def nccl_comm_ptr():
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        raise RuntimeError("torch.distributed is not initialised")
    pg = dist.distributed_c10d._get_default_group()
    be = pg._get_backend(torch.device("cuda", torch.cuda.current_device()))
    if not hasattr(be, "_comm_ptr"):
        raise RuntimeError(f"process group backend {type(be).__name__} has no NCCL communicator")
    ptr = be._comm_ptr()
    if not ptr:
        # the communicator is created lazily: one collective creates it
        t = torch.zeros(1, device="cuda")
        dist.all_reduce(t)
        torch.cuda.synchronize()
        ptr = be._comm_ptr()
    if not ptr:
        raise RuntimeError("NCCL communicator not available")
    return int(ptr)


def attach(model, rank: int, world: int, policy: int = D.DYCL_REBALANCE_ALL):
    """dycl_set_comm(model.g, <the job's ncclComm_t>, rank, world, policy)."""
    D.dycl_set_comm(model.g, nccl_comm_ptr() if world > 1 else None, rank, world, policy)
    return model
