"""Process-group plumbing of the z-slab path: one process per
GPU, torch.distributed for the bootstrap only.  Rank 0 draws the NCCL
unique id through the C ABI (sip_comm_unique_id) and broadcasts it over the
process group; every rank then creates its grid with
``comm=comm_desc(...)``; the library's own NCCL communicator carries the
halos and reductions.  Marshalling only: no arithmetic of the method."""
from __future__ import annotations

import ctypes as C

import numpy as np

from .sip import SIP_OK, SipError, lib


def slab(nz: int, nranks: int, rank: int) -> tuple[int, int]:
    """(z0, nz_local) of `rank` under the library's slab rule (sip_slab)."""
    z0, n = C.c_int64(0), C.c_int64(0)
    s = lib().sip_slab(int(nz), int(nranks), int(rank), C.byref(z0), C.byref(n))
    if s != SIP_OK:
        raise SipError(s, lib().sip_status_string(s).decode())
    return z0.value, n.value


def unique_id() -> np.ndarray:
    buf = np.zeros(128, dtype=np.uint8)
    s = lib().sip_comm_unique_id(C.c_void_p(buf.ctypes.data))
    if s != SIP_OK:
        raise SipError(s, lib().sip_status_string(s).decode())
    return buf


def comm_desc(group=None) -> dict:
    """{'nranks', 'rank', 'uid'} for Grid(comm=...): uid from rank 0, broadcast
    over the (initialised) torch.distributed group (nccl: via the current
    CUDA device; gloo: on the host)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = unique_id() if rank == 0 else np.zeros(128, dtype=np.uint8)
    backend = dist.get_backend(group)
    t = torch.from_numpy(uid.copy())
    if backend == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=0, group=group)
    return {"nranks": world, "rank": rank, "uid": np.ascontiguousarray(t.cpu().numpy())}


def local_slab_of(array: np.ndarray, nranks: int, rank: int) -> np.ndarray:
    """this rank's planes of a whole-grid array (z = axis 0)"""
    z0, n = slab(array.shape[0], nranks, rank)
    return np.ascontiguousarray(array[z0:z0 + n])


def max_over_ranks(value: float, group=None, device=None) -> float:
    """max of a per-rank scalar (timings are reported as the slowest rank)"""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
