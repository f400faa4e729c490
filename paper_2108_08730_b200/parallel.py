"""Host-side plumbing of the z-slab decomposition: one process per GPU.

The data path (halo planes of v / p / s, dot-product allreduces) runs inside libhz over NCCL; this
module holds only the host logic around it, so it can be exercised with the gloo backend on CPU:

  * ``slab_partition``  contiguous z-slabs, nz_loc = ⌊nz/P⌋ or +1 (§8(e) "Partitioning")
  * ``make_context``    rank 0 draws the NCCL unique id (hz_get_unique_id), torch.distributed
                        broadcasts it, every rank calls hz_ctx_create (SURVEY §3 "init")
  * ``rank_max`` / ``rank_sum``  device-timed results reduced over ranks (bench: max over ranks)
  * ``gather_slabs``    rank-local owned planes → the global field on rank 0 (I/O, tests)
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np


def slab_partition(nz: int, nranks: int, rank: int) -> Tuple[int, int]:
    """(z0, nz_local) of `rank`: contiguous slabs, the first nz % P ranks get one extra plane."""
    if nranks < 1 or not (0 <= rank < nranks):
        raise ValueError("bad rank / nranks")
    if nz < nranks:
        raise ValueError(f"nz = {nz} < {nranks} ranks: every slab needs at least one plane")
    base, rem = divmod(nz, nranks)
    nzl = base + (1 if rank < rem else 0)
    z0 = rank * base + min(rank, rem)
    return z0, nzl


def all_slabs(nz: int, nranks: int) -> List[Tuple[int, int]]:
    return [slab_partition(nz, nranks, r) for r in range(nranks)]


def sources_on_rank(nodes: np.ndarray, z0: int, nzl: int, halo: int = 1) -> np.ndarray:
    """Indices of the point sources whose consistent-source stencil (±1 plane, A15) touches the
    slab's owned planes [z0, z0 + nzl)."""
    z = np.asarray(nodes)[:, 2]
    return np.nonzero((z + halo >= z0) & (z - halo < z0 + nzl))[0]


def _dist():
    import torch.distributed as dist
    return dist


def broadcast_bytes(payload: Optional[bytes], src: int = 0) -> bytes:
    """Broadcast a byte string (the 128-byte NCCL unique id) from `src` over the default group."""
    dist = _dist()
    obj = [payload]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def make_context(local_device: int):
    """hz context for this rank: NCCL communicator over all ranks of the default process group."""
    from . import hz
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return hz.hz_ctx_create(local_device)
    rank, ws = dist.get_rank(), dist.get_world_size()
    uid = broadcast_bytes(hz.hz_get_unique_id() if rank == 0 else None)
    return hz.hz_ctx_create(local_device, ws, rank, uid)


def _reduce(values: Sequence[float], op_name: str, device=None) -> List[float]:
    import torch
    dist = _dist()
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=getattr(dist.ReduceOp, op_name))
    return t.tolist()


def rank_max(values: Sequence[float], device=None) -> List[float]:
    """Element-wise max over ranks (device-timed durations: the job takes as long as its slowest rank)."""
    return _reduce(values, "MAX", device)


def rank_sum(values: Sequence[float], device=None) -> List[float]:
    """Element-wise sum over ranks (work done: grid points × RHS × applies)."""
    return _reduce(values, "SUM", device)


def gather_slabs(local: np.ndarray, nz: int, dst: int = 0) -> Optional[np.ndarray]:
    """Gather owned planes [..., nz_local, ny, nx] of every rank into [..., nz, ny, nx] on `dst`
    (None elsewhere).  `local` excludes the halo planes."""
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    ws, rank = dist.get_world_size(), dist.get_rank()
    parts = [None] * ws
    dist.gather_object(local, parts if rank == dst else None, dst=dst)
    if rank != dst:
        return None
    out = np.concatenate(parts, axis=-3)
    assert out.shape[-3] == nz
    return out
