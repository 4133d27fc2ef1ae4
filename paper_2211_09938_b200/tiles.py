"""Multi-GPU decomposition: contiguous row bands of the hologram plane, one
per rank (one process per GPU), every rank seeing the full compacted point
list; the only exchange is one all-gather of the row tiles (NCCL over
NVLink/NVSwitch on B200 boxes, gloo in the CPU tests). Row-major bands are
contiguous, so the gathered buffer is the plane with no repacking. The
per-pixel summation order does not depend on the band split (see
csrc/wcgh_direct.cu), so the gathered plane is bitwise identical for any
GPU count (the GPU analogue of the reference's worker-count invariance,
parallel.hpp:163-171).
"""
from __future__ import annotations

import numpy as np


def band(rank: int, world: int, plane_size: int) -> tuple[int, int]:
    """(row0, rows) of `rank`'s band: equal contiguous splits (remainder to
    the first ranks)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("band: bad rank/world")
    base, rem = divmod(plane_size, world)
    row0 = rank * base + min(rank, rem)
    rows = base + (1 if rank < rem else 0)
    return row0, rows


class CudaView:
    """Zero-copy __cuda_array_interface__ over a device pointer owned by the
    C ABI (e.g. wcgh_job_plane_dev), so torch can hand it to NCCL."""

    def __init__(self, ptr: int, shape: tuple[int, ...], typestr: str = "<f4"):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
            "version": 3, "strides": None, "stream": None,
        }


def tile_tensor(job):
    """torch view (rows, 2*Nh) float32 of the job's device row band."""
    import torch

    return torch.as_tensor(CudaView(job.plane_dev_ptr(), (job.rows, 2 * job.spec.plane_size)),
                           device="cuda")


def gather_tiles(tile, world: int, plane_size: int, out=None):
    """All-gather equal row bands into the full (Nh, 2*Nh) float32 plane."""
    import torch
    import torch.distributed as dist

    if plane_size % world:
        # unequal bands: pad to the largest band, gather, then trim
        base = -(-plane_size // world)
        padded = torch.zeros((base, tile.shape[1]), dtype=tile.dtype, device=tile.device)
        padded[: tile.shape[0]] = tile
        full = torch.empty((base * world, tile.shape[1]), dtype=tile.dtype, device=tile.device)
        dist.all_gather_into_tensor(full, padded)
        parts = [full[r * base: r * base + band(r, world, plane_size)[1]] for r in range(world)]
        res = torch.cat(parts)
        if out is not None:
            out.copy_(res)
            return out
        return res
    if out is None:
        out = torch.empty((plane_size, tile.shape[1]), dtype=tile.dtype, device=tile.device)
    dist.all_gather_into_tensor(out, tile.contiguous())
    return out


def as_complex(plane_f32) -> np.ndarray:
    a = plane_f32.detach().cpu().numpy() if hasattr(plane_f32, "detach") else plane_f32
    return np.ascontiguousarray(a).view(np.complex64)
