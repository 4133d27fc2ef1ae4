"""Multi-GPU decomposition: contiguous row bands of the hologram plane, one
per rank (one process per GPU), every rank seeing the full compacted point
list; the only exchange is the all-gather of the row tiles — fused into the
band's final kernel as NVLink P2P stores into CUDA-IPC-mapped peer planes
(PeerPlaneExchange), or as an NCCL all-gather (gather_tiles; gloo in the CPU
tests). Row-major bands are
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


class PeerPlaneExchange:
    """Fused row-tile gather over NVLink (one process per GPU): every rank
    allocates its full plane with an exported CUDA IPC handle, the handles
    are all-gathered once (host objects, any torch.distributed backend), and
    each rank maps its peers' planes. A job registered with `register` then
    writes its band into every rank's plane from the epilogue of the kernel
    that produces it (wcgh_job_set_peer_planes) — no collective per step; a
    barrier tells the ranks when all bands have landed.

    The planes are double-buffered with a step epoch: step k stores into
    buffer k % 2 on every rank, so a rank still reading step k's plane after
    the barrier (e.g. its D2H copy) is never overwritten by a faster peer
    already producing step k + 1; step k + 2 reuses the buffer only after
    every rank has passed step k + 1's barrier, i.e. after its read of step k.
    Use `run(job)` per step (flip + run) and `plane_tensor()` for the plane of
    the last step."""

    NBUF = 2

    def __init__(self, world: int, rank: int, plane_size: int, device: int):
        import ctypes as C

        import torch.distributed as dist

        from . import _lib as L

        self.lib = L.load()
        self.n, self.world, self.rank, self.device = plane_size, world, rank, device
        self.own, self.ptrs, self.opened = [], [[] for _ in range(self.NBUF)], []
        self.epoch, self.current, self.job = 0, None, None
        # every step is agreed on by all ranks, so a failure on one rank makes
        # all of them raise (and fall back) instead of leaving some blocked
        handles_own, err = None, ""
        try:
            hs = []
            for _ in range(self.NBUF):
                own = C.c_void_p()
                buf = C.create_string_buffer(64)
                L.check(self.lib.wcgh_ipc_alloc_plane(device, plane_size, C.byref(own), buf))
                self.own.append(int(own.value))
                hs.append(buf.raw)
            handles_own = hs
        except Exception as e:  # noqa: BLE001
            err = f"rank {rank}: {e}"
        handles = [None] * world
        dist.all_gather_object(handles, handles_own)
        if any(h is None for h in handles):
            self.close()
            raise RuntimeError("peer planes: IPC allocation failed on some rank"
                               + (f" ({err})" if handles_own is None else ""))
        ok = True
        try:
            for b in range(self.NBUF):
                for r, hs in enumerate(handles):
                    if r == rank:
                        self.ptrs[b].append(self.own[b])
                        continue
                    p = C.c_void_p()
                    L.check(self.lib.wcgh_ipc_open_plane(device, hs[b], C.byref(p)))
                    self.ptrs[b].append(int(p.value))
                    self.opened.append(int(p.value))
        except Exception as e:  # noqa: BLE001
            ok, err = False, f"rank {rank}: {e}"
        oks = [None] * world
        dist.all_gather_object(oks, ok)
        if not all(oks):
            self.close()
            raise RuntimeError("peer planes: IPC mapping failed on some rank"
                               + (f" ({err})" if not ok else ""))

    def register(self, job) -> None:
        self.job = job

    def run(self, job=None) -> None:
        """One step: point the job's fused gather at this epoch's buffers and
        run it. The caller's barrier after this marks every band landed."""
        job = job or self.job
        b = self.epoch % self.NBUF
        job.set_peer_planes(self.ptrs[b])
        job.run()
        self.current = b
        self.epoch += 1

    def plane_tensor(self):
        """torch (Nh, 2*Nh) float32 view of this rank's plane assembled by the
        last step."""
        import torch

        if self.current is None:
            raise RuntimeError("peer planes: no step has run")
        return torch.as_tensor(CudaView(self.own[self.current], (self.n, 2 * self.n)), device="cuda")

    def close(self) -> None:
        import ctypes as C

        for p in self.opened:
            self.lib.wcgh_ipc_close_plane(C.c_void_p(p))
        self.opened = []
        for p in self.own:
            self.lib.wcgh_ipc_free_plane(C.c_void_p(p))
        self.own = []


def as_complex(plane_f32) -> np.ndarray:
    a = plane_f32.detach().cpu().numpy() if hasattr(plane_f32, "detach") else plane_f32
    return np.ascontiguousarray(a).view(np.complex64)
