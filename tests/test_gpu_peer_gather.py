"""Fused row-tile gather over CUDA IPC (tiles.PeerPlaneExchange +
wcgh_job_set_peer_planes): two ranks (processes) each compute their row band
and, from the band's final kernel, store it into BOTH ranks' full planes;
after a host barrier every rank holds the whole plane, bit-identical to a
single-process run. Only one GPU is available here, so both processes map
each other's planes on the same device: the kernels never wait on one
another (host barrier only), and on a multi-GPU box the same stores go over
NVLink (cudaIpcMemLazyEnablePeerAccess)."""
import os
import socket
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FRACS = (0.25, 0.5, 0.1, 1.0, 0.0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, method, out_dir):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist

    from paper_2211_09938_b200 import _lib, scenes, tiles
    from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = _lib.Context(0)
    sc = scenes.make_scene(0)
    n = sc.config.plane_size
    r0, rows = tiles.band(rank, world, n)
    job = HologramJob(spec_for_scene(sc, method=method, row0=r0, rows=rows), ctx)
    ex = tiles.PeerPlaneExchange(world, rank, n, 0)
    ex.register(job)
    for _ in range(2):  # twice: the planes are overwritten, not accumulated
        job.upload(sc.objects, sc.masks)
        ex.run()
        torch.cuda.synchronize()
        dist.barrier()
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), tiles.as_complex(ex.plane_tensor()))
    np.save(os.path.join(out_dir, f"band{rank}.npy"), job.download())
    dist.barrier()
    # new inputs every step, no barrier after the read: rank 0 reads each
    # step's plane late (after a sleep) while rank 1 already produces the next
    # step — the double-buffered planes (step epoch) keep rank 0's copy intact
    for k, frac in enumerate(FRACS):
        sk = scenes.make_scene(0, saliency_frac=frac)
        job.upload(sk.objects, sk.masks)
        ex.run()
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            time.sleep(0.3)
        np.save(os.path.join(out_dir, f"step{k}_rank{rank}.npy"), tiles.as_complex(ex.plane_tensor()))
    dist.barrier()
    ex.close()
    job.close()
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("method", ["direct", "lut", "fft"])
def test_two_rank_fused_gather_equals_single_process(ctx, method, tmp_path):
    import torch.multiprocessing as mp

    from paper_2211_09938_b200 import scenes
    from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene

    sc = scenes.make_scene(0)
    full = HologramJob(spec_for_scene(sc, method=method))(sc.objects, sc.masks)
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), method, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npy")
        assert np.array_equal(got, full), (method, r)
        band = np.load(tmp_path / f"band{r}.npy")
        assert np.array_equal(band, full[r * 64:(r + 1) * 64])
    for k, frac in enumerate(FRACS):
        sk = scenes.make_scene(0, saliency_frac=frac)
        ref = HologramJob(spec_for_scene(sk, method=method))(sk.objects, sk.masks)
        for r in range(world):
            assert np.array_equal(np.load(tmp_path / f"step{k}_rank{r}.npy"), ref), (method, k, r)
