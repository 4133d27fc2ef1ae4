"""Multi-rank row-tile decomposition on CPU (gloo, world size 2): every rank
computes its row band of the hologram, one all-gather assembles the plane,
and the result equals the single-process plane bit for bit. The device
kernels are replaced by the fp64 oracle here (no GPU in this container); the
band split, the gather and the assembly are the product code (tiles.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_09938_b200 import tiles


def test_band_partition_covers_the_plane():
    for n in (8, 30, 64, 1024, 4096):
        for world in (1, 2, 3, 4, 8):
            rows = [tiles.band(r, world, n) for r in range(world)]
            assert rows[0][0] == 0
            for (a0, an), (b0, _) in zip(rows, rows[1:]):
                assert a0 + an == b0
            assert rows[-1][0] + rows[-1][1] == n
            assert max(r[1] for r in rows) - min(r[1] for r in rows) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _scene():
    rng = np.random.default_rng(3)
    n = 32
    xs = rng.integers(8, 24, 60).astype(np.int32)
    ys = rng.integers(8, 24, 60).astype(np.int32)
    amps = rng.integers(1, 256, 60).astype(np.float64)
    lay = np.zeros(60, np.int32)
    return n, (xs, ys, amps, lay), [(532e-9, 8e-6, 0.05)]


def _band_hologram(n, pts, layers, row0, rows):
    from oracle import oracle as O

    yy, xx = np.mgrid[row0:row0 + rows, 0:n]
    h = O.direct_pixels(*pts, layers, xx.ravel(), yy.ravel()).astype(np.complex64)
    return h.reshape(rows, n)


def _worker(rank, world, port, n_rows, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, pts, layers = _scene()
    row0, rows = tiles.band(rank, world, n_rows)
    band = _band_hologram(n, pts, layers, row0, rows)
    tile = torch.from_numpy(np.ascontiguousarray(band).view(np.float32))
    full = tiles.gather_tiles(tile, world, n_rows)
    if rank == 0:
        np.save(out_path, tiles.as_complex(full))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_tiles_gather_equals_single_rank(tmp_path, world):
    n, pts, layers = _scene()
    out = tmp_path / "plane.npy"
    mp.start_processes(_worker, args=(world, _free_port(), n, str(out)), nprocs=world,
                       join=True, start_method="spawn")
    gathered = np.load(out)
    single = _band_hologram(n, pts, layers, 0, n)
    assert gathered.shape == (n, n)
    assert np.array_equal(gathered, single)


def _exchange_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    msg = "ok"
    try:
        tiles.PeerPlaneExchange(world, rank, 64, 0)
    except RuntimeError as e:
        msg = str(e)
    with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as f:
        f.write(msg)
    dist.barrier()
    dist.destroy_process_group()


def test_peer_plane_exchange_fails_consistently_without_gpu(tmp_path):
    """The fused-gather setup agrees on every step across ranks: with no GPU
    (IPC allocation fails everywhere) every rank raises, none is left blocked
    in a collective, so bench.py can fall back together."""
    if torch.cuda.is_available():
        pytest.skip("needs a host without a GPU")
    mp.spawn(_exchange_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        msg = (tmp_path / f"r{r}.txt").read_text()
        assert "IPC allocation failed" in msg, msg
