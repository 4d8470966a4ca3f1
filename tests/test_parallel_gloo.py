"""World-size-2 gloo tests of the multi-GPU tile path on CPU: band layout,
the all-gather of row-padded tiles and the image assembly, for one frame
and for a batch of frames in one collective (the per-rank
render is replaced by a synthetic tile whose pixels encode their global
row, so the check is exact)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, height, width, band_rows, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, height, width, band_rows, q)
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _body(rank, world, height, width, band_rows, q):
    if True:
        from paper_2101_10994_b200 import parallel
        layout = parallel.band_layout(height, world, band_rows)
        rows = layout[rank]
        local = torch.zeros((len(rows), width, 3), dtype=torch.int32)
        local[:, :, 0] = torch.as_tensor(rows, dtype=torch.int32)[:, None]
        local[:, :, 1] = torch.arange(width, dtype=torch.int32)[None, :]
        local[:, :, 2] = rank
        img = parallel.gather_tiles(local, layout, height)
        # gathered to one rank only: the others get None
        to1 = parallel.gather_tiles(local, layout, height, dst=1)
        assert (to1 is None) == (rank != 1)
        if to1 is not None:
            assert torch.equal(to1, img)
        # a batch of 3 frames (frame f's pixels also carry f) in one collective
        frames = torch.stack([local + 1000 * f for f in range(3)])
        imgs = parallel.gather_frames(frames, layout, height)
        assert tuple(imgs.shape) == (3, height, width, 3)
        for f in range(3):
            assert torch.equal(imgs[f], img + 1000 * f)
        to0 = parallel.gather_frames(frames, layout, height, dst=0)
        assert (to0 is None) == (rank != 0)
        if to0 is not None:
            assert torch.equal(to0, imgs)
        q.put((rank, img.numpy()))


@pytest.mark.parametrize("height,band_rows", [(72, 8), (45, 8), (10, 4)])
def test_two_rank_band_gather(height, band_rows):
    world, width = 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, height, width, band_rows, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=90) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        img = got[r]
        assert not isinstance(img, str), img
        assert img.shape == (height, width, 3)
        np.testing.assert_array_equal(img[:, :, 0], np.repeat(np.arange(height)[:, None], width, axis=1))
        np.testing.assert_array_equal(img[:, :, 1], np.repeat(np.arange(width)[None, :], height, axis=0))
        owner = (np.arange(height) // band_rows) % world
        np.testing.assert_array_equal(img[:, 0, 2], owner)


def test_band_layout_partition():
    from paper_2101_10994_b200 import parallel
    for h, w, b in [(720, 8, 8), (1080, 3, 8), (7, 4, 2), (1, 2, 8)]:
        lay = parallel.band_layout(h, w, b)
        allrows = np.sort(np.concatenate(lay))
        np.testing.assert_array_equal(allrows, np.arange(h))
        for r, rows in enumerate(lay):
            assert np.all((rows // b) % w == r)
            assert np.all(np.diff(rows) > 0)
