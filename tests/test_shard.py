"""Multi-process path on CPU (gloo, world size 2 and 3): strip partitioning
with the L-row halo, round-robin frame sharding and the final strip gather
(paper_2202_13926_b200/shard.py).  Each rank reconstructs its strip with the
oracle restatement (the checker) from ONLY its halo rows; the gathered frame
must equal the single-process reconstruction bitwise (SURVEY §8e
determinism; the analogue of pkg/tests/test_acceptance.py:174-183)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2202_13926_b200 import shard  # noqa: E402
from oracle import port as oracle  # noqa: E402

B, L, I = 4, 6, 12  # N = 16 keeps the oracle fast


def _frame(seed=3, h=45, w=36, hole=False):
    img = oracle.synthetic_frame(h, w, seed)
    sampled, mask = oracle.quarter_sample(img, seed + 1)
    if hole:
        # an unsampled hole larger than the support (N = 16): its blocks have an
        # empty window and take the frame-wide mean (reconstruction.py:236-237)
        mask[4:40, 6:30] = False
        sampled[~mask] = 0.0
    return sampled, mask


def _oracle_strip(px_rows, mask_rows, ya, row0, row1, fill, height):
    """Strip with the oracle, given only the halo rows [ya, ya + len) and the
    frame-wide empty-support value."""
    full_px = np.zeros((height, px_rows.shape[1]))
    full_mk = np.zeros((height, px_rows.shape[1]), bool)
    full_px[ya:ya + px_rows.shape[0]] = px_rows
    full_mk[ya:ya + mask_rows.shape[0]] = mask_rows
    out = oracle.reconstruct_image(full_px, full_mk, B, L, I, threads=1, block_rows=(row0, row1),
                                   fill_value=fill)
    return out[min(height, row0 * B):min(height, row1 * B)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, hole):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sampled, mask = _frame(hole=hole)
        H, W = sampled.shape
        row0, row1, rows = shard.reconstruct_strip_host(
            sampled, mask, B, L, rank, world,
            lambda p, m, ya, r0, r1, fill: _oracle_strip(p, m, ya, r0, r1, fill, H))
        full = shard.gather_strips(torch.from_numpy(np.ascontiguousarray(rows)), row0, row1, B, H, W,
                                   world)
        # frame stream: each rank takes its round-robin frames, rank 0 collects the count
        mine = shard.frame_shard(7, rank, world)
        n = torch.tensor([len(mine)])
        dist.all_reduce(n)
        if rank == 0:
            q.put((full.numpy(), int(n.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,hole", [(2, False), (3, False), (3, True)])
def test_strip_gather_matches_single_process(world, hole):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, hole)) for r in range(world)]
    for p in procs:
        p.start()
    full, nframes = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sampled, mask = _frame(hole=hole)
    ref = oracle.reconstruct_image(sampled, mask, B, L, I, threads=1)
    assert np.array_equal(full, ref)
    assert nframes == 7


def test_hole_frame_has_empty_windows_and_global_fill():
    # the hole test above only means something if some window is empty and the
    # strip-local mean would differ from the frame's
    sampled, mask = _frame(hole=True)
    H = sampled.shape[0]
    fill = shard.frame_fill(sampled, mask)
    ref = oracle.reconstruct_image(sampled, mask, B, L, I, threads=1)
    assert np.any(ref == fill)
    top = _oracle_strip(sampled[:26], mask[:26], 0, 0, 5, float(sampled[:26].sum()) / mask[:26].sum(), H)
    assert not np.array_equal(top, ref[:20])


def test_partition_arithmetic():
    # 4K: 540 block rows over 8 ranks -> 67/68 rows, contiguous, covering
    spans = [shard.strip_rows(540, r, 8) for r in range(8)]
    assert spans[0][0] == 0 and spans[-1][1] == 540
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert {b - a for a, b in spans} <= {67, 68}
    # halo rows clipped at the frame edges
    assert shard.strip_io_rows(0, 68, 4, 14, 2160) == (0, 286, 0, 272)
    assert shard.strip_io_rows(472, 540, 4, 14, 2160) == (1874, 2160, 1888, 2160)
    assert shard.frame_shard(64, 3, 8) == list(range(3, 64, 8))
    with pytest.raises(ValueError):
        shard.strip_rows(10, 2, 2)
