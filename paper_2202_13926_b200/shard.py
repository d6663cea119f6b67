"""Multi-GPU sharding of the FSR image path: one process per GPU.

Target blocks are independent (reference PAPER.md:81; reconstruction.py:220-226
keeps per-block results independent of how blocks are scheduled), so the work
shards with no collective on the data path:

* strips: the ceil(H/B) block rows of one frame are split into contiguous
  ranges, one per rank (``strip_rows``).  A rank reads image rows
  [row0*B - L, row1*B + L) clipped to the frame -- its strip plus the L-row
  halo above and below (``strip_io_rows``) -- and writes only output rows
  [row0*B, row1*B).  This is the same split the C engine uses across the
  devices it is given (fsr_abi.cu, reconstruct_host).
* frames: a stream of frames is dealt round-robin (``frame_shard``), no halo.

The only collective is the final assembly of a frame on one rank
(``gather_strips``): every rank contributes its output rows with one
``all_gather_into_tensor`` (NCCL over NVLink on GPUs, gloo on CPU).  Output
is bitwise identical for any world size because no block's arithmetic
depends on placement.
"""

from __future__ import annotations

from typing import Callable

import numpy as np


def block_rows(height: int, block: int) -> int:
    return -(-height // block)


def strip_rows(n_block_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block-row range [row0, row1) of ``rank`` (balanced to one row)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of size {world}")
    return n_block_rows * rank // world, n_block_rows * (rank + 1) // world


def strip_io_rows(row0: int, row1: int, block: int, border: int, height: int):
    """(ya, yb, oa, ob): input image rows incl. the L-row halo, output rows."""
    ya = max(0, row0 * block - border)
    yb = min(height, row1 * block + border)
    oa = min(height, row0 * block)
    ob = min(height, row1 * block)
    return ya, yb, oa, ob


def frame_shard(n_frames: int, rank: int, world: int) -> list[int]:
    """Frames of ``rank`` when a stream is dealt round-robin (BASELINE configs[3])."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of size {world}")
    return list(range(rank, n_frames, world))


def gather_strips(local_rows, row0: int, row1: int, block: int, height: int, width: int,
                  world: int, group=None):
    """Assemble the full frame from every rank's output rows.

    ``local_rows`` is a torch tensor [ob - oa, width] (this rank's output rows)
    on the device the process group communicates on.  Strips differ by at most
    one block row, so each rank pads to the largest strip and one
    ``all_gather_into_tensor`` moves everything; the result [height, width] is
    returned on every rank.
    """
    import torch
    import torch.distributed as dist

    nbr = block_rows(height, block)
    spans = [strip_rows(nbr, r, world) for r in range(world)]
    rows_of = [min(height, b * block) - min(height, a * block) for a, b in spans]
    cap = max(rows_of)
    pad = torch.zeros((cap, width), dtype=local_rows.dtype, device=local_rows.device)
    pad[: local_rows.shape[0]] = local_rows
    allbuf = torch.empty((world * cap, width), dtype=local_rows.dtype, device=local_rows.device)
    dist.all_gather_into_tensor(allbuf, pad, group=group)
    out = torch.empty((height, width), dtype=local_rows.dtype, device=local_rows.device)
    for r, (a, b) in enumerate(spans):
        oa, ob = min(height, a * block), min(height, b * block)
        out[oa:ob] = allbuf[r * cap: r * cap + (ob - oa)]
    return out


def reconstruct_strip_host(pixels: np.ndarray, mask: np.ndarray, block: int, border: int,
                           rank: int, world: int,
                           strip_fn: Callable[[np.ndarray, np.ndarray, int, int, int], np.ndarray]):
    """Run ``strip_fn`` on this rank's halo rows and return (row0, row1, out_rows).

    ``strip_fn(px_rows, mask_rows, ya, row0, row1)`` reconstructs block rows
    [row0, row1) of the frame given the image rows [ya, ya + len(px_rows)) and
    returns the full-width output rows [row0*B, row1*B) clipped to the frame.
    """
    height = pixels.shape[0]
    row0, row1 = strip_rows(block_rows(height, block), rank, world)
    ya, yb, oa, ob = strip_io_rows(row0, row1, block, border, height)
    out = strip_fn(pixels[ya:yb], mask[ya:yb], ya, row0, row1)
    if out.shape[0] != ob - oa:
        raise ValueError(f"strip_fn returned {out.shape[0]} rows, expected {ob - oa}")
    return row0, row1, out


def engine_strip_fn(params, height: int, width: int, engine=None):
    """strip_fn backed by the CUDA engine (fsr_reconstruct_rows_f32: only the
    strip's halo rows travel to the device), for ``reconstruct_strip_host``."""
    from . import _lib

    eng = engine or _lib.default_engine()

    def run(px_rows, mask_rows, ya, row0, row1):
        full_px = np.zeros((height, width), np.float32)
        full_mk = np.zeros((height, width), np.uint8)
        full_px[ya:ya + px_rows.shape[0]] = px_rows
        full_mk[ya:ya + mask_rows.shape[0]] = mask_rows
        out = np.zeros((height, width), np.float32)
        eng.reconstruct_rows(full_px, full_mk, params, row0, row1, out)
        oa, ob = min(height, row0 * params.block), min(height, row1 * params.block)
        return out[oa:ob]

    return run
