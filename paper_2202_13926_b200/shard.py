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

The one frame-wide quantity is the empty-support fill (reconstruction.py:
236-237: the mean of ALL known samples of the frame).  A rank that holds the
whole frame computes it exactly as the reference does (``frame_fill``); the
strips then receive it as an argument, so a rank's blocks never depend on
which rows it happens to hold.

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


def frame_fill(pixels: np.ndarray, mask: np.ndarray) -> float:
    """The reference's empty-support value (reconstruction.py:236-237): the sum of
    the frame's pixels over the number of known samples, in the same numpy
    arithmetic (so the bits match); NaN when the frame has no known sample (the
    engine then raises "no known samples" if a block needs the fill)."""
    known = int(np.count_nonzero(mask))
    return float(np.asarray(pixels, dtype=np.float64).sum()) / known if known else float("nan")


def reconstruct_strip_host(pixels: np.ndarray, mask: np.ndarray, block: int, border: int,
                           rank: int, world: int,
                           strip_fn: Callable[..., np.ndarray], fill: float | None = None):
    """Run ``strip_fn`` on this rank's halo rows and return (row0, row1, out_rows).

    ``strip_fn(px_rows, mask_rows, ya, row0, row1, fill)`` reconstructs block
    rows [row0, row1) of the frame given the image rows [ya, ya + len(px_rows))
    and the frame-wide empty-support value ``fill``, and returns the full-width
    output rows [row0*B, row1*B) clipped to the frame.  ``fill`` defaults to
    ``frame_fill(pixels, mask)`` (every rank holds the frame here).
    """
    height = pixels.shape[0]
    row0, row1 = strip_rows(block_rows(height, block), rank, world)
    ya, yb, oa, ob = strip_io_rows(row0, row1, block, border, height)
    if fill is None:
        fill = frame_fill(pixels, mask)
    out = strip_fn(pixels[ya:yb], mask[ya:yb], ya, row0, row1, fill)
    if out.shape[0] != ob - oa:
        raise ValueError(f"strip_fn returned {out.shape[0]} rows, expected {ob - oa}")
    return row0, row1, out


def engine_strip_fn(params, height: int, width: int, engine=None):
    """strip_fn backed by the CUDA engine (fsr_reconstruct_rows_f32/_f64: only
    the strip's halo rows are read and travel to the device; the empty-support
    value comes in as ``fill``), for ``reconstruct_strip_host``."""
    from . import _lib

    eng = engine or _lib.default_engine()

    def run(px_rows, mask_rows, ya, row0, row1, fill):
        io = np.float32 if px_rows.dtype == np.float32 else np.float64
        full_px = np.zeros((height, width), io)
        full_mk = np.zeros((height, width), np.uint8)
        full_px[ya:ya + px_rows.shape[0]] = px_rows
        full_mk[ya:ya + mask_rows.shape[0]] = mask_rows
        out = np.zeros((height, width), io)
        eng.reconstruct_rows(full_px, full_mk, params, row0, row1, out, fill=fill)
        oa, ob = min(height, row0 * params.block), min(height, row1 * params.block)
        return out[oa:ob]

    return run
