"""8-bit binary PGM (P5) read/write with the reference's conventions
(pkg/src/fsrkit/pgm.py:40-79): comments and any whitespace in the header are
accepted on read; writes are byte-stable (maxval 255, no comments, one
newline before the raster, values clamped to [0, 255] and rounded half away
from zero)."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np

from .frames import GrayImage


class PgmError(ValueError):
    """Unreadable or unsupported PGM data."""


_TOKEN = re.compile(rb"(?:\s|#[^\r\n]*(?:\r\n|\r|\n|$))*([^\s#]+)")


def read_pgm(path) -> GrayImage:
    data = Path(path).read_bytes()
    if not data.startswith(b"P5"):
        raise PgmError("not a binary PGM (P5) file")
    pos, vals = 2, []
    for _ in range(3):
        m = _TOKEN.match(data, pos)
        if not m:
            raise PgmError("truncated PGM header")
        try:
            vals.append(int(m.group(1)))
        except ValueError:
            raise PgmError(f"bad PGM header token {m.group(1)!r}") from None
        pos = m.end()
    width, height, maxval = vals
    if width < 1 or height < 1:
        raise PgmError("PGM dimensions must be positive")
    if not 1 <= maxval <= 255:
        raise PgmError("only 8-bit PGM (maxval <= 255) is supported")
    pos += 1  # exactly one whitespace byte separates the header from the raster
    raster = np.frombuffer(data, dtype=np.uint8, count=min(width * height, max(0, len(data) - pos)),
                           offset=min(pos, len(data)))
    if raster.size < width * height:
        raise PgmError("truncated PGM raster")
    return GrayImage(raster.reshape(height, width).astype(np.float64))


def write_pgm(path, image) -> None:
    arr = image.pixels if isinstance(image, GrayImage) else np.asarray(image, dtype=np.float64)
    if arr.ndim != 2:
        raise PgmError("expected a 2D grid")
    q = np.floor(np.clip(arr, 0.0, 255.0) + 0.5).astype(np.uint8)
    Path(path).write_bytes(b"P5\n%d %d\n255\n" % (arr.shape[1], arr.shape[0]) + q.tobytes())
