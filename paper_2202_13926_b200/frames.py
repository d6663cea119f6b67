"""Host-side image, mask and parameter types -- the reference's data contract.

Mirrors fsrkit's public types so callers switch packages without changes:
  GrayImage      core.py:12-42      (f64 pixels, 2-D, finite, read-only)
  FsrParams      core.py:45-85      (same fields, defaults and ValueErrors)
  BlockDescriptor, block_partition  core.py:88-103, 136-162
  SampledBlock   core.py:106-133
  SampledImage   sampling.py:32-50  (bool mask, unknown pixels zero)
  quarter_sample / mean_fill / splitmix64 / extract_support_block
                 sampling.py:18-107 (SplitMix64 quarter sampling, bit-exact)
These are input validation and test-input generation; the reconstruction
itself runs in libfsr.so on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

LANE_GROUP_WIDTH = 32
MAX_BLOCK_RECORDS = LANE_GROUP_WIDTH * LANE_GROUP_WIDTH  # tree reducer capacity


@dataclass(frozen=True)
class GrayImage:
    """Float64 grayscale image on the nominal 0..255 scale (unquantised)."""

    pixels: np.ndarray

    def __post_init__(self):
        px = np.array(self.pixels, dtype=np.float64, order="C")
        if px.ndim != 2 or min(px.shape) < 1:
            raise ValueError("image must be a 2D grid with at least one pixel")
        if not np.isfinite(px).all():
            raise ValueError("image pixels must be finite")
        px.setflags(write=False)
        object.__setattr__(self, "pixels", px)

    @property
    def height(self) -> int:
        return self.pixels.shape[0]

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    @property
    def shape(self) -> tuple[int, int]:
        return self.pixels.shape


@dataclass(frozen=True)
class FsrParams:
    """Reconstruction parameters; support side = block + 2 * border.

    ``threads`` is accepted for compatibility and ignored: work is spread
    over GPU warps, not host threads.
    """

    block: int = 4
    border: int = 6
    rho: float = 0.7
    gamma: float = 0.5
    iterations: int = 200
    threads: int = 1
    seed: int = 0

    def __post_init__(self):
        checks = (
            (self.block >= 1, "target block size must be at least 1"),
            (self.border >= 0, "border must be non-negative"),
            (0.0 < self.rho < 1.0, "decay factor rho must lie in (0, 1)"),
            (0.0 < self.gamma <= 1.0, "compensation factor gamma must lie in (0, 1]"),
            (self.iterations >= 0, "iteration count must be non-negative"),
            (self.threads >= 1, "thread count must be at least 1"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)
        s = self.support
        if s * s > MAX_BLOCK_RECORDS:
            raise ValueError(f"support block {s}x{s} exceeds the {MAX_BLOCK_RECORDS}-lane "
                             "reduction capacity")

    @property
    def support(self) -> int:
        return self.block + 2 * self.border


@dataclass(frozen=True)
class BlockDescriptor:
    target_row: int
    target_col: int
    height: int
    width: int
    support_row: int
    support_col: int


@dataclass(frozen=True)
class SampledBlock:
    """Square support window with its known-sample mask (unknown = 0)."""

    signal: np.ndarray
    mask: np.ndarray

    def __post_init__(self):
        sig = np.asarray(self.signal)
        if not np.iscomplexobj(sig):
            sig = sig.astype(np.float64)
        m = np.asarray(self.mask, dtype=bool)
        if sig.ndim != 2 or sig.shape[0] != sig.shape[1]:
            raise ValueError("support block must be square")
        if m.shape != sig.shape:
            raise ValueError("signal and mask dimensions differ")
        if np.any(sig[~m] != 0):
            raise ValueError("unknown positions must hold zero")
        object.__setattr__(self, "signal", sig)
        object.__setattr__(self, "mask", m)

    @property
    def support(self) -> int:
        return self.signal.shape[0]


@dataclass(frozen=True)
class SampledImage:
    """Image plus boolean known-pixel mask; unknown pixels must hold zero."""

    image: GrayImage
    mask: np.ndarray

    def __post_init__(self):
        m = np.array(self.mask, dtype=bool, order="C")
        if m.shape != self.image.shape:
            raise ValueError("image and mask dimensions differ")
        if np.any(self.image.pixels[~m] != 0):
            raise ValueError("unknown pixels must hold zero")
        m.setflags(write=False)
        object.__setattr__(self, "mask", m)

    @property
    def shape(self) -> tuple[int, int]:
        return self.image.shape


def block_partition(height: int, width: int, params: FsrParams) -> list[BlockDescriptor]:
    """Row-major B x B target tiles (edge tiles truncated), supports shifted by -border."""
    if height < 1 or width < 1:
        raise ValueError("image must have at least one pixel")
    b, L = params.block, params.border
    return [BlockDescriptor(r, c, min(b, height - r), min(b, width - c), r - L, c - L)
            for r in range(0, height, b) for c in range(0, width, b)]


def n_blocks(height: int, width: int, block: int) -> int:
    return -(-height // block) * -(-width // block)


# SplitMix64 constants (sampling.py:18-20)
_INC = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """Outputs 1..count of SplitMix64 seeded with ``seed`` mod 2**64."""
    z = np.uint64(seed & (2**64 - 1)) + np.arange(1, count + 1, dtype=np.uint64) * _INC
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def quarter_sample_mask(height: int, width: int, seed: int) -> np.ndarray:
    """One known pixel per 2x2 cell (edge cells 1x2/2x1/1x1), cell c uses draw c."""
    rows, cols = (height + 1) // 2, (width + 1) // 2
    draws = splitmix64(seed, rows * cols).reshape(rows, cols)
    ch = np.where(np.arange(rows) == rows - 1, 2 - height % 2, 2).astype(np.uint64)[:, None]
    cw = np.where(np.arange(cols) == cols - 1, 2 - width % 2, 2).astype(np.uint64)[None, :]
    pick = draws % (ch * cw)
    yy = (2 * np.arange(rows)[:, None] + (pick // cw).astype(np.int64)).ravel()
    xx = (2 * np.arange(cols)[None, :] + (pick % cw).astype(np.int64)).ravel()
    mask = np.zeros((height, width), dtype=bool)
    mask[yy, xx] = True
    return mask


def quarter_sample(original: GrayImage, seed: int) -> SampledImage:
    mask = quarter_sample_mask(original.height, original.width, seed)
    return SampledImage(GrayImage(np.where(mask, original.pixels, 0.0)), mask)


def mean_fill(sampled: SampledImage) -> GrayImage:
    known = int(np.count_nonzero(sampled.mask))
    if known == 0:
        raise ValueError("no known samples")
    mean = float(sampled.image.pixels.sum()) / known
    return GrayImage(np.where(sampled.mask, sampled.image.pixels, mean))


def extract_support_block(sampled: SampledImage, desc: BlockDescriptor, support: int) -> SampledBlock:
    """Support window; positions outside the image are unknown (zero)."""
    h, w = sampled.shape
    sig = np.zeros((support, support))
    m = np.zeros((support, support), dtype=bool)
    y0, x0 = desc.support_row, desc.support_col
    ya, yb = max(y0, 0), min(y0 + support, h)
    xa, xb = max(x0, 0), min(x0 + support, w)
    if yb > ya and xb > xa:
        sig[ya - y0:yb - y0, xa - x0:xb - x0] = sampled.image.pixels[ya:yb, xa:xb]
        m[ya - y0:yb - y0, xa - x0:xb - x0] = sampled.mask[ya:yb, xa:xb]
    return SampledBlock(signal=sig, mask=m)


def quarter_sample_device(image, seed: int, engine=None, stream=None):
    """``quarter_sample`` on the GPU (sampling.py:53-80, bit-exact): ``image`` is
    a float32 CUDA tensor [H, W]; returns (sampled, mask) CUDA tensors (float32,
    uint8) produced by libfsr's fsr_quarter_sample_device."""
    import torch

    from . import _lib

    img = image.contiguous()
    h, w = img.shape
    eng = engine or _lib.default_engine([img.device.index or 0])
    sampled = torch.empty_like(img)
    mask = torch.empty((h, w), dtype=torch.uint8, device=img.device)
    st = stream or torch.cuda.current_stream(img.device)
    eng.quarter_sample_device(img.data_ptr(), w, h, w, seed, sampled.data_ptr(), w, mask.data_ptr(), w,
                              st.cuda_stream)
    return sampled, mask
