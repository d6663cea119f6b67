"""Synthetic test frames (no datasets offline): the reference test suite's
natural-image recipe (pkg/tests/conftest.py:8-25: 1/f^2 clouds, gradient,
disc edge, textured band), cropped to non-square frames as BASELINE.md §3
prescribes, plus a uniform-noise frame."""

from __future__ import annotations

import numpy as np


def natural_image(size: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal((size, size))
    fy = np.fft.fftfreq(size)[:, None]
    fx = np.fft.fftfreq(size)[None, :]
    smooth = np.fft.ifft2(np.fft.fft2(noise) / (1.0 + (np.hypot(fy, fx) * size / 6.0) ** 2)).real
    smooth = (smooth - smooth.min()) / np.ptp(smooth)
    yy, xx = np.mgrid[0:size, 0:size] / size
    img = 30.0 + 150.0 * smooth + 35.0 * yy
    img = np.where((yy - 0.35) ** 2 + (xx - 0.6) ** 2 < 0.04, 0.5 * img + 110.0, img)
    band = (yy > 0.7) & (yy < 0.85)
    img = img + band * 12.0 * np.sin(2 * np.pi * 14 * xx) * np.sin(2 * np.pi * 9 * yy)
    return np.clip(img, 0.0, 255.0)


def frame(height: int, width: int, seed: int, kind: str = "natural") -> np.ndarray:
    if kind == "uniform":
        return np.random.default_rng(seed).uniform(0.0, 255.0, (height, width))
    return np.ascontiguousarray(natural_image(max(height, width), seed)[:height, :width])
