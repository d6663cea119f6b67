"""FFT-free spatial-domain oracle on the GPU.

The reference validates its frequency-domain fast path against a
direct-summation oracle (pkg/src/fsrkit/oracle.py:25-132, acceptance
criterion 1 in pkg/tests/test_acceptance.py:32-91).  This module keeps that
oracle's API -- ``oracle_reconstruct_traced(block, weights, params)`` returning
an ``OracleRun`` and ``oracle_reconstruct`` -- served by the
``spatial_oracle_kernel`` (csrc/fsr_spatial.cuh) through ``fsr_spatial_oracle``:
every iteration projects the weighted residual onto all S^2 basis images by
explicit summation, takes the first maximum of wf*|proj|^2, and recomputes
the model, residual and weighted energy from scratch.  Supports S <= 16 (the
reference's stated scope, "intended for supports up to 16").

It shares no code with the frequency-domain kernels (no FFT, no residual
spectrum, no shifted weight spectrum), so agreement between the two GPU
routes is an independent check of the engine's math.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .frames import SampledBlock
from .spectra import WeightSet

# objectives this close to the maximum count as tied (oracle.py:23)
TIE_RELATIVE = 1e-9


@dataclass(frozen=True)
class OracleRun:
    """Trace of a full spatial-domain reconstruction (oracle.py:104-112)."""

    output: np.ndarray
    objectives: np.ndarray
    selections: np.ndarray   # flat frequency index per iteration
    ties: np.ndarray
    energies: np.ndarray     # weighted residual energy, length iterations + 1


def oracle_batch(signals, masks, spatial, frequency, gamma: float, iterations: int, devices=None):
    """Spatial oracle on [count, S, S] blocks in one launch (one CTA per block)."""
    eng = _lib.default_engine(devices)
    return eng.spatial_oracle(signals, masks, spatial, frequency, gamma, iterations)


def oracle_reconstruct_traced(block: SampledBlock, weights: WeightSet, params) -> OracleRun:
    """Reference reconstruction with the full per-iteration trace (oracle.py:115-132)."""
    w = np.asarray(weights.spatial, dtype=np.float64)
    if float(np.sum(w)) <= 0.0:
        raise ValueError("empty support")  # oracle.py:86-87
    out, obj, sel, ties, en = oracle_batch(np.asarray(block.signal)[None], np.asarray(block.mask)[None],
                                           w[None], weights.frequency, params.gamma,
                                           params.iterations)
    return OracleRun(out[0], obj[0], sel[0].astype(np.int64), ties[0], en[0])


def oracle_reconstruct(block: SampledBlock, weights: WeightSet, params) -> np.ndarray:
    """Reference reconstruction; known samples are copied through (oracle.py:135-137)."""
    return oracle_reconstruct_traced(block, weights, params).output
