"""Reconstruction entry points: the reference's API served by libfsr.so.

  reconstruct_image(sampled, params, reducer, early_stop)
        = fsrkit.reconstruction.reconstruct_image (reconstruction.py:216-290);
          same signature plus engine keywords (precision, devices, argmax).
  reconstruct(image, mask, block, support, iterations, rho, gamma, ...)
        = the explicit-parameter entry of BASELINE.json's north star.
  reconstruct_batch(residuals, models, spectra, freq_weight, gamma, iterations,
                    width, use_tree, stop_thresholds)
        = fsrkit._kernels.reconstruct_batch (_kernels.py:129-149), in place,
          on the GPU (fp64, bitwise equal to the reference).
  run_iterations / reconstruct_block_full / reconstruct_block
        = the traced per-block path (reconstruction.py:138-209); transforms on
          the host with numpy.fft as the reference does, the loop on the GPU.

Precision modes: "fp64" (default: the reference's arithmetic, the validation
mode -- N=32 on the warp-pair register kernel, N=16 on warp16d), "fp32" (the
production mode: fp32 register loop with the near-tie guard, blocks whose
greedy decisions were near-tied re-run in fp64; within the north-star
tolerance) and "fp32_unguarded" (pure fp32 ablation: PSNR
close, max |error| not bounded).  There is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .frames import FsrParams, GrayImage, SampledBlock, SampledImage, n_blocks
from .spectra import WeightSet

REDUCERS = ("tree", "linear")
EARLY_STOP_RELATIVE = 1e-12
DEFAULT_GUARD_TAU = 0.0  # 0: chosen by the engine from N and I (fsr.h)
DEFAULT_GUARD_KAPPA = 0.0  # 0: the engine's default scale term (fsr.h)


def effective_guard_tau(support: int, iterations: int, guard_tau: float = DEFAULT_GUARD_TAU) -> float:
    """The near-tie guard's relative term as the engine applies it (fsr_abi.cu
    guard_tau_for): an explicit tau > 0 as given, else 5e-5 (1e-4 for N=64)."""
    if guard_tau > 0.0:
        return float(guard_tau)
    return 1e-4 if support >= 64 else 2e-4 if support <= 14 else 5e-5


def effective_guard_kappa(iterations: int, guard_kappa: float = DEFAULT_GUARD_KAPPA,
                          support: int = 32) -> float:
    """The guard's scale term (fsr_abi.cu guard_kappa_for): a block is re-run in
    fp64 when b1 - b2 <= tau b1 + kappa sqrt(b1 B0) at some iteration; explicit
    kappa > 0 as given, < 0 off, else 1e-7 * max(0, I/100 - 1) (0 for N <= 14)."""
    if guard_kappa > 0.0:
        return float(guard_kappa)
    if guard_kappa < 0.0 or support <= 14:
        return 0.0
    return 1e-7 * max(0.0, iterations / 100.0 - 1.0)


def _check_reducer(reducer: str) -> bool:
    if reducer not in REDUCERS:
        raise ValueError(f"unknown argmax strategy {reducer!r}, expected one of {REDUCERS}")
    return reducer == "tree"


@dataclass(frozen=True)
class Trace:
    """Per-block selected flat bins (u*N+v; -1 past an early stop) and counts."""

    selections: np.ndarray  # [n_blocks, iterations] int32, partition order
    done: np.ndarray        # [n_blocks] int32
    stats: dict


def reconstruct(image, mask, block: int = 4, support: int = 32, iterations: int = 100,
                rho: float = 0.7, gamma: float = 0.5, *, reducer: str = "tree",
                early_stop: bool = False, precision: str = "fp64", devices=None,
                argmax: str = "redux", guard_tau: float = DEFAULT_GUARD_TAU,
                guard_kappa: float = DEFAULT_GUARD_KAPPA, return_trace: bool = False):
    """Reconstruct the unknown pixels of ``image`` (0..255 scale) given ``mask``.

    ``support`` is the FFT size N = block + 2*border; N - block must be even
    (reference cli.py:186-188).  Supports up to 64 are accepted (the tree
    reducer is limited to N*N <= 1024, like the reference).  Returns float64 for
    float64 input (the reference's pixel type, in every precision: the fp32 loop
    reads the f64 pixels directly) and float32 for float32 input in the fp32
    modes; or ``(array, Trace)`` with ``return_trace``.  ``argmax`` picks the warp
    argmax implementation -- "redux" (redux.sync + ballot, the fastest on
    B200), "shfl" (the paper's shuffle butterfly) or "smem" (the paper's
    shared-memory comparison point); all three give bitwise-identical results.
    """
    _check_reducer(reducer)
    if (support - block) % 2 or support < block:
        raise ValueError("support minus block size must be even and non-negative")
    border = (support - block) // 2
    img = np.asarray(image)
    m = np.asarray(mask)
    if img.ndim != 2 or min(img.shape) < 1:
        raise ValueError("image must be a 2D grid with at least one pixel")
    if m.shape != img.shape:
        raise ValueError("image and mask dimensions differ")
    # every precision takes the reference's f64 pixels as they are (the fp32
    # kernels' prologue reads and transforms them in fp64); f32 input stays f32
    io = np.float32 if (img.dtype == np.float32 and precision != "fp64") else np.float64
    img = np.ascontiguousarray(img, dtype=io)
    m = np.ascontiguousarray(m, dtype=bool)
    params = _lib.make_params(block, border, iterations, rho, gamma, reducer, early_stop,
                              precision, argmax, guard_tau, guard_kappa=guard_kappa)
    eng = _lib.default_engine(devices)
    sel = done = None
    if return_trace:
        nb = n_blocks(img.shape[0], img.shape[1], block)
        sel = np.empty((nb, max(iterations, 1)), np.int32)
        done = np.empty(nb, np.int32)
    out = eng.reconstruct(img, m, params, sel, done)
    if return_trace:
        return out, Trace(sel[:, :iterations], done, eng.last_stats())
    return out


def reconstruct_image(sampled: SampledImage, params: FsrParams, reducer: str = "tree",
                      early_stop: bool = False, *, precision: str = "fp64", devices=None,
                      argmax: str = "redux", guard_tau: float = DEFAULT_GUARD_TAU,
                      guard_kappa: float = DEFAULT_GUARD_KAPPA) -> GrayImage:
    """Drop-in for fsrkit.reconstruct_image: every target block reconstructed
    independently on the GPU and stitched; empty-support blocks get the mean of
    the known samples ("no known samples" ValueError if there is none).
    The result is identical for any ``devices`` set."""
    _check_reducer(reducer)
    out = reconstruct(sampled.image.pixels, sampled.mask, params.block, params.support,
                      params.iterations, params.rho, params.gamma, reducer=reducer,
                      early_stop=early_stop, precision=precision, devices=devices,
                      argmax=argmax, guard_tau=guard_tau, guard_kappa=guard_kappa)
    return GrayImage(out)


# ------------------------------------------------------------ loop operator
def reconstruct_batch(residuals, models, spectra, freq_weight, gamma, iterations,
                      width=32, use_tree=True, stop_thresholds=None, *, devices=None,
                      trace=False):
    """GPU twin of _kernels.reconstruct_batch: in place on complex128 arrays.

    Blocks whose spectrum has W[0,0].real <= 0 are skipped (model stays zero).
    With ``trace`` returns (selections, objectives, ties, done) [count, I]."""
    if width != 32:
        raise ValueError("lane group width is fixed at 32")
    count = residuals.shape[0]
    n = residuals.shape[1]
    p = _lib.make_params(iterations=iterations, gamma=gamma,
                         reducer="tree" if use_tree else "linear", precision="fp64")
    eng = _lib.default_engine(devices)
    it = max(iterations, 1)
    sel = np.zeros((count, it), np.int32) if trace else None
    obj = np.zeros((count, it), np.float64) if trace else None
    ties = np.zeros((count, it), np.uint8) if trace else None
    done = np.zeros(count, np.int32) if trace else None
    eng.iterate_spectra(residuals, models, spectra, np.asarray(freq_weight).reshape(n, n), p,
                        stop_thresholds, sel, obj, ties, done)
    if trace:
        return sel, obj, ties, done
    return None


@dataclass
class BlockState:
    model: np.ndarray
    residual: np.ndarray
    nu: int = 0


@dataclass(frozen=True)
class BlockResult:
    output: np.ndarray
    objectives: np.ndarray
    selections: np.ndarray
    ties: np.ndarray
    empty_support: bool
    iterations_run: int


def init_residual(block: SampledBlock, weights: WeightSet) -> BlockState:
    if block.support != weights.support:
        raise ValueError("block and weight dimensions differ")
    r = np.fft.fft2(block.signal * weights.spatial)
    return BlockState(model=np.zeros_like(r), residual=r, nu=0)


def _loop(residual, model, weights, gamma, iterations, reducer, thr):
    use_tree = _check_reducer(reducer)
    R = residual.reshape(1, *residual.shape)
    G = model.reshape(1, *model.shape)
    sel, obj, ties, done = reconstruct_batch(
        R, G, weights.spectrum.reshape(1, *residual.shape), weights.frequency, gamma,
        iterations, 32, use_tree, np.array([thr]), trace=True)
    d = int(done[0])
    return d, obj[0, :d], sel[0, :d].astype(np.int64), ties[0, :d].astype(bool)


def run_iterations(state: BlockState, weights: WeightSet, gamma: float, iterations: int,
                   reducer: str = "tree") -> int:
    """Advance ``state`` in place by ``iterations`` greedy steps on the GPU."""
    if not (state.residual.flags.c_contiguous and state.model.flags.c_contiguous):
        raise ValueError("state arrays must be C-contiguous")
    if weights.spectrum[0, 0].real <= 0.0:
        return 0
    d, _, _, _ = _loop(state.residual, state.model, weights, gamma, iterations, reducer, 0.0)
    state.nu += d
    return d


def reconstruct_block_full(block: SampledBlock, weights: WeightSet, params, reducer: str = "tree",
                           early_stop: bool = False) -> BlockResult:
    """One support window with its per-iteration trace (selections, objectives, ties)."""
    _check_reducer(reducer)
    s = weights.support
    if block.support != s:
        raise ValueError("block and weight dimensions differ")
    if weights.spectrum[0, 0].real <= 0.0:
        return BlockResult(np.zeros((s, s)), np.zeros(0), np.zeros(0, np.int64),
                           np.zeros(0, bool), True, 0)
    residual = np.fft.fft2(block.signal * weights.spatial)
    model = np.zeros((s, s), dtype=np.complex128)
    thr = 0.0
    if early_stop:
        sig = block.signal
        thr = EARLY_STOP_RELATIVE * float(np.sum((sig.real ** 2 + np.imag(sig) ** 2) * weights.spatial))
    d, obj, sel, ties = _loop(residual, model, weights, params.gamma, params.iterations, reducer, thr)
    g = np.fft.ifft2(model)
    if not np.iscomplexobj(block.signal):
        g = g.real
    return BlockResult(np.where(block.mask, block.signal, g), obj, sel, ties, False, d)


def reconstruct_block(block: SampledBlock, weights: WeightSet, params, reducer: str = "tree"):
    return reconstruct_block_full(block, weights, params, reducer).output
