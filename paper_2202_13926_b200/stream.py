"""Sustained frame stream on one GPU (BASELINE configs[3]).

``FrameStream`` pipelines a sequence of quarter-sampled frames through the
C-ABI device entry point (fsr_reconstruct_device_f32): while frame i is being
reconstructed on the compute stream, frame i+1's pixels and mask are copied
host->device on a copy stream and frame i-1's result device->host on a third,
so the steady-state rate is that of the slowest stage (the kernels) rather
than their sum.  Buffers are double-buffered per slot and reused; host staging
is pinned.  torch provides device memory, streams and events (plumbing only);
all compute is libfsr.

One process per GPU: shard a stream across GPUs with ``shard.frame_shard``.
"""

from __future__ import annotations

from typing import Iterable, Iterator, Optional

import numpy as np

from . import _lib


class FrameStream:
    def __init__(self, height: int, width: int, params: "_lib.FsrParamsC", device: int = 0,
                 engine: Optional["_lib.Engine"] = None, depth: int = 2):
        import torch

        self.torch = torch
        self.H, self.W, self.params = int(height), int(width), params
        self.dev = torch.device("cuda", device)
        self.eng = engine or _lib.Engine([device])
        self.depth = max(2, int(depth))
        H, W = self.H, self.W
        with torch.cuda.device(self.dev):
            self.s_in = torch.cuda.Stream(self.dev)
            self.s_run = torch.cuda.Stream(self.dev)
            self.s_out = torch.cuda.Stream(self.dev)
            self.d_px = [torch.empty((H, W), dtype=torch.float32, device=self.dev) for _ in range(self.depth)]
            self.d_mk = [torch.empty((H, W), dtype=torch.uint8, device=self.dev) for _ in range(self.depth)]
            self.d_out = [torch.empty((H, W), dtype=torch.float32, device=self.dev) for _ in range(self.depth)]
            self.ev_in = [torch.cuda.Event() for _ in range(self.depth)]
            self.ev_run = [torch.cuda.Event() for _ in range(self.depth)]
            self.ev_out = [torch.cuda.Event() for _ in range(self.depth)]
        self.h_out = [torch.empty((H, W), dtype=torch.float32).pin_memory() for _ in range(self.depth)]
        self.h2d_bytes_per_frame = H * W * 5
        self.d2h_bytes_per_frame = H * W * 4

    def _submit(self, i: int, px, mk):
        """Enqueue frame i (px, mk: pinned torch tensors [H, W]) into slot i % depth."""
        torch = self.torch
        s = i % self.depth
        n_block_rows = -(-self.H // self.params.block)
        if i >= self.depth:
            # the slot's previous frame must be fully out (D2H done, hence its
            # kernels too) before its device buffers are overwritten
            self.s_in.wait_event(self.ev_out[s])
        with torch.cuda.stream(self.s_in):
            self.d_px[s].copy_(px, non_blocking=True)
            self.d_mk[s].copy_(mk, non_blocking=True)
            self.ev_in[s].record(self.s_in)
        self.s_run.wait_event(self.ev_in[s])
        self.eng.reconstruct_device(self.d_px[s].data_ptr(), self.W, self.d_mk[s].data_ptr(), self.W,
                                    self.H, self.W, 0, n_block_rows, self.d_out[s].data_ptr(), self.W,
                                    self.params, self.s_run.cuda_stream, io="f32")
        self.ev_run[s].record(self.s_run)
        self.s_out.wait_event(self.ev_run[s])
        with torch.cuda.stream(self.s_out):
            self.h_out[s].copy_(self.d_out[s], non_blocking=True)
            self.ev_out[s].record(self.s_out)

    def run(self, frames: Iterable) -> Iterator[np.ndarray]:
        """Yield each frame's reconstruction (a copy) in order.  ``frames``
        yields (pixels, mask) pairs: pinned torch tensors (fastest) or numpy
        arrays (staged through pinned memory here)."""
        torch = self.torch
        pending = []
        for i, (px, mk) in enumerate(frames):
            if not isinstance(px, torch.Tensor):
                px = torch.from_numpy(np.ascontiguousarray(px, dtype=np.float32)).pin_memory()
            if not isinstance(mk, torch.Tensor):
                mk = torch.from_numpy(np.ascontiguousarray(mk).astype(np.uint8, copy=False)).pin_memory()
            if len(pending) == self.depth:
                j = pending.pop(0)
                self.ev_out[j % self.depth].synchronize()
                yield self.h_out[j % self.depth].numpy().copy()
            self._submit(i, px, mk)
            pending.append(i)
        for j in pending:
            self.ev_out[j % self.depth].synchronize()
            yield self.h_out[j % self.depth].numpy().copy()

    def run_timed(self, frames_pinned) -> float:
        """Push all frames (pinned torch tensor pairs) through the pipeline
        without copying results out of the pinned staging; returns seconds of
        wall time from the first H2D to the last D2H (synchronised)."""
        import time

        torch = self.torch
        torch.cuda.synchronize(self.dev)
        t0 = time.perf_counter()
        for i, (px, mk) in enumerate(frames_pinned):
            self._submit(i, px, mk)  # slot reuse is ordered on the device (see _submit)
        torch.cuda.synchronize(self.dev)
        return time.perf_counter() - t0
