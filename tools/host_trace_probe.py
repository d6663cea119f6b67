"""Host-side timeline of one 4K public-API call (run on the GPU box):
FSR_HOST_TRACE=1 FSR_CHUNK_TRACE=1 python tools/host_trace_probe.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_13926_b200 as fsr  # noqa: E402
from paper_2202_13926_b200 import frames, synth  # noqa: E402

H, W = 2160, 3840
img = synth.frame(H, W, 7, "natural")
mask = frames.quarter_sample_mask(H, W, 42)
px = np.where(mask, img, 0.0)
for _ in range(4):
    out = fsr.reconstruct(px, mask, 4, 32, 100, precision="fp32")
del out
sys.stderr.flush()
print("---- traced call", file=sys.stderr, flush=True)
t0 = time.perf_counter()
out = fsr.reconstruct(px, mask, 4, 32, 100, precision="fp32")
t1 = time.perf_counter()
sys.stderr.flush()
print(f"python call: {1e3 * (t1 - t0):.3f} ms", file=sys.stderr, flush=True)
