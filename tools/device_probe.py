"""Device-resident 4K call timed three ways (run on the GPU box): CUDA events
with an L2 flush before each call (bench.py's `value`), CUDA events without
the flush, and wall clock; FSR_CHUNK_TRACE=1 prints the chunk timeline."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_13926_b200 import _lib, frames, synth  # noqa: E402

H, W = (int(x) for x in os.environ.get("SHAPE", "2160x3840").split("x"))
NS = int(os.environ.get("SUPPORT", "32"))
img = synth.frame(H, W, 7, "natural")
mask = frames.quarter_sample_mask(H, W, 42)
px = np.where(mask, img, 0.0)
m8 = mask.astype(np.uint8)
p = _lib.make_params(4, (NS - 4) // 2, 100, precision="fp32")
eng = _lib.default_engine()
brows = -(-H // 4)
dp, dm = torch.from_numpy(px).cuda(), torch.from_numpy(m8).cuda()
do = torch.empty_like(dp)
s = torch.cuda.current_stream()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def dev():
    eng.reconstruct_device(dp.data_ptr(), W, dm.data_ptr(), W, H, W, 0, brows, do.data_ptr(), W, p,
                           s.cuda_stream, io="f64")


def events(do_flush, reps=8):
    ts = []
    for i in range(reps):
        if do_flush:
            flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        dev()
        b.record(s)
        st = eng.last_stats()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return ts, st


for _ in range(3):
    dev()
torch.cuda.synchronize()
for fl in (True, False):
    ts, st = events(fl)
    print("events flush=%d: mean %.2f median %.2f ms  (kernel_ms %.2f, reruns %d, launches %d)"
          % (fl, np.mean(ts), np.median(ts), st["kernel_ms"], st["rerun_blocks"], st["kernel_launches"]))
wall = []
for _ in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev()
    s.synchronize()
    wall.append(1e3 * (time.perf_counter() - t0))
print("wall clock: median %.2f ms" % np.median(wall))
t0 = time.perf_counter()
for _ in range(20):
    dev()
s.synchronize()
print("20 back-to-back calls: %.2f ms each" % (1e3 * (time.perf_counter() - t0) / 20))
