"""Break down the 4K end-to-end host-buffer call (run on the GPU box):
fresh numpy output per call (the public API) vs a reused pageable output vs
caller-pinned buffers, against the device-resident call."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_13926_b200 as fsr  # noqa: E402
from paper_2202_13926_b200 import _lib, frames, synth  # noqa: E402

H, W = (int(x) for x in os.environ.get("SHAPE", "2160x3840").split("x"))
img = synth.frame(H, W, 7, "natural")
mask = frames.quarter_sample_mask(H, W, 42)
px = np.where(mask, img, 0.0)
m8 = mask.astype(np.uint8)
NS = int(os.environ.get("SUPPORT", "32"))
p = _lib.make_params(4, (NS - 4) // 2, 100, precision="fp32")
eng = _lib.default_engine()


def timed(fn, reps=8):
    fn(); fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


out = np.zeros((H, W))
brows = -(-H // 4)
print("api fresh out   %.2f ms" % timed(lambda: fsr.reconstruct(px, mask, 4, NS, 100, precision="fp32")))
print("rows reused out %.2f ms" % timed(lambda: eng.reconstruct_rows(px, m8, p, 0, brows, out)))
hp = torch.from_numpy(px).pin_memory().numpy()
hm = torch.from_numpy(m8).pin_memory().numpy()
ho = torch.zeros((H, W), dtype=torch.float64).pin_memory().numpy()
print("rows pinned     %.2f ms" % timed(lambda: eng.reconstruct_rows(hp, hm, p, 0, brows, ho)))
st = eng.last_stats()
print("kernel_ms %.2f main_ms %.2f" % (st["kernel_ms"], st["main_ms"]))
dp, dm = torch.from_numpy(px).cuda(), torch.from_numpy(m8).cuda()
do = torch.empty_like(dp)
s = torch.cuda.current_stream()
def dev():
    eng.reconstruct_device(dp.data_ptr(), W, dm.data_ptr(), W, H, W, 0, brows, do.data_ptr(), W, p,
                           s.cuda_stream, io="f64")
    s.synchronize()
print("device          %.2f ms" % timed(dev))
t0 = time.perf_counter(); a = np.empty((H, W)); a[:] = 1.0; t1 = time.perf_counter()
print("numpy first-touch of a %d MB array: %.2f ms" % (a.nbytes >> 20, 1e3 * (t1 - t0)))
