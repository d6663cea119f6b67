"""Where the public API's host time goes around the C call (run on the GPU box):
python tools/py_overhead_probe.py -- median of 8 calls each for the numpy API
(fsr.reconstruct), the Engine method, the bare ctypes call on pre-made buffers,
and the pieces the wrappers add (params, output allocation)."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_13926_b200 as fsr  # noqa: E402
from paper_2202_13926_b200 import _lib, frames, synth  # noqa: E402

H, W = 2160, 3840
img = synth.frame(H, W, 7, "natural")
mask = frames.quarter_sample_mask(H, W, 42)
px = np.ascontiguousarray(np.where(mask, img, 0.0))
m8 = mask.view(np.uint8)
p = _lib.make_params(4, 14, 100, precision="fp32")
eng = _lib.default_engine()
L = eng._L


def med(fn, n=8):
    fn()
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        r = fn()
        ts.append(1e3 * (time.perf_counter() - t0))
        del r
    return float(np.median(ts))


out = np.empty((H, W))
_lib.load().fsr_pin_host(out.ctypes.data, out.nbytes)


def bare():
    rc = L.fsr_reconstruct_f64(eng._h, ctypes.byref(p), px.ctypes.data_as(ctypes.c_void_p),
                               m8.ctypes.data_as(ctypes.c_void_p), H, W,
                               out.ctypes.data_as(ctypes.c_void_p), None, None)
    assert rc == 0


print("fsr.reconstruct        %.3f ms" % med(lambda: fsr.reconstruct(px, mask, 4, 32, 100, precision="fp32")))
print("Engine.reconstruct     %.3f ms" % med(lambda: eng.reconstruct(px, mask, p)))
print("bare ctypes (pinned)   %.3f ms" % med(bare))
print("make_params            %.3f ms" % med(lambda: _lib.make_params(4, 14, 100, precision="fp32"), 50))
print("new_image              %.3f ms" % med(lambda: _lib.new_image((H, W), np.float64), 50))
st = eng.last_stats()
print("last call kernel_ms    %.3f ms" % st["kernel_ms"])
