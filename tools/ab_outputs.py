"""Output digests of a fixed set of calls (run on the GPU box), for bitwise A/B
of two library builds: FSR_LIBFSR=<lib> python tools/ab_outputs.py > a.txt;
diff the two files.  Covers the register kernels' supports in guarded fp32
and fp64 on f64 pixels, both reducers."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_13926_b200 as fsr  # noqa: E402
from paper_2202_13926_b200 import frames, synth  # noqa: E402

CASES = [  # (H, W, N, I, reducer, precision)
    (2160, 3840, 32, 100, "tree", "fp32"),
    (540, 960, 32, 100, "linear", "fp32"),
    (540, 960, 32, 60, "tree", "fp64"),
    (540, 960, 16, 100, "tree", "fp32"),
    (540, 960, 16, 100, "tree", "fp64"),
    (540, 960, 64, 100, "linear", "fp32"),
    (270, 480, 64, 60, "linear", "fp64"),
    (540, 960, 24, 100, "tree", "fp32"),
    (540, 960, 8, 100, "tree", "fp32"),
    (540, 960, 8, 100, "linear", "fp64"),
    (540, 960, 4, 100, "tree", "fp32"),
    (540, 960, 4, 200, "linear", "fp64"),
    (540, 960, 12, 100, "tree", "fp32"),
    (270, 480, 32, 100, "tree", "fp32"),
    (540, 960, 32, 200, "tree", "fp32"),
    (540, 960, 16, 200, "tree", "fp32"),
    (540, 960, 64, 200, "linear", "fp32"),
    (540, 960, 24, 200, "tree", "fp32"),
]
for H, W, N, I, red, prec in CASES:
    img = synth.frame(H, W, 7, "natural")
    mask = frames.quarter_sample_mask(H, W, 42)
    px = np.where(mask, img, 0.0)
    out = fsr.reconstruct(px, mask, 4, N, I, reducer=red, precision=prec)
    h = hashlib.sha1(np.ascontiguousarray(out).tobytes()).hexdigest()[:16]
    print(f"{H}x{W} N={N} I={I} {red} {prec}: {h}")
