"""Replay of the fp64 re-runs' unambiguous prefix (fsr_pair64.cuh): the guarded
N=32 output with replay against the same call without it (full fp64 re-runs),
and the reference.  python tools/replay_check.py [H W I]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import port as oracle  # noqa: E402  (checker only)

from paper_2202_13926_b200 import _lib, frames, synth  # noqa: E402


def engine(replay_min):
    os.environ["FSR_REPLAY_MIN"] = str(replay_min)
    e = _lib.Engine([0])
    del os.environ["FSR_REPLAY_MIN"]
    return e


def main():
    H, W, I = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (540, 960, 200)
    N = int(sys.argv[4]) if len(sys.argv) > 4 else 32
    img = synth.frame(H, W, 7, "natural")
    mask = frames.quarter_sample_mask(H, W, 42)
    px = np.where(mask, img, 0.0)
    red = "linear" if N == 64 else "tree"
    p = _lib.make_params(4, (N - 4) // 2, I, precision="fp32", reducer=red)
    on, off = engine(1), engine(0)
    o_on = on.reconstruct(px, mask, p)
    st_on = on.last_stats()
    o_off = off.reconstruct(px, mask, p)
    st_off = off.last_stats()
    diff = np.abs(o_on - o_off)
    print(f"{H}x{W} N={N} I={I}: re-runs {st_on['rerun_blocks']} / {st_off['rerun_blocks']}, "
          f"pixels differing {int((diff > 0).sum())}, max |d| {diff.max():.3e}, "
          f"kernel ms {st_on['kernel_ms']:.2f} (replay) vs {st_off['kernel_ms']:.2f}")
    if H * W <= 600 * 1000:
        ref = oracle.reconstruct_image(px, mask, 4, (N - 4) // 2, I, 0.7, 0.5, red)
        print(f"  vs reference: replay max |d| {np.abs(o_on - ref).max() / 255:.3e}, "
              f"full re-run {np.abs(o_off - ref).max() / 255:.3e} (0..1)")


if __name__ == "__main__":
    main()
