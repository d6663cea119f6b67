"""Guarded fp32 vs the reference restatement on the SAME f32-rounded inputs, by
support and iteration count (does the near-tie guard hold beyond I=100?).

    python tools/guard_check.py [size] [seed]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import port as oracle  # noqa: E402  (checker only)

import paper_2202_13926_b200 as fsr  # noqa: E402


def main():
    size = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    kind = os.environ.get("KIND", "natural")
    rho, gamma = float(os.environ.get("RHO", "0.7")), float(os.environ.get("GAMMA", "0.5"))
    img = oracle.synthetic_frame(size, size, seed, kind)
    sampled, mask = oracle.quarter_sample(img, 42)
    s32 = sampled.astype(np.float32)
    cases = [tuple(int(x) for x in c.split(":")) for c in
             (sys.argv[3].split(",") if len(sys.argv) > 3 else ["16:100", "16:200", "16:500", "32:100",
                                                              "32:200", "32:500", "64:100", "64:200",
                                                              "64:500"])]
    taus = [float(t) for t in (sys.argv[4].split(",") if len(sys.argv) > 4 else ["0"])]
    for N, I in cases:
        B = 4
        red = "linear" if N == 64 else "tree"
        L = (N - B) // 2
        ref32 = oracle.reconstruct_image(s32.astype(np.float64), mask, B, L, I, rho, gamma, red)
        for tau in taus:
            out, tr = fsr.reconstruct(s32, mask, B, N, I, rho, gamma, reducer=red, precision="fp32",
                                      argmax="redux", return_trace=True, guard_tau=tau)
            err = np.abs(out.astype(np.float64) - ref32)
            bad = int((err > 0.255).sum())
            print(f"rho={rho} gamma={gamma} N={N} I={I} tau={tau:g} (0 = auto): max|d|={err.max():.4f} (tol 0.255) pixels over "
                  f"tol={bad} reruns={tr.stats['rerun_blocks']}/{tr.stats['blocks']}", flush=True)


if __name__ == "__main__":
    main()
