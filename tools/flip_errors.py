"""Per-block max pixel error of the unguarded fp32 loop against fp64 (GPU), on
the frames of tools/guard_scale_study.py, and of the guarded loop for each
(tau, kappa) in GUARDS="tau:kappa,..." (0 = engine default, kappa < 0 = off),
for calibrating the guard.

    GUARDS=0:0,5e-5:1e-7 python tools/flip_errors.py <npz-out> frame:N:I [...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from guard_scale_study import frame  # noqa: E402

import paper_2202_13926_b200 as fsr  # noqa: E402


def block_max(err, B):
    H, W = err.shape
    hp, wp = -(-H // B) * B, -(-W // B) * B
    e = np.zeros((hp, wp))
    e[:H, :W] = err
    return e.reshape(hp // B, B, wp // B, B).max(axis=(1, 3)).ravel()


def main():
    out = {}
    for case in sys.argv[2:]:
        name, N, I = case.split(":")
        N, I = int(N), int(I)
        px, mask = frame(name)
        red = "linear" if N == 64 else "tree"
        o64 = fsr.reconstruct(px, mask, 4, N, I, reducer=red, precision="fp64")
        o32 = fsr.reconstruct(px, mask, 4, N, I, reducer=red, precision="fp32_unguarded")
        e = block_max(np.abs(o32 - o64), 4)
        out[f"{name}_{N}_{I}"] = e
        print(f"{case}: unguarded max {e.max():.4f} (blocks > 0.1: {(e > 0.1).sum()})", flush=True)
        for g in os.environ.get("GUARDS", "0:0").split(","):
            tau, kappa = (float(x) for x in g.split(":"))
            og, tr = fsr.reconstruct(px, mask, 4, N, I, reducer=red, precision="fp32",
                                     return_trace=True, guard_tau=tau, guard_kappa=kappa)
            eg = block_max(np.abs(og - o64), 4)
            out[f"{name}_{N}_{I}_g{g}"] = eg
            st = tr.stats
            print(f"   tau={tau:g} kappa={kappa:g}: max {eg.max():.4f} (> 0.1: {(eg > 0.1).sum()}) "
                  f"reruns {100 * st['rerun_blocks'] / st['blocks']:.1f} %", flush=True)
    np.savez_compressed(sys.argv[1], **out)


if __name__ == "__main__":
    main()
