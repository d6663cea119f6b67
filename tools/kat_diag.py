"""Where does guarded fp32 miss the reference on a golden frame?  For the blocks
whose pixels differ by more than the tolerance: the first iteration where the
fp32 path parts from the reference's (mirror-aware) and the reference's own
relative top-2 objective gap there.

    python tools/kat_diag.py [golden-name] [tau]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import golden_image  # noqa: E402
from oracle import port as oracle  # noqa: E402  (checker only)

import paper_2202_13926_b200 as fsr  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "acc6_512_s16"
    tau = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
    d = golden_image(name)
    B, L, I = int(d["block"]), int(d["border"]), int(d["iterations"])
    N = B + 2 * L
    px, mask, ref = d["sampled"], d["mask"], d["out_tree"]
    out, tr = fsr.reconstruct(px, mask, B, N, I, reducer="tree", precision="fp32",
                              return_trace=True, guard_tau=tau)
    _, t64 = fsr.reconstruct(px, mask, B, N, I, reducer="tree", precision="fp64",
                             return_trace=True)
    err = np.abs(out - ref)
    H, W = px.shape
    bc = -(-W // B)
    print(f"{name}: N={N} I={I} tau={tau:g} max|d|={err.max():.4f} gray "
          f"reruns={tr.stats['rerun_blocks']}/{tr.stats['blocks']}")
    bad = np.argwhere(err > 0.05)
    blocks = sorted({(int(y) // B) * bc + int(x) // B for y, x in bad})
    for b in blocks[:20]:
        r, c = divmod(b, bc)
        e = err[r * B:(r + 1) * B, c * B:(c + 1) * B].max()
        s32 = tr.selections[b]
        s64 = t64.selections[b]
        same = np.all(s32 == s64) or np.all(s32 == oracle.mirror_index(s64, N))
        split, f, gap = oracle.coemaximal_split(px, mask, B, L, I, 0.7, 0.5, "tree", b, s32)
        print(f"block {b} ({r},{c}) max|d|={e:.4f} seq==fp64:{same} first-div it={f} "
              f"ref-gap={gap:.3e}")


if __name__ == "__main__":
    main()
