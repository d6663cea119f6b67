"""Full-frame parity record at the BASELINE configs.

Runs the GPU engine and the CPU restatement of the reference (oracle/port.py,
pinned bitwise to fsrkit by tests/golden) on the SAME whole frame -- every
block, no sampling -- and reports, per precision:

  fp64 validation: per-block selection sequences equal / equal modulo the
      conjugate mirror / diverged (each divergence checked against the
      reference's co-maximal-split rule, pkg/tests/test_acceptance.py:73-87),
      max |d| on the 0..1 scale;
  fp32 production (f64 pixels in, as the reference takes them): max |d|
      (0..1) and dPSNR against the reference output, re-run blocks.

  python tools/full_frame_parity.py --shape 1080x1920 [--shape 2160x3840]
        [--out gpurun_out/full_frame_parity.json]

Test infrastructure: the oracle is the checker here, never the thing measured.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(H, W, N, I, B, kind, reducer, splits_cap):
    import paper_2202_13926_b200 as fsr
    from oracle import port as oracle

    L = (N - B) // 2
    img = oracle.synthetic_frame(H, W, 7, kind)
    sampled, mask = oracle.quarter_sample(img, 42)
    t0 = time.time()
    ref, rtr = oracle.reconstruct_image(sampled, mask, B, L, I, 0.7, 0.5, reducer, trace=True)
    t_cpu = time.time() - t0
    rec = {"shape": [H, W], "N": N, "B": B, "iterations": I, "image": kind, "reducer": reducer,
           "blocks": int(rtr["sel"].shape[0]), "cpu_s": t_cpu, "cpu_threads": os.cpu_count(),
           "psnr_ref_db": oracle.psnr(img, ref)}
    # fp64 validation
    t0 = time.time()
    out64, tr = fsr.reconstruct(sampled, mask, B, N, I, reducer=reducer, precision="fp64",
                                return_trace=True)
    rec["gpu_fp64_call_s"] = time.time() - t0
    counts, div = oracle.compare_sequences(tr.selections[:, :I].astype(np.int64),
                                           rtr["sel"][:, :I].astype(np.int64), N)
    nb = rec["blocks"]
    split_ok, split_checked = 0, 0
    for b in np.nonzero(div)[0][:splits_cap]:
        ok, _, _ = oracle.coemaximal_split(sampled, mask, B, L, I, 0.7, 0.5, reducer, int(b),
                                           tr.selections[b])
        split_checked += 1
        split_ok += bool(ok)
    err64 = float(np.abs(out64 - ref).max()) / 255.0
    rec["fp64"] = {"equal": counts["equal"], "mirror": counts["mirror"],
                   "diverged": counts["diverged"],
                   "mirror_equal_pct": 100.0 * (counts["equal"] + counts["mirror"]) / nb,
                   "diverged_checked": split_checked, "diverged_proven_splits": split_ok,
                   "max_abs_err_0_1": err64,
                   "dpsnr_db": oracle.psnr(img, out64) - rec["psnr_ref_db"],
                   "known_exact": bool(np.array_equal(out64[mask], sampled[mask]))}
    # fp32 production on the reference's own f64 pixels
    t0 = time.time()
    out32, tr32 = fsr.reconstruct(sampled, mask, B, N, I, reducer=reducer, precision="fp32",
                                  return_trace=True)
    rec["gpu_fp32_call_s"] = time.time() - t0
    err32 = np.abs(out32 - ref)
    rec["fp32"] = {"max_abs_err_0_1": float(err32.max()) / 255.0,
                   "pixels_over_1e-3": int((err32 > 0.255).sum()),
                   "dpsnr_db": oracle.psnr(img, out32) - rec["psnr_ref_db"],
                   "rerun_blocks": int(tr32.stats["rerun_blocks"]),
                   "known_exact": bool(np.array_equal(out32[mask], sampled[mask]))}
    rec["pass"] = bool(rec["fp64"]["max_abs_err_0_1"] <= 1e-9 or split_ok == counts["diverged"]) and \
        rec["fp32"]["max_abs_err_0_1"] <= 1e-3 and abs(rec["fp32"]["dpsnr_db"]) <= 0.01
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", action="append", default=[])
    ap.add_argument("--support", type=int, default=32)
    ap.add_argument("--iterations", type=int, default=100)
    ap.add_argument("--image", default="natural", choices=["natural", "uniform"])
    ap.add_argument("--reducer", default="tree")
    ap.add_argument("--splits-cap", type=int, default=200)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "full_frame_parity.json"))
    args = ap.parse_args()
    shapes = args.shape or ["1080x1920"]
    recs = []
    for sh in shapes:
        H, W = (int(x) for x in sh.split("x"))
        r = run(H, W, args.support, args.iterations, 4, args.image, args.reducer, args.splits_cap)
        print(json.dumps(r), flush=True)
        recs.append(r)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "a") as fh:
        for r in recs:
            fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
