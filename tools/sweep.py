"""BASELINE configs[4] sweep: iterations 50/100/200/500 x N = 16/32/64, and the
register-shuffle vs shared-memory (vs redux) argmax ablation.

Runs on one GPU through the C-ABI device entry point on a synthetic 1080p
quarter-sampled frame (natural image), strip-limited per case so each case
takes about a second; reports Mpixel/s and fps extrapolated to the full frame
(per-block cost is data-independent at fixed I), the fp64 re-run fraction of
the guarded fp32 mode, and the kernel that served the case.

    python tools/sweep.py [--precision fp32] > gpurun_out/sweep.jsonl
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--budget-ms", type=float, default=1000.0)
    ap.add_argument("--supports", default="16,32,64")
    ap.add_argument("--iterations", default="50,100,200,500")
    ap.add_argument("--argmax", default="shfl,smem,redux")
    args = ap.parse_args()

    import torch
    from paper_2202_13926_b200 import _lib, frames, synth

    H, W, B = args.height, args.width, 4
    img = synth.frame(H, W, 7, "natural")
    mask = frames.quarter_sample_mask(H, W, 42)
    dev = torch.device("cuda", 0)
    d_px = torch.from_numpy(np.where(mask, img, 0.0).astype(np.float32)).to(dev)
    d_mk = torch.from_numpy(mask.astype(np.uint8)).to(dev)
    d_out = torch.empty_like(d_px)
    eng = _lib.Engine([0])
    st = torch.cuda.current_stream()
    brows, bcols = -(-H // B), -(-W // B)

    def timed(p, rows, reps=1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.reconstruct_device(d_px.data_ptr(), W, d_mk.data_ptr(), W, H, W, 0, rows, d_out.data_ptr(), W,
                               p, st.cuda_stream, io="f32")
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(reps):
            eng.reconstruct_device(d_px.data_ptr(), W, d_mk.data_ptr(), W, H, W, 0, rows,
                                   d_out.data_ptr(), W, p, st.cuda_stream, io="f32")
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps, eng.last_stats()

    for N in [int(x) for x in args.supports.split(",")]:
        L = (N - B) // 2
        reducer = "linear" if N * N > 1024 else "tree"  # the tree reducer caps at 1024 records
        for I in [int(x) for x in args.iterations.split(",")]:
            for am in args.argmax.split(","):
                p = _lib.make_params(B, L, I, 0.7, 0.5, reducer, False, args.precision, am)
                ms4, _ = timed(p, 4)  # 4 block rows to size the strip
                rows = int(max(4, min(brows, 4 * args.budget_ms / max(ms4, 1e-3))))
                ms, stats = timed(p, rows)
                frame_ms = ms * brows / rows
                line = {"N": N, "B": B, "iterations": I, "argmax": am, "reducer": reducer,
                        "precision": args.precision, "rows_timed": rows, "frame": f"{W}x{H}",
                        "frame_ms": frame_ms, "fps": 1e3 / frame_ms,
                        "mpixel_per_s": H * W / (frame_ms * 1e-3) / 1e6,
                        "rerun_fraction": stats["rerun_blocks"] / max(1, rows * bcols),
                        # guarded fp32 beyond 300 iterations is served in fp64 (fsr_abi.cu)
                        "kernel": {(32, False): "warp32 (+pair64 re-runs)", (32, True): "pair64",
                                   (16, False): "warp16 (+warp16d re-runs)", (16, True): "warp16d",
                                   (64, False): "cta64, in-warp redux (+cta64d fp64 re-runs)",
                                   (64, True): "cta64d",
                                   (24, False): "warpn (+warpnd re-runs)", (24, True): "warpnd",
                                   (8, False): "warpseg, 4 blocks/warp (+warpsegd re-runs)",
                                   (8, True): "warpsegd",
                                   (4, False): "warpsegd (a guarded N=4 request is served in fp64)",
                                   (4, True): "warpsegd"}
                                  .get((N, args.precision == "fp64" or I > 300),
                                       ("warpnd" if args.precision == "fp64" or I > 300 else
                                        "warpn (+warpnd re-runs)") if N % 2 == 0 and N <= 20 else "generic")}
                line["served_fp64"] = stats.get("served_fp64")
                print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
