"""Run tools/micro/peak_flops (saturating FFMA / FFMA2 / DFMA) on the GPU box
with nvidia-smi clock sampling and write the measured non-tensor peaks that
bench.py divides by (profiles/r02/b200_fp_peaks.json).

  python tools/micro/peak_flops.py [--reps 40000] [--out profiles/r02/b200_fp_peaks.json]
"""

from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=40000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "b200_fp_peaks.json"))
    args = ap.parse_args()
    binary = os.path.join(HERE, "peak_flops")
    smi = subprocess.Popen(
        ["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
         "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "100"],
        stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    t0 = time.time()
    res = subprocess.run([binary, str(args.reps)], capture_output=True, text=True, check=True)
    wall = time.time() - t0
    time.sleep(0.2)
    smi.terminate()
    smi_out, _ = smi.communicate(timeout=5)
    print(res.stdout)
    rows = []
    pat = re.compile(r"(\S+)\s+warps/SMSP=\s*(\d+) chains=(\d+)\s+([\d.]+) ms\s+([\d.]+) MHz\s+"
                     r"([\d.]+) TFLOP/s\s+([\d.]+) warp-instr")
    for ln in res.stdout.splitlines():
        m = pat.search(ln)
        if m:
            rows.append({"form": m.group(1), "warps_per_smsp": int(m.group(2)),
                         "chains": int(m.group(3)), "ms": float(m.group(4)),
                         "sm_mhz": float(m.group(5)), "tflops": float(m.group(6)),
                         "warp_instr_per_clk_smsp": float(m.group(7))})
    clocks = []
    for ln in smi_out.strip().splitlines():
        f = [x.strip() for x in ln.split(",")]
        try:
            clocks.append((float(f[0]), float(f[1]), float(f[2]), f[3]))
        except (ValueError, IndexError):
            pass
    loaded = [c for c in clocks if c[2] > 300.0]
    full = {r["form"]: r for r in rows if r["warps_per_smsp"] == 16}
    out = {
        "fp32_tflops": max(full["FFMA"]["tflops"], full["FFMA2"]["tflops"]),
        "fp32_form": "FFMA2" if full["FFMA2"]["tflops"] >= full["FFMA"]["tflops"] else "FFMA",
        "fp32_ffma_scalar_tflops": full["FFMA"]["tflops"],
        "fp64_tflops": full["DFMA"]["tflops"],
        "how": ("tools/micro/peak_flops.cu: 148 x 2 CTAs x 1024 threads (16 warps/SMSP), 8 "
                "independent FMA chains per thread, best of 3 launches, CUDA events; "
                "an FMA = 2 flop, FFMA2 = 4 flop per lane"),
        "rows": rows,
        "clocks_under_load": {
            "samples": len(loaded),
            "sm_mhz_median": sorted(c[0] for c in loaded)[len(loaded) // 2] if loaded else None,
            "sm_max_mhz": max((c[1] for c in clocks), default=None),
            "power_w_max": max((c[2] for c in clocks), default=None),
            "reasons_seen": sorted({c[3] for c in loaded}),
        },
        "wall_s": wall,
    }
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: out[k] for k in ("fp32_tflops", "fp32_form", "fp64_tflops")}))


if __name__ == "__main__":
    main()
