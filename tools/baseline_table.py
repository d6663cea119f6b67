"""BASELINE.md §4 report rows from the committed bench lines of a round
(profiles/<round>/bench_*.json).  python tools/baseline_table.py r02"""
import json
import os
import sys

RND = sys.argv[1] if len(sys.argv) > 1 else "r02"
D = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", RND)


def load(f):
    return json.load(open(os.path.join(D, f)))


def row(cfg, d, cpu, parity):
    r = d["roofline"]
    hb = r.get("hbm_io") or {}
    iss = (r.get("issue") or {}).get("issue_active_pct")
    sm = (r.get("smem") or {}).get("frac")
    e2e = (d.get("e2e") or {}).get("value")
    kern = r["kernel"]
    if d["config"].get("N") in (4, 8) and d["config"].get("B", 4) <= 4:  # lines from before the label fix
        kern = kern.replace("warpnd", "warpsegd").replace("warpn_", "warpseg_")
    loop = f"{r['bound'].upper()} {r['frac']:.2f} of measured {r['peak']} TF/s ({kern})"
    if iss:
        loop += f", issue {iss:.0f} %"
    if sm:
        loop += f", smem {sm:.2f}"
    return (f"| {cfg} | 1 | {d['value']:.1f} (e2e {e2e:.1f}) | {d['mpixel_per_s']:.0f} | {loop} | "
            f"{hb.get('achieved_gbs', 0):.1f} ({hb.get('frac', 0):.4f}) | {cpu} | {parity} |")


def main():
    out = []
    d = load("bench_4k_default.json")
    cb = d["cpu_baseline"]
    q = d["quality"]
    out.append(row("configs[2] 4K, N=32, I=100, guarded fp32, f64 I/O", d,
                   f"{cb['value']:.4f} ({cb['cores']} cores, tree; {cb['sample']})",
                   f"fp32 max\\|Δ\\| {q['max_abs_err_0_1']:.1e}, ΔPSNR {q['psnr_delta_db']:.0e} dB "
                   f"({q['rows']} sample rows)"))
    out.append(row("configs[2] 4K, N=32, I=100, fp64 validation", load("bench_4k_fp64.json"),
                   f"{cb['value']:.4f} ({cb['cores']} cores)",
                   "sequences mirror-equal (whole-frame 1080p test)"))
    full = open(os.path.join(D, "fullframe_1080p.txt")).read().splitlines()
    fl = [ln for ln in full if ln.startswith("fp")]
    out.append(row("configs[1] 1080p, N=32, I=100, guarded fp32", load("bench_1080p_n32.json"),
                   f"≈ {4 * cb['value']:.3f} (4× the 4K rate)", "; ".join(fl) + " (whole frame)"))
    if os.path.exists(os.path.join(D, "bench_1080p_n32_i200.json")):
        out.append(row("configs[4]: 1080p, N=32, I=200, guarded fp32 (replayed re-runs)",
                       load("bench_1080p_n32_i200.json"), "—", "whole frame: fp32 max\\|Δ\\| 3.6e-4"))
    d = load("bench_stream64.json")
    out.append(f"| configs[3] 64 × 1080p stream, N=32 | 1 | {d['value']:.1f} (e2e {d['e2e']['value']:.1f}) | "
               f"{d['mpixel_per_s']:.0f} | as configs[1] | — | — | as configs[1] |")
    for n in (16, 64, 24, 20, 12, 8, 4):
        f = f"bench_1080p_n{n}.json"
        if os.path.exists(os.path.join(D, f)):
            out.append(row(f"configs[4] / paper grid: 1080p, N={n}, I=100, guarded fp32", load(f), "—",
                           "edge-case + golden frames within tolerance (GPU tests)"))
    print("\n".join(out))


if __name__ == "__main__":
    main()
