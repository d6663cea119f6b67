"""Summarise an ncu report of the FSR kernels into a committed JSON + text file.

Usage (here, after a gpurun capture brought the .ncu-rep back):
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01/warp32_ncu

Writes <out>.json (key metrics per launch, used by bench.py for roofline.traffic)
and <out>.txt (human summary: metrics, stall reasons, opcode mix, hot regions).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import Counter

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True,
                         check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = ncu_csv(rep, "--page", "raw")
    hdr, units = raw[0], raw[1]
    launches = []
    for row in raw[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                v = row[hdr.index(m)].replace(",", "")
                try:
                    d[m] = float(v)
                except ValueError:
                    d[m] = v
                d[m + ".unit"] = units[hdr.index(m)]
        stalls = {}
        for i, n in enumerate(hdr):
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
                try:
                    stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(row[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["stall_share"] = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda x: -x[1])
                            if v / tot >= 0.005}
        mb = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
        rd = d.get("dram__bytes_read.sum", 0.0) * mb.get(d.get("dram__bytes_read.sum.unit", "byte"), 1.0)
        wr = d.get("dram__bytes_write.sum", 0.0) * mb.get(d.get("dram__bytes_write.sum.unit", "byte"), 1.0)
        d["dram_bytes_per_launch"] = rd + wr
        launches.append(d)
    # per-instruction source page of the first launch: opcode mix and hot regions
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    shdr = src[1]
    ix = {n: i for i, n in enumerate(shdr)}
    rows = src[2:]
    ops, samp = Counter(), Counter()
    tot_e = sum(int(r[ix["Instructions Executed"]]) for r in rows) or 1
    tot_s = sum(int(r[ix["# Samples"]]) for r in rows) or 1
    for r in rows:
        t = r[ix["Source"]].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[op] += int(r[ix["Instructions Executed"]])
        samp[op] += int(r[ix["# Samples"]])
    summary = {"report": rep, "launches": launches,
               "opcode_mix": {k: round(v / tot_e, 4) for k, v in ops.most_common(20)},
               "opcode_samples": {k: round(samp[k] / tot_s, 4) for k, _ in ops.most_common(20)}}
    with open(out + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    with open(out + ".txt", "w") as f:
        for d in launches:
            f.write(f"kernel: {d['kernel']}\n")
            for m in METRICS:
                if m in d:
                    f.write(f"  {m:60s} {d[m]} {d.get(m + '.unit', '')}\n")
            f.write(f"  dram bytes per launch: {d['dram_bytes_per_launch']:.0f}\n")
            f.write("  stall share: " + ", ".join(f"{k} {v:.3f}" for k, v in d["stall_share"].items()) + "\n")
        f.write("opcode mix (executed share / sample share):\n")
        for k, v in summary["opcode_mix"].items():
            f.write(f"  {k:10s} {v:.4f} {summary['opcode_samples'][k]:.4f}\n")
    print(open(out + ".txt").read())


if __name__ == "__main__":
    main()
